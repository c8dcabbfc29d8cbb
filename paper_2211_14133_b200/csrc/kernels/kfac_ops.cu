// Host launchers and the C-ABI (include/pf_kfac.h) of the K-FAC hot path:
//   curvature SYRK        bf16 tcgen05 (kind::f16), one grouped launch;
//   damped inverse        recursive blocked Cholesky + triangular inverse:
//                         128x128 diagonal blocks in shared memory (leaf.cuh),
//                         off-diagonal products as digit-form int8 tcgen05 GEMMs;
//   precondition/update   two chained digit-form GEMMs, W -= eta*P in the epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <atomic>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../host/capi_common.hpp"
#include "leaf.cuh"
#include "pf_kfac.h"
#include "pf_sched.h"
#include "slice.cuh"
#include "umma_gemm.cuh"

namespace pf {
namespace {

std::atomic<int64_t> g_launches{0};

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
using pf_detail::ShapeError;

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void after_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    check(cudaGetLastError(), what);
}

// Every kernel of this library is launched with programmatic stream
// serialisation (PDL): it may start while the previous kernel on the stream
// drains, runs its prologue (barrier init, TMEM alloc, descriptor prefetch),
// and calls ptx::grid_dep_wait() before touching any global data the previous
// kernel produced.  PF_NO_PDL=1 launches plainly (A/B measurement).
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PF_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

// Launch priority of the next launches (cudaLaunchAttributePriority; 0 = the
// stream's own).  The inversion marks its critical chain high and its side
// branches low, so that when a wide side GEMM holds every SM the block
// scheduler hands the next free SM to the critical kernel.  PF_NO_PRIO=1
// disables (A/B measurement).
thread_local int g_launch_prio = 0;

bool prio_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PF_NO_PRIO");
        return !(e && e[0] == '1');
    }();
    return on;
}

// (least, greatest) of the device's priority range, e.g. (0, -5)
std::pair<int, int> prio_range() {
    int least = 0, greatest = 0;
    check(cudaDeviceGetStreamPriorityRange(&least, &greatest), "cudaDeviceGetStreamPriorityRange");
    return {least, greatest};
}

struct ScopedPrio {
    int saved;
    explicit ScopedPrio(int p) : saved(g_launch_prio) { g_launch_prio = prio_enabled() ? p : 0; }
    ~ScopedPrio() { g_launch_prio = saved; }
};

// cluster_x > 1: thread-block clusters of cluster_x CTAs along x
template <typename... KArgs, typename... Args>
void launch_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                    int cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[3];
    int na = 0;
    if (cluster_x > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = static_cast<unsigned>(cluster_x);
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (g_launch_prio != 0) {
        attr[na].id = cudaLaunchAttributePriority;
        attr[na].val.priority = g_launch_prio;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

template <typename... KArgs, typename... Args>
void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
            Args&&... args) {
    launch_cluster(kernel, grid, block, smem, st, 1, std::forward<Args>(args)...);
}

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }
inline size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }
bool aligned16(const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; }

// ------------------------------------------------------------ TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable (driver too old / no GPU)");
    return fn;
}

// 2-D K-major tile map: `rows` rows of `k` elements, pitch `pitch_bytes`.
void encode(CUtensorMap* m, const void* ptr, bool bf16, int rows, int k, size_t pitch_bytes) {
    if (!aligned16(ptr) || pitch_bytes % 16 != 0)
        throw std::invalid_argument("TMA operand needs 16-byte aligned base and row pitch");
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch_bytes)};
    const cuuint32_t box[2] = {64, 128};  // 64 elements: 128 B bf16 rows / 64 B int8 rows
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encoder()(
        m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
        const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        bf16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

// MN-major bf16 operand [k x rows] (rows contiguous, pitch per k): dims
// {rows, k}, box {64, 64}; a 128-row tile is two boxes (umma_gemm.cuh).
void encode_mn(CUtensorMap* m, const void* ptr, int rows, int k, size_t pitch_bytes) {
    if (!aligned16(ptr) || pitch_bytes % 16 != 0)
        throw std::invalid_argument("TMA operand needs 16-byte aligned base and row pitch");
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(k)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch_bytes)};
    const cuuint32_t box[2] = {64, 64};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(mn) failed: " + std::to_string(r));
}

// 3-D map over the 4 digit planes of a sliced operand: dims {k, rows, plane},
// box {64, 128, 4} (one TMA per operand tile per k-block).
void encode_planes(CUtensorMap* m, const int8_t* planes, int rows, int k, int kpad, int64_t plane_stride,
                   int box_rows = 128) {
    if (!aligned16(planes) || kpad % 16 != 0 || plane_stride % 16 != 0)
        throw std::invalid_argument("digit planes need 16-byte aligned rows and planes");
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows), 4};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(kpad), static_cast<cuuint64_t>(plane_stride)};
    const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 4};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(planes), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled(3d) failed: " + std::to_string(r));
}

// ------------------------------------------------------------ digit form
struct Sliced {
    int8_t* planes = nullptr;
    int64_t plane_stride = 0;
    int rows = 0, k = 0, kpad = 0;
    int* exps = nullptr;
    double* sqnorm = nullptr;
};

size_t sliced_bytes(int rows, int k) {
    const size_t plane = align256(static_cast<size_t>(rows) * round_up(k, 16));
    return kDigits * plane + align256(static_cast<size_t>(rows) * 4) +
           align256(static_cast<size_t>(rows) * 8);
}

Sliced sliced_view(void* base, int rows, int k) {
    Sliced s;
    s.planes = static_cast<int8_t*>(base);
    s.rows = rows;
    s.k = k;
    s.kpad = round_up(k, 16);
    s.plane_stride = static_cast<int64_t>(align256(static_cast<size_t>(rows) * s.kpad));
    s.exps = reinterpret_cast<int*>(static_cast<char*>(base) + kDigits * s.plane_stride);
    s.sqnorm = reinterpret_cast<double*>(static_cast<char*>(base) + kDigits * s.plane_stride +
                                         align256(static_cast<size_t>(rows) * 4));
    return s;
}

// rows [r0, r0 + n) of a sliced operand (same planes, 16-byte aligned offset)
Sliced rows_of(const Sliced& s, int r0, int n) {
    Sliced t = s;
    t.planes = s.planes + static_cast<int64_t>(r0) * s.kpad;
    t.rows = n;
    t.exps = s.exps + r0;
    t.sqnorm = s.sqnorm + r0;
    return t;
}

struct SliceReq {
    const float* src;
    int ld;
    int mode;
    Sliced dst;
    const int* ready = nullptr;  // SliceJob::ready (slice_short only; the others wait for the launch)
};

// PF_READY_FLAGS=0: the chain's X_kk slice waits for the leaf launch to
// complete instead of for its published X (A/B switch)
bool ready_flags_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PF_READY_FLAGS");
        return !(e && e[0] == '0');
    }();
    return on;
}

// PF_DIAG_FP32=0: the right-looking chain's diagonal update of block k+1 as
// slice(L) + a one-tile digit GEMM on the chain (round-2 schedule) instead
// of one fp32 SIMT launch (diag_update_kernel) reading the TRSM's fp32
// output, the slice of L moved to the side branch.  Changes results by
// rounding (fp32 FMA sums instead of exact digit products; inverse residual
// 2.02e-6 vs 2.04e-6 at d = 4096).
bool diag_fp32_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PF_DIAG_FP32");
        return !(e && e[0] == '0');
    }();
    return on;
}

int diag_fp32_min_d() {
    static const int v = [] {
        const char* e = std::getenv("PF_DIAG_FP32_MIN_D");
        return e ? std::atoi(e) : 2048;
    }();
    return v;
}

bool warp_slice_2k() {  // PF_WARP_SLICE_2K=0: rows of 1025..2048 by the block-per-row kernel (A/B)
    static const bool on = [] {
        const char* e = std::getenv("PF_WARP_SLICE_2K");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool slice_short_enabled() {  // PF_SLICE_SHORT=0: rows <= 256 by the warp-per-row kernel (A/B)
    static const bool on = [] {
        const char* e = std::getenv("PF_SLICE_SHORT");
        return !(e && e[0] == '0');
    }();
    return on;
}

void launch_slices(const std::vector<SliceReq>& reqs, cudaStream_t st) {
    for (std::size_t i = 0; i < reqs.size(); i += kMaxSliceJobs) {
        SliceBatch b{};
        const int cnt = static_cast<int>(std::min<std::size_t>(kMaxSliceJobs, reqs.size() - i));
        int rows = 1, kmax = 0;
        for (int j = 0; j < cnt; ++j) {
            const SliceReq& r = reqs[i + j];
            b.j[j] = SliceJob{r.src, r.dst.rows, r.dst.k, r.ld, r.mode, r.dst.planes,
                              r.dst.plane_stride, r.dst.kpad, r.dst.exps, r.dst.sqnorm, r.ready};
            rows = std::max(rows, r.dst.rows);
            kmax = std::max(kmax, r.dst.k);
        }
        bool aligned = true;  // every row's valid range 16-byte aligned (ranges start at multiples of 128)
        for (int j = 0; j < cnt; ++j) {
            const SliceReq& r = reqs[i + j];
            aligned = aligned && aligned16(r.src) && r.ld % 4 == 0 && r.dst.k % 4 == 0 && r.dst.kpad % 4 == 0 &&
                      r.dst.plane_stride % 4 == 0 && aligned16(r.dst.planes);
        }
        if (kmax <= 256 && aligned && slice_short_enabled()) {  // 8 lanes per row
            launch(slice_short_kernel<8, 8>, dim3((rows + 31) / 32, cnt), dim3(256), 0, st, b);
            after_launch("slice_short_kernel");
        } else if (kmax > 1024 && kmax <= 2048 && warp_slice_2k()) {  // warp per row, 16 float4 per lane
            launch(slice_kernel<16>, dim3((rows + 7) / 8, cnt), dim3(256), 0, st, b);
            after_launch("slice_kernel");
        } else if (kmax > 1024 && kmax <= 4 * 128 * kLongVec) {
            launch(slice_long_kernel<128>, dim3(rows, cnt), dim3(128), 0, st, b);  // block of 128 per row
            after_launch("slice_long_kernel");
        } else if (kmax > 1024 && kmax <= 4 * kLongThreads * kLongVec) {  // block per row, one pass
            launch(slice_long_kernel<kLongThreads>, dim3(rows, cnt), dim3(kLongThreads), 0, st, b);
            after_launch("slice_long_kernel");
        } else {
            launch(slice_kernel<8>, dim3((rows + 7) / 8, cnt), dim3(256), 0, st, b);
            after_launch("slice_kernel");
        }
    }
}

// ------------------------------------------------------------ grouped GEMM
struct GemmSpec {
    // kBF16 operands
    const void* a_bf16 = nullptr;
    const void* b_bf16 = nullptr;
    int lda = 0, ldb = 0;
    // kOZ8 operands
    Sliced a, b;
    int rows = 0, cols = 0, k = 0;
    bool lower = false;
    int k_mode = K_FULL;
    float alpha = 1.0f, beta = 0.0f;
    uint32_t flags = 0;
    float* c = nullptr;
    float* c_t = nullptr;
    int ldc = 0, ldc_t = 0;
    const float* aux = nullptr;  // EPI_DIAG_SPLIT: X and X^T
    const float* aux_t = nullptr;
    int ld_aux = 0;
    bool mn_major = false;  // kBF16: a_bf16 / b_bf16 are [k x rows] with pitch lda / ldb
};

// GemmSpec -> GemmDesc, encoding its operand tensor maps at maps[*n_maps...]
// (tile_begin left to the caller).  Returns the number of maps used.
template <int kFmt, int kN = 128>
int make_desc(const GemmSpec& s, GemmDesc& d, CUtensorMap* maps, int n_maps) {
    using T = GemmTraits<kFmt, kN>;
    const bool shared_ab = kFmt == kBF16 ? (s.a_bf16 == s.b_bf16 && s.lda == s.ldb) : (s.a.planes == s.b.planes);
    int m = n_maps;
    auto put_maps = [&](bool is_a) {
        const int first = m;
        if constexpr (kFmt == kBF16) {
            if (s.mn_major)
                encode_mn(&maps[m++], is_a ? s.a_bf16 : s.b_bf16, is_a ? s.rows : s.cols, s.k,
                          static_cast<size_t>(is_a ? s.lda : s.ldb) * 2);
            else
                encode(&maps[m++], is_a ? s.a_bf16 : s.b_bf16, true, is_a ? s.rows : s.cols, s.k,
                       static_cast<size_t>(is_a ? s.lda : s.ldb) * 2);
        } else {
            const Sliced& o = is_a ? s.a : s.b;
            encode_planes(&maps[m++], o.planes, o.rows, o.k, o.kpad, o.plane_stride, is_a ? kTile : kN);
        }
        return first;
    };
    std::memset(&d, 0, sizeof(d));
    d.a_map = put_maps(true);
    // (bf16 boxes are 128 rows for both operands; digit-plane B boxes are kN rows)
    d.b_map = shared_ab && (kFmt == kBF16 || kN == kTile) ? d.a_map : put_maps(false);
    if (kFmt == kOZ8 && shared_ab) d.flags |= EPI_EXACT_DIAG;
    d.rows = s.rows;
    d.cols = s.cols;
    d.k = s.k;
    d.tiles_m = (s.rows + kTile - 1) / kTile;
    d.tiles_n = (s.cols + kN - 1) / kN;
    d.lower = s.lower ? (kN == 2 * kTile ? 2 : 1) : 0;  // 2: 128 x 256 lower tiles
    d.k_mode = s.k_mode;
    d.alpha = s.alpha;
    d.beta = s.beta;
    d.flags |= s.flags;
    d.a_exp = s.a.exps;
    d.b_exp = s.b.exps;
    d.a_sqnorm = s.a.sqnorm;
    d.c = s.c;
    d.c_t = s.c_t;
    d.ldc = s.ldc;
    d.ldc_t = s.ldc_t;
    d.aux = s.aux;
    d.aux_t = s.aux_t;
    d.ld_aux = s.ld_aux;
    d.mn_major = kFmt == kBF16 && s.mn_major ? 1 : 0;
    (void)sizeof(T);
    return m - n_maps;
}

inline int desc_tiles(const GemmDesc& d) {
    if (d.lower == 2) {  // row tile tm holds tm / 2 + 1 tiles of 256 columns
        const int a = d.tiles_m / 2;
        return a * (a + 1) + (d.tiles_m % 2 ? a + 1 : 0);
    }
    return d.lower ? d.tiles_m * (d.tiles_m + 1) / 2 : d.tiles_m * d.tiles_n;
}

int sm_count();

// Background calls (pf_set_background, per host thread): work issued to run
// UNDER a latency-bound chain on another stream (e.g. a layer's 1024-wide
// factors while its 4096-wide chains run).  Every launch of the call goes at
// the device's least priority and long-K GEMMs use one CTA per tile instead
// of persistent CTAs, so a critical kernel of the other stream gets the next
// free SM within one tile instead of after the whole persistent launch.
thread_local bool g_background = false;

bool gemm_persist_enabled() {  // PF_GEMM_PERSIST=0: one CTA per tile for long-K launches too (A/B)
    static const bool on = [] {
        const char* e = std::getenv("PF_GEMM_PERSIST");
        return !(e && e[0] == '0');
    }();
    return on && !g_background;
}

// Ticket counter of one persistent-GEMM launch (g_tickets, umma_gemm.cuh).
// The CTA that finishes last resets its slot, so a slot is free again once
// its launch has completed.  Eager launches rotate over kEagerSlots (two
// launches share a counter only if they are kEagerSlots launches apart AND
// run at the same time).  A launch captured into a CUDA graph bakes its slot
// into the graph, so it takes a slot of its own from the never-recycled
// range above: replays of that graph cannot collide with eager launches or
// with other captures (only a graph replayed concurrently with ITSELF would
// share a counter -- replay one graph on one stream at a time).
int ticket_slot(cudaStream_t stream) {
    static std::atomic<unsigned> next_eager{0};
    static std::atomic<unsigned> next_captured{0};
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    check(cudaStreamIsCapturing(stream, &cs), "cudaStreamIsCapturing");
    if (cs == cudaStreamCaptureStatusNone) return static_cast<int>(next_eager.fetch_add(1u) % kEagerSlots);
    const unsigned c = next_captured.fetch_add(1u);
    if (c >= static_cast<unsigned>(kTicketSlots - kEagerSlots))
        throw std::runtime_error("persistent GEMM: captured-launch ticket slots exhausted (" +
                                 std::to_string(kTicketSlots - kEagerSlots) + " per process)");
    return kEagerSlots + static_cast<int>(c);
}

// Split-K factor of a bf16 (SYRK) launch.  A CTA of the SYRK streams 32 KB
// of operands per 64-wide k-block through its SM, and one SM pulls ~100-120
// GB/s from L2 (measured: a lone 128x128 tile runs ~0.33 us per k-block, 4x
// its MMA time) -- so a launch of few tiles (a d = 1024 factor has 36) is
// bound by the bandwidth of the few SMs it occupies.  Splitting every tile's
// k-blocks over a cluster of 2 or 4 CTAs puts more SMs on it; the partial
// tiles are summed over DSMEM in a fixed order (umma_gemm.cuh
// split_k_epilogue), so results do not depend on timing.
//   4 slices: only while all CTAs get an SM of their own (tiles x 4 <=
//             0.8 SMs; a cluster must fit inside one GPC, and 4-CTA clusters
//             beyond that double up on SMs);
//   2 slices: while tiles x 2 <= 2 CTAs per SM (the kernel's occupancy);
// each slice keeps >= PF_KSPLIT_MINKB (default 8) k-blocks.  8-CTA clusters
// measured slower than 4 everywhere (ubench_syrk_splitk.txt).  PF_KSPLIT=n
// forces n (1 = off) for measurements.
int bf16_k_split(const GemmBatch& b, int tiles) {
    static const int force = [] { const char* e = std::getenv("PF_KSPLIT"); return e ? std::atoi(e) : 0; }();
    static const int min_kb = [] { const char* e = std::getenv("PF_KSPLIT_MINKB"); return e ? std::atoi(e) : 8; }();
    int kb = 1 << 30;
    for (int q = 0; q < b.n_probs; ++q) {
        if (b.probs[q].k_mode != K_FULL) return 1;
        kb = std::min(kb, (b.probs[q].k + 63) / 64);
    }
    if (force >= 1) {
        int f = 1;
        while (f * 2 <= std::min(force, 8)) f *= 2;
        return f;
    }
    const long sms = sm_count();
    if (static_cast<long>(tiles) * 4 * 5 <= sms * 4 && kb / 4 >= min_kb) return 4;
    if (static_cast<long>(tiles) * 2 <= 2 * sms && kb / 2 >= min_kb) return 2;
    return 1;
}

template <int kFmt, int kN, bool kSplit = false>
void launch_gemms_n(const std::vector<GemmSpec>& specs_in, cudaStream_t stream) {
    using T = GemmTraits<kFmt, kN>;
    auto kernel = umma_gemm_kernel<kFmt, kN, kSplit>;
    // Longest per-tile K first (problems of one launch are independent): the
    // block scheduler hands out CTAs roughly in blockIdx order, so long tiles
    // queued last would run as a tail on few SMs (the preconditioner mixes
    // K = 1024 and K = 4096 products in one launch).
    std::vector<GemmSpec> specs(specs_in);
    std::stable_sort(specs.begin(), specs.end(), [](const GemmSpec& a, const GemmSpec& b) { return a.k > b.k; });
    static std::once_flag attr_once;
    std::call_once(attr_once, [&] {
        check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, T::kSmemBytes),
              "cudaFuncSetAttribute(gemm)");
    });
    std::size_t i = 0;
    while (i < specs.size()) {
        GemmBatch batch;
        std::memset(&batch, 0, sizeof(batch));
        int maps = 0, probs = 0, tiles = 0;
        while (i < specs.size() && probs < kMaxProbs) {
            if (maps + 2 > kMaxMaps) break;
            GemmDesc& d = batch.probs[probs];
            maps += make_desc<kFmt, kN>(specs[i], d, batch.maps, maps);
            d.tile_begin = tiles;
            tiles += desc_tiles(d);
            ++probs;
            ++i;
        }
        batch.n_probs = probs;
        batch.total_tiles = tiles;
        batch.interleave = probs > 1 ? 1 : 0;
        for (int q = 1; q < probs; ++q) {
            const GemmDesc& a = batch.probs[0];
            const GemmDesc& b = batch.probs[q];
            if (desc_tiles(a) != desc_tiles(b) || a.k_mode != b.k_mode || a.lower != b.lower ||
                a.tiles_m != b.tiles_m || a.tiles_n != b.tiles_n || a.k != b.k)
                batch.interleave = 0;
        }
        if (tiles == 0) continue;
        if constexpr (kFmt == kOZ8 && kN == kTile) {
            // long-K launches with more tiles than SMs: persistent CTAs
            int kmin = 1 << 30;
            for (int q = 0; q < probs; ++q) kmin = std::min(kmin, batch.probs[q].k);
            static const int pk = [] { const char* e = std::getenv("PF_PERSIST_KMIN"); return e ? std::atoi(e) : 512; }();
            if (gemm_persist_enabled() && kmin > pk && tiles > sm_count()) {
                static std::once_flag once;
                std::call_once(once, [] {
                    check(cudaFuncSetAttribute(umma_gemm_persist_kernel<kSplit>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               T::kSmemBytes),
                          "cudaFuncSetAttribute(gemm persist)");
                });
                const int slot = ticket_slot(stream);
                launch(umma_gemm_persist_kernel<kSplit>, dim3(std::min(tiles, sm_count())), dim3(kPersistThreads),
                       T::kSmemBytes, stream, batch, slot);
                after_launch("umma_gemm_persist_kernel");
                continue;
            }
        }
        if constexpr (kFmt == kBF16 && kN == kTile) {
            batch.k_split = bf16_k_split(batch, tiles);
            if (batch.k_split > 1) {
                launch_cluster(kernel, dim3(tiles * batch.k_split), dim3(T::kThreads), T::kSmemBytes, stream,
                               batch.k_split, batch);
                after_launch("umma_gemm_kernel");
                continue;
            }
        }
        launch(kernel, dim3(tiles), dim3(T::kThreads), T::kSmemBytes, stream, batch);
        after_launch("umma_gemm_kernel");
    }
}

int sm_count() {
    thread_local int n = 0;
    if (!n) {
        int dev = 0;
        check(cudaGetDevice(&dev), "cudaGetDevice");
        check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    }
    return n;
}

// Tile width for a kOZ8 launch: a short-K, K_FULL, rectangular update whose
// 128-wide tiles would leave most SMs idle is split 2 or 4 ways along N
// (PF_NO_NSPLIT=1 disables, for A/B).
int pick_tile_n(const std::vector<GemmSpec>& specs) {
    static const bool off = [] {
        const char* e = std::getenv("PF_NO_NSPLIT");
        return e && e[0] == '1';
    }();
    if (off || specs.empty()) return kTile;
    long tiles = 0;
    for (const GemmSpec& g : specs) {
        if (g.k_mode != K_FULL || g.lower || (g.flags & EPI_MIRROR) || g.k > 512) return kTile;
        tiles += static_cast<long>((g.rows + kTile - 1) / kTile) * ((g.cols + kTile - 1) / kTile);
    }
    const int sms = sm_count();
    // a launch of at most sms / f32 (sms / f64) 128-wide tiles splits them 4 (2)
    // ways; re-tuned in round 2 with the faster leaf (layer inversion 2.49 ->
    // 2.44 ms against f32 = 4, f64 = 2) and again for the separate lead
    // chains of the fp32 diagonal update (f32 = f64 = 16 against 8 / 4:
    // layer 2.365 -> 2.331 ms, 4x4096 3.53 -> 3.36 ms); PF_NSPLIT32 /
    // PF_NSPLIT64 override
    static const int f32 = [] { const char* e = std::getenv("PF_NSPLIT32"); return e ? std::atoi(e) : 16; }();
    static const int f64 = [] { const char* e = std::getenv("PF_NSPLIT64"); return e ? std::atoi(e) : 16; }();
    if (tiles * f32 <= sms) return 32;
    if (tiles * f64 <= sms) return 64;
    return kTile;
}

// bf16 (SYRK) launches: 128 x 256 or 128 x 128 tiles, whichever needs fewer
// wave-times.  Both keep two CTAs per SM; all tiles of a SYRK launch have the
// same K, so a launch takes ceil(tiles / (2 SMs)) waves, and a 256-wide wave
// takes ~1.75x a 128-wide one (measured: d = 4096 alone, 1 wide wave 60 us
// against 2 narrow waves 69 us; the grouped 12-factor layer launch, 3 wide
// waves against 5 narrow, is ~2 % faster narrow).  Few 128-wide tiles: split
// over k instead (bf16_k_split).  PF_SYRK_WIDE=0: never 256-wide; =2: always.
void gemm_bf16(const std::vector<GemmSpec>& s, cudaStream_t st) {
    static const int wide = [] { const char* e = std::getenv("PF_SYRK_WIDE"); return e ? std::atoi(e) : 1; }();
    long narrow_tiles = 0, wide_tiles = 0;
    bool all_lower = true;
    for (const GemmSpec& g : s) {
        const long tm = (g.rows + kTile - 1) / kTile, a = tm / 2;
        narrow_tiles += g.lower ? tm * (tm + 1) / 2 : tm * ((g.cols + kTile - 1) / kTile);
        wide_tiles += a * (a + 1) + (tm % 2 ? a + 1 : 0);
        all_lower = all_lower && g.lower && g.k_mode == K_FULL;
    }
    const long slots = 2L * sm_count();
    const long nn = (narrow_tiles + slots - 1) / slots, nw = (wide_tiles + slots - 1) / slots;
    const bool use_wide = all_lower && (wide == 2 || (wide == 1 && narrow_tiles > sm_count() && 7 * nw < 4 * nn));
    if (use_wide)
        launch_gemms_n<kBF16, 2 * kTile>(s, st);
    else
        launch_gemms_n<kBF16, kTile>(s, st);
}
void gemm_oz8(const std::vector<GemmSpec>& s, cudaStream_t st) {
    if (!s.empty() && (s.front().flags & EPI_DIAG_SPLIT)) {  // the LAUUM (mirrored: 128-wide tiles)
        for (const GemmSpec& g : s)
            if (!(g.flags & EPI_DIAG_SPLIT)) throw std::logic_error("gemm_oz8: mixed EPI_DIAG_SPLIT launch");
        launch_gemms_n<kOZ8, 128, true>(s, st);
        return;
    }
    switch (pick_tile_n(s)) {
        case 32: launch_gemms_n<kOZ8, 32>(s, st); break;
        case 64: launch_gemms_n<kOZ8, 64>(s, st); break;
        default: launch_gemms_n<kOZ8, 128>(s, st);
    }
}

// ------------------------------------------------------------ small kernels
// dst = src + damping * I (lower triangle) of one factor
struct Damp2D {
    const float* src;
    float* dst;
    int* info;  // reset to 0 (success) before the factorisation
    int d, ld_src, ld_dst;
    float damping;
};
constexpr int kMaxDamp = 16;
struct DampBatch {
    Damp2D e[kMaxDamp];
};

constexpr int kDiagTiles = 36;
struct DiagUpd {
    const float* l;
    float* a;
    int ld;
    int n;
};
struct DiagBatch {
    DiagUpd e[kMaxLeafBatch];
};
__global__ void __launch_bounds__(256) diag_update_kernel(const __grid_constant__ DiagBatch b) {
    __shared__ float sa[kLeaf][33], sb[kLeaf][33];
    const DiagUpd& P = b.e[blockIdx.y];
    int ti = 0, tj = blockIdx.x;
    while (tj > ti) tj -= ++ti;
    const int tid = threadIdx.x;
    ptx::grid_dep_wait();
    ptx::grid_dep_launch();
    if (32 * tj >= P.n) return;
    float va[16], vb[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int r = (tid >> 5) + 8 * (q & 3), k = (tid & 31) + 32 * (q >> 2);
        const int ra = 32 * ti + r, rb = 32 * tj + r;
        va[q] = ra < P.n ? __ldcg(P.l + (size_t)ra * P.ld + k) : 0.0f;
        vb[q] = rb < P.n ? __ldcg(P.l + (size_t)rb * P.ld + k) : 0.0f;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int r = (tid >> 5) + 8 * (q & 3), k = (tid & 31) + 32 * (q >> 2);
        sa[k][r] = va[q];
        sb[k][r] = vb[q];
    }
    __syncthreads();
    const int ri = 2 * (tid >> 4), cj = 2 * (tid & 15);
    float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll 16
    for (int k = 0; k < kLeaf; ++k) {
        const float a0 = sa[k][ri], a1 = sa[k][ri + 1], b0 = sb[k][cj], b1 = sb[k][cj + 1];
        acc[0][0] = fmaf(a0, b0, acc[0][0]);
        acc[0][1] = fmaf(a0, b1, acc[0][1]);
        acc[1][0] = fmaf(a1, b0, acc[1][0]);
        acc[1][1] = fmaf(a1, b1, acc[1][1]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const int r = 32 * ti + ri + u, c = 32 * tj + cj + v;
            if (r < P.n && c <= r) {
                float* d = P.a + (size_t)r * P.ld + c;
                *d = fmaf(-1.0f, acc[u][v], *d);
            }
        }
}

// dst = M + damping * I, lower triangle incl. diagonal (the rest is never
// read; whole float4 groups are copied).  One warp per row, 8 rows per CTA.
__global__ void __launch_bounds__(256) damp_kernel(const __grid_constant__ DampBatch b) {
    const Damp2D& s = b.e[blockIdx.y];
    ptx::grid_dep_wait();
    ptx::grid_dep_launch();
    if (blockIdx.x == 0 && threadIdx.x == 0) *s.info = 0;
    const int r = blockIdx.x * 8 + static_cast<int>(threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= s.d) return;
    const float* src = s.src + static_cast<int64_t>(r) * s.ld_src;
    float* dst = s.dst + static_cast<int64_t>(r) * s.ld_dst;
    const bool vec = (s.ld_src % 4 == 0) && (s.ld_dst % 4 == 0) && ((reinterpret_cast<uintptr_t>(s.src) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(s.dst) & 15) == 0);
    if (vec) {
        // four float4 per lane in flight per round (the rows are long: a
        // one-load-per-iteration loop is latency-bound)
        const int n4 = (r + 4) / 4;  // float4 groups covering columns [0, r]
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(dst);
        for (int b = 0; b < n4; b += 128) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c4 = b + lane + 32 * u;
                v[u] = c4 < n4 ? __ldcg(s4 + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c4 = b + lane + 32 * u;
                if (c4 >= n4) continue;
                if (c4 == r / 4) {
                    const int e = r % 4;
                    if (e == 0) v[u].x += s.damping;
                    if (e == 1) v[u].y += s.damping;
                    if (e == 2) v[u].z += s.damping;
                    if (e == 3) v[u].w += s.damping;
                }
                d4[c4] = v[u];
            }
        }
    } else {
        for (int c = lane; c <= r; c += 32) dst[c] = __ldcg(src + c) + (c == r ? s.damping : 0.0f);
    }
}

__global__ void f32_to_bf16_kernel(const float* x, int64_t n, __nv_bfloat16* out) {
    ptx::grid_dep_wait();
    ptx::grid_dep_launch();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __float2bfloat16_rn(x[i]);
}

// pf_cholesky_factor: L = the leaves' diagonal blocks (already in `l`) + the
// strictly-lower blocks of the right-looking factorisation (w.l), zeros above
__global__ void assemble_l_kernel(const float* __restrict__ wl, int ldw, float* __restrict__ l, int ldl, int d) {
    const int i = blockIdx.x;
    const int diag0 = i / kLeaf * kLeaf;  // first column of row i's diagonal block
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        if (j > i)
            l[static_cast<size_t>(i) * ldl + j] = 0.0f;
        else if (j < diag0)
            l[static_cast<size_t>(i) * ldl + j] = wl[static_cast<size_t>(i) * ldw + j];
    }
}

// ------------------------------------------------------------ damped inverse
// Workspace of one factor (ld = round_up(d, 4)):
//   fp32  A (damped factor, updated in place), L (panel blocks L21),
//         X = L^-1 (lower), XT = L^-T (upper), T^T of every recursion depth
//   digit form  two operand slots S0, S1 sized for d x d, plus two per depth
//               for the side branch
struct InvWs {
    int d = 0, ld = 0;
    float *a, *l, *x, *xt, *t;
    void* s0;
    void* s1;
    // per-recursion-depth digit slots of the node's side branch (T^T = (L21 X11)^T
    // runs concurrently with the recursion on A22, so nested nodes must not share)
    void* side0[8] = {};
    void* side1[8] = {};
    int t_row[8] = {};  // row of w.t where the depth's T^T lives (ld = w.ld)
    // right-looking factorisation: per-panel digit slots (3-deep ring) for the
    // A panel, the leaf inverse X_kk and the L panel
    void* pa[3] = {};
    void* px[3] = {};
    void* pl[3] = {};
    int* info = nullptr;
    int* ready = nullptr;   // one flag per 128-column panel (LeafArgs::ready)
    float* lout = nullptr;  // pf_cholesky_factor: leaves also write their block of L here
    int ldl = 0;
};

// n1 bound of the internal nodes, depth by depth (left child is the larger)
std::vector<int> node_n1_bounds(int d) {
    std::vector<int> b;
    for (int n = d; n > kLeaf; n = kTile * ((n + 2 * kTile - 1) / (2 * kTile))) b.push_back(kTile * ((n + 2 * kTile - 1) / (2 * kTile)));
    if (b.size() > 8) throw std::invalid_argument("damped inverse: d too large");
    return b;
}

// T^T of every depth, stacked: sum of the depth bounds (can exceed d: the
// left child takes the larger part, e.g. d = 300 -> 256 + 128 rows)
int t_rows(int d) {
    int r = 0;
    for (int n1 : node_n1_bounds(d)) r += n1;
    return std::max(r, d);  // >= d: the bottom-up TRTRI keeps T^T of node (o, n) at rows [o, o + n1)
}

size_t inverse_ws_bytes(int d) {
    const size_t plane = align256(static_cast<size_t>(round_up(d, 4)) * d * sizeof(float));
    const size_t tplane = align256(static_cast<size_t>(round_up(d, 4)) * t_rows(d) * sizeof(float));
    size_t side = 0;
    for (int n1 : node_n1_bounds(d)) side += 2 * align256(sliced_bytes(n1, n1));
    const size_t panel = 2 * align256(sliced_bytes(d, kLeaf)) + align256(sliced_bytes(kLeaf, kLeaf));
    const size_t flags = align256(static_cast<size_t>((d + kLeaf - 1) / kLeaf) * sizeof(int));
    return 4 * plane + tplane + 2 * align256(sliced_bytes(d, d)) + side + 3 * panel + flags;
}

InvWs carve(void* base, int d) {
    InvWs w;
    w.d = d;
    w.ld = round_up(d, 4);
    const size_t plane = align256(static_cast<size_t>(w.ld) * d * sizeof(float));
    const size_t tplane = align256(static_cast<size_t>(w.ld) * t_rows(d) * sizeof(float));
    char* p = static_cast<char*>(base);
    float** f[4] = {&w.a, &w.l, &w.x, &w.xt};
    for (int i = 0; i < 4; ++i) *f[i] = reinterpret_cast<float*>(p + i * plane);
    w.t = reinterpret_cast<float*>(p + 4 * plane);
    p += 4 * plane + tplane;
    w.s0 = p;
    w.s1 = p + align256(sliced_bytes(d, d));
    char* q = p + 2 * align256(sliced_bytes(d, d));
    int row = 0;
    const std::vector<int> b = node_n1_bounds(d);
    for (std::size_t k = 0; k < b.size(); ++k) {
        w.side0[k] = q;
        q += align256(sliced_bytes(b[k], b[k]));
        w.side1[k] = q;
        q += align256(sliced_bytes(b[k], b[k]));
        w.t_row[k] = row;  // T^T of a depth-k node: n1 <= b[k] rows
        row += b[k];
    }
    for (int i = 0; i < 3; ++i) {
        w.pa[i] = q;
        q += align256(sliced_bytes(d, kLeaf));
        w.pl[i] = q;
        q += align256(sliced_bytes(d, kLeaf));
        w.px[i] = q;
        q += align256(sliced_bytes(kLeaf, kLeaf));
    }
    w.ready = reinterpret_cast<int*>(q);  // reset by each leaf before use: no initialisation needed
    return w;
}

float* at(float* base, int ld, int r, int c) { return base + static_cast<size_t>(r) * ld + c; }

// The inversion is written once against an Emitter (StreamEmitter: one
// PDL launch per step on a stream, fork/join and event edges to side streams).
// (A persistent task-graph executor behind the same interface was measured
// 1.3-2x slower -- cold instruction cache in the leaf, serialised epilogues --
// and removed in round 2.)
struct Emitter {
    virtual ~Emitter() = default;
    virtual void damp(const std::vector<Damp2D>& jobs) = 0;
    virtual void slices(const std::vector<SliceReq>& reqs) = 0;
    virtual void gemms(const std::vector<GemmSpec>& specs) = 0;
    // publish: each leaf releases its panel's `ready` flag once X is stored
    // (the right-looking chain's slice of X_kk starts on it)
    virtual void leaves(const std::vector<InvWs>& ws, int o, int n, bool publish = false) = 0;
    virtual void diag_updates(const std::vector<InvWs>& ws, int r0, int n, int c) = 0;
    // work emitted between side_begin(k) and side_end(k) may run concurrently
    // with what follows on the main chain until side_join(k)
    virtual void side_begin(int) {}
    virtual void side_end(int) {}
    virtual void side_join(int) {}
    // explicit stream/event form for DAGs the fork/join pairs cannot express:
    // on(s) directs what follows to stream s (0 = main), record(e) / wait(e)
    // mark and await event e.  Program order must itself be a valid
    // sequential order (the persistent back end ignores all three).
    virtual void on(int) {}
    virtual void record(int) {}
    virtual void wait(int) {}
    // lead chain progress mark (shorter groups of the same call start there)
    virtual void mark_lead(int /*panel*/, int /*panels*/) {}
};

// A group with a SHORTER chain than the lead (smaller d) of a right-looking
// call starts when the lead's factorisation reaches panel nb_lead - 1.5 nb_g
// (PF_DELAY_MUL, re-tuned in round 2; was 2 nb_g):
// started together it takes SMs from the lead's launch-latency-bound chain for
// its whole length; started late it still finishes before the lead's TRTRI /
// LAUUM tail (2x4096 + 10x1024, start panel of the 1024 groups: 0 -> 2.79 ms,
// 4: 2.77, 10: 2.74, 16: 2.72, 22: 2.72, 28: 2.93).  PF_INV_DELAY=0 disables.
bool lead_delay_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PF_INV_DELAY");
        return !(e && e[0] == '0');
    }();
    return on;
}
constexpr int kMarkGroup = 1000;  // pool_event(kMarkGroup, panel): lead progress marks
thread_local int g_lead_panels = 0;  // panels marked by the lead group of the current call

// Per-thread, per-device pool of (stream, done event) pairs for the side
// branches of the recursion, indexed by (group slot, depth).
struct SideSlot {
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, done = nullptr;
};

SideSlot& side_slot(int group, int depth) {
    thread_local std::vector<std::vector<SideSlot>> pools;  // [device][group * 16 + slot]
    int dev = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    if (pools.size() <= static_cast<std::size_t>(dev)) pools.resize(dev + 1);
    auto& v = pools[dev];
    const std::size_t i = static_cast<std::size_t>(group) * 16 + depth;
    if (v.size() <= i) v.resize(i + 1);
    SideSlot& sl = v[i];
    if (!sl.stream) {
        check(cudaStreamCreateWithFlags(&sl.stream, cudaStreamNonBlocking), "cudaStreamCreate(side)");
        check(cudaEventCreateWithFlags(&sl.fork, cudaEventDisableTiming), "cudaEventCreate(side)");
        check(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming), "cudaEventCreate(side)");
    }
    return sl;
}

cudaEvent_t pool_event(int group, int id) {
    thread_local std::vector<std::vector<cudaEvent_t>> pools;  // [device][group * 32 + id]
    int dev = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    if (pools.size() <= static_cast<std::size_t>(dev)) pools.resize(dev + 1);
    auto& v = pools[dev];
    const std::size_t i = static_cast<std::size_t>(group) * 32 + id;
    if (v.size() <= i) v.resize(i + 1, nullptr);
    if (!v[i]) check(cudaEventCreateWithFlags(&v[i], cudaEventDisableTiming), "cudaEventCreate(pool)");
    return v[i];
}

LeafArgs leaf_args(const InvWs& w, int o, int n) {
    LeafArgs a{at(w.a, w.ld, o, o), at(w.x, w.ld, o, o), at(w.xt, w.ld, o, o), w.info, w.ld, n, o};
    if (w.lout) {
        a.l = at(w.lout, w.ldl, o, o);
        a.ldl = w.ldl;
    }
    return a;
}


struct StreamEmitter final : Emitter {
    cudaStream_t st;
    cudaStream_t main;
    int group;
    int prio_main, prio_side, prio;  // launch priorities: critical chain high, side branches low
    // `lead`: the group has the largest factor size of the call (the longest
    // chain).  Only lead chains get the top priority; the shorter groups run
    // entirely at the lowest, filling the SMs the lead chain leaves idle
    // (2x4096 + 10x1024: 3.07 -> 2.97 ms).
    explicit StreamEmitter(cudaStream_t s, int g = 0, bool lead = true) : st(s), main(s), group(g) {
        const auto [least, greatest] = prio_range();
        prio_main = prio = lead && !g_background ? greatest : least;
        prio_side = least;
    }
    void side_begin(int depth) override {
        SideSlot& sl = side_slot(group, depth);
        check(cudaEventRecord(sl.fork, main), "cudaEventRecord(side fork)");
        check(cudaStreamWaitEvent(sl.stream, sl.fork, 0), "side fork");
        st = sl.stream;
        prio = prio_side;
    }
    void side_end(int depth) override {
        SideSlot& sl = side_slot(group, depth);
        check(cudaEventRecord(sl.done, sl.stream), "cudaEventRecord(side done)");
        st = main;
        prio = prio_main;
    }
    void side_join(int depth) override {
        check(cudaStreamWaitEvent(main, side_slot(group, depth).done, 0), "side join");
    }
    void mark_lead(int panel, int panels) override {
        if (group != 0 || !lead_delay_enabled()) return;
        check(cudaEventRecord(pool_event(kMarkGroup, panel), main), "cudaEventRecord(lead mark)");
        g_lead_panels = std::max(g_lead_panels, std::min(panel + 1, panels));
    }
    void on(int s) override {
        st = s == 0 ? main : side_slot(group, 11 + s).stream;
        prio = s == 0 ? prio_main : prio_side;
    }
    void record(int e) override { check(cudaEventRecord(pool_event(group, e), st), "cudaEventRecord(pool)"); }
    void wait(int e) override { check(cudaStreamWaitEvent(st, pool_event(group, e), 0), "cudaStreamWaitEvent(pool)"); }
    void damp(const std::vector<Damp2D>& jobs) override {
        DampBatch db{};
        int d = 1;
        for (std::size_t i = 0; i < jobs.size(); ++i) {
            db.e[i] = jobs[i];
            d = std::max(d, jobs[i].d);
        }
        ScopedPrio sp(prio);
        launch(damp_kernel, dim3((d + 7) / 8, static_cast<unsigned>(jobs.size())), dim3(256), 0, st, db);
        after_launch("damp_kernel");
    }
    void slices(const std::vector<SliceReq>& reqs) override {
        ScopedPrio sp(prio);
        launch_slices(reqs, st);
    }
    void gemms(const std::vector<GemmSpec>& specs) override {
        ScopedPrio sp(prio);
        gemm_oz8(specs, st);
    }
    void diag_updates(const std::vector<InvWs>& ws, int r0, int n, int c) override {
        ScopedPrio sp(prio);
        for (std::size_t i = 0; i < ws.size(); i += kMaxLeafBatch) {
            DiagBatch b{};
            const int cnt = static_cast<int>(std::min<std::size_t>(kMaxLeafBatch, ws.size() - i));
            for (int j = 0; j < cnt; ++j)
                b.e[j] = DiagUpd{at(ws[i + j].l, ws[i + j].ld, r0, c), at(ws[i + j].a, ws[i + j].ld, r0, r0),
                                 ws[i + j].ld, n};
            launch(diag_update_kernel, dim3(kDiagTiles, cnt), dim3(256), 0, st, b);
            after_launch("diag_update_kernel");
        }
    }
    void leaves(const std::vector<InvWs>& ws, int o, int n, bool publish = false) override {
        ScopedPrio sp(prio);
        static std::once_flag once;
        std::call_once(once, [] {
            check(cudaFuncSetAttribute(leaf_chol_inv_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kLeafSmemBytes),
                  "cudaFuncSetAttribute(leaf)");
            check(cudaFuncSetAttribute(leaf_chol_inv_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kLeafSmemBytes),
                  "cudaFuncSetAttribute(leaf)");
        });
        for (std::size_t i = 0; i < ws.size(); i += kMaxLeafBatch) {
            LeafBatch b{};
            const int cnt = static_cast<int>(std::min<std::size_t>(kMaxLeafBatch, ws.size() - i));
            bool with_l = false;
            for (int j = 0; j < cnt; ++j) {
                b.e[j] = leaf_args(ws[i + j], o, n);
                if (publish && ready_flags_enabled()) b.e[j].ready = ws[i + j].ready + o / kLeaf;
                with_l = with_l || b.e[j].l;
            }
            if (with_l) {
                for (int j = 0; j < cnt; ++j)
                    if (!b.e[j].l) throw std::invalid_argument("leaf batch mixes factor-only and inverse problems");
                launch(leaf_chol_inv_kernel<true>, dim3(cnt), dim3(kLeafThreads), kLeafSmemBytes, st, b);
            } else {
                launch(leaf_chol_inv_kernel<false>, dim3(cnt), dim3(kLeafThreads), kLeafSmemBytes, st, b);
            }
            after_launch("leaf_chol_inv_kernel");
        }
    }
};

// Slice [rows x k] at (r0, c0) of `src` into slot `slot`.
SliceReq slice_of(float* src, int ld, int r0, int c0, int rows, int k, void* slot, int mode) {
    return SliceReq{at(src, ld, r0, c0), ld, mode, sliced_view(slot, rows, k)};
}

// Recursive blocked Cholesky + triangular inverse of the diagonal block
// [o, o+n) of every workspace (all of equal d).  On return X = L^-1 and
// XT = L^-T hold that block.  Per level (n = n1 + n2):
//   L21  = A21 X11^T            (TRSM as a GEMM with the block inverse)
//   A22 -= L21 L21^T            (SYRK, lower tiles)
//   recurse on A22
//   T^T  = (L21 X11)^T          (via XT11)
//   X21  = -X22 T,  XT12 = X21^T
// `pending`: depth of an ancestor side branch that still updates this node's
// A21 / A22 (the parent's look-ahead), joined before this node's first GEMM.
void inverse_rec(const std::vector<InvWs>& ws, int o, int n, Emitter& em, int depth = 0, int pending = -1) {
    if (n <= kLeaf) {
        em.leaves(ws, o, n);
        return;
    }
    const int n1 = kTile * ((n + 2 * kTile - 1) / (2 * kTile));
    const int n2 = n - n1;
    // look-ahead: when A22 is itself an internal node, only its top-left
    // n1' x n1' block must be updated before the recursion descends into it;
    // the rest of the trailing update joins the side branch
    const int n1c = kTile * ((n2 + 2 * kTile - 1) / (2 * kTile));
    const bool split = n2 > kLeaf;
    inverse_rec(ws, o, n1, em, depth + 1);
    if (pending >= 0) em.side_join(pending);

    std::vector<SliceReq> sl;
    std::vector<GemmSpec> g;
    // ---- L21 = A21 X11^T
    for (const InvWs& w : ws) {
        sl.push_back(slice_of(w.a, w.ld, o + n1, o, n2, n1, w.s0, SLICE_FULL));
        sl.push_back(slice_of(w.x, w.ld, o, o, n1, n1, w.s1, SLICE_LOWER_BLOCK));
        GemmSpec s;
        s.a = sliced_view(w.s0, n2, n1);
        s.b = sliced_view(w.s1, n1, n1);
        s.rows = n2;
        s.cols = n1;
        s.k = n1;
        s.k_mode = K_TO_COL_TILE_END;
        s.flags = EPI_VEC4;
        s.c = at(w.l, w.ld, o + n1, o);
        s.ldc = w.ld;
        g.push_back(s);
    }
    em.slices(sl);
    em.gemms(g);
    // ---- side branch: T^T = (L21 X11)^T (B operand rows = XT11, upper
    // block-triangular) only needs L21 and X11, so it runs concurrently with
    // the trailing update and the recursion on A22; depth-private buffers
    em.side_begin(depth);
    sl.clear();
    g.clear();
    for (const InvWs& w : ws) {
        sl.push_back(slice_of(w.l, w.ld, o + n1, o, n2, n1, w.side0[depth], SLICE_FULL));
        sl.push_back(slice_of(w.xt, w.ld, o, o, n1, n1, w.side1[depth], SLICE_UPPER_BLOCK));
        GemmSpec s;
        s.a = sliced_view(w.side0[depth], n2, n1);
        s.b = sliced_view(w.side1[depth], n1, n1);
        s.rows = n2;
        s.cols = n1;
        s.k = n1;
        s.k_mode = K_FROM_COL_TILE;
        s.flags = EPI_TRANSPOSE;
        s.c = at(w.t, w.ld, w.t_row[depth], 0);  // T^T [n1 x n2]
        s.ldc = w.ld;
        g.push_back(s);
    }
    if (split) {  // the rest of A22 -= L21 L21^T (rows n1c .. n2), from the side's L21 digits
        for (const InvWs& w : ws) {
            const Sliced l21 = sliced_view(w.side0[depth], n2, n1);
            GemmSpec a;  // A22[n1c:, :n1c] -= L21[n1c:] L21[:n1c]^T
            a.a = rows_of(l21, n1c, n2 - n1c);
            a.b = rows_of(l21, 0, n1c);
            a.rows = n2 - n1c;
            a.cols = n1c;
            a.k = n1;
            a.alpha = -1.0f;
            a.beta = 1.0f;
            a.flags = EPI_VEC4;
            a.c = at(w.a, w.ld, o + n1 + n1c, o + n1);
            a.ldc = w.ld;
            g.push_back(a);
            GemmSpec b;  // A22[n1c:, n1c:] -= L21[n1c:] L21[n1c:]^T  (lower)
            b.a = rows_of(l21, n1c, n2 - n1c);
            b.b = b.a;
            b.rows = b.cols = n2 - n1c;
            b.k = n1;
            b.lower = true;
            b.alpha = -1.0f;
            b.beta = 1.0f;
            b.flags = EPI_VEC4;
            b.c = at(w.a, w.ld, o + n1 + n1c, o + n1 + n1c);
            b.ldc = w.ld;
            g.push_back(b);
        }
    }
    em.slices(sl);
    em.gemms(g);
    em.side_end(depth);
    // ---- A22 -= L21 L21^T  (look-ahead: only the top-left n1c x n1c block here)
    sl.clear();
    g.clear();
    const int nu = split ? n1c : n2;
    for (const InvWs& w : ws) {
        sl.push_back(slice_of(w.l, w.ld, o + n1, o, nu, n1, w.s0, SLICE_FULL));
        GemmSpec s;
        s.a = sliced_view(w.s0, nu, n1);
        s.b = s.a;
        s.rows = s.cols = nu;
        s.k = n1;
        s.lower = true;
        s.alpha = -1.0f;
        s.beta = 1.0f;
        s.flags = EPI_VEC4;
        s.c = at(w.a, w.ld, o + n1, o + n1);
        s.ldc = w.ld;
        g.push_back(s);
    }
    em.slices(sl);
    em.gemms(g);

    inverse_rec(ws, o + n1, n2, em, depth + 1, split ? depth : -1);

    // ---- X21 = -X22 T  (B operand rows = T^T), also stored as XT12
    em.side_join(depth);
    sl.clear();
    g.clear();
    for (const InvWs& w : ws) {
        sl.push_back(slice_of(w.x, w.ld, o + n1, o + n1, n2, n2, w.s0, SLICE_LOWER_BLOCK));
        sl.push_back(slice_of(w.t, w.ld, w.t_row[depth], 0, n1, n2, w.s1, SLICE_FULL));
        GemmSpec s;
        s.a = sliced_view(w.s0, n2, n2);
        s.b = sliced_view(w.s1, n1, n2);
        s.rows = n2;
        s.cols = n1;
        s.k = n2;
        s.k_mode = K_TO_ROW_TILE_END;
        s.alpha = -1.0f;
        s.flags = EPI_ALSO_T | EPI_VEC4;
        s.c = at(w.x, w.ld, o + n1, o);
        s.ldc = w.ld;
        s.c_t = at(w.xt, w.ld, o, o + n1);
        s.ldc_t = w.ld;
        g.push_back(s);
    }
    em.slices(sl);
    em.gemms(g);
}

// ------------------------------------------------------------ right-looking Cholesky + TRTRI
// Side-slot indices: 0..7 the TRTRI depths, 12..13 the panel side streams (on(1), on(2)).

// Blocked right-looking Cholesky with a two-level look-ahead, 128-column
// panels.  Per panel k the CRITICAL chain (main stream) is
//   leaf(k) -> slice X_kk -> TRSM L[>k, k] = A[>k, k] X_kk^T -> slice L
//   -> A[k+1, k+1] -= L[k+1, k] L[k+1, k]^T (one tile) -> leaf(k+1)
// and everything else runs on two alternating side streams R(k % 2):
//   col  A[>k+1, k+1] -= L[>k+1, k] L[k+1, k]^T, then slice that column
//        (the A panel of k+1, awaited before TRSM(k+1))      -> event A
//   BU   block column k+2 (awaited by the diagonal update and col of k+1) -> U
//   BR   the rest, columns >= k+3, lower (awaited by BU(k+1))             -> B
// so the trailing update overlaps leaf(k+1) instead of preceding it.
// w.l receives the strictly-lower L, w.x / w.xt the diagonal blocks of L^-1.
void cholesky_blocked(const std::vector<InvWs>& ws, Emitter& em,
                      const std::function<void(int)>& after_leaf = nullptr) {
    const int d = ws.front().d;
    const int nb = (d + kLeaf - 1) / kLeaf;
    // event ids (pool_event, 32 per group): F fork, A/U/B rings of 2, END per side stream;
    // 29-30 are the early-TRTRI fork/done (damped_inverse_group)
    auto evA = [](int k) { return 1 + (k & 1); };
    auto evU = [](int k) { return 3 + (k & 1); };
    auto evB = [](int k) { return 5 + (k & 1); };
    constexpr int evF = 0, evEnd0 = 7;
    auto update = [](const InvWs& w, const Sliced& a, const Sliced& b, int rows, int cols, int r, int c,
                     bool lower) {
        GemmSpec u;
        u.a = a;
        u.b = b;
        u.rows = rows;
        u.cols = cols;
        u.k = kLeaf;
        u.lower = lower;
        u.alpha = -1.0f;
        u.beta = 1.0f;
        u.flags = EPI_VEC4;
        u.c = at(w.a, w.ld, r, c);
        u.ldc = w.ld;
        return u;
    };
    std::vector<SliceReq> sl;
    std::vector<GemmSpec> g;
    if (nb > 1) {  // A panel of panel 0
        for (const InvWs& w : ws) sl.push_back(slice_of(w.a, w.ld, kLeaf, 0, d - kLeaf, kLeaf, w.pa[0], SLICE_FULL));
        em.slices(sl);
    }
    bool side_used[2] = {false, false};
    for (int k = 0; k < nb; ++k) {
        const int o = k * kLeaf;
        em.mark_lead(k, nb);
        em.leaves(ws, o, std::min(kLeaf, d - o), true);
        if (after_leaf) after_leaf(k);
        if (k == nb - 1) break;
        const int r0 = o + kLeaf, m = d - r0, slot = k % 3;
        const int nc = std::min(kLeaf, m);  // width of block column k+1
        sl.clear();
        g.clear();
        for (const InvWs& w : ws) {
            sl.push_back(slice_of(w.x, w.ld, o, o, kLeaf, kLeaf, w.px[slot], SLICE_FULL));
            if (ready_flags_enabled()) sl.back().ready = w.ready + k;  // starts on the leaf's X, not its end
        }
        em.slices(sl);
        if (k >= 1) em.wait(evA(k));  // A panel of k (col of k-1)
        // ---- TRSM: L[r0:, k] = A[r0:, k] X_kk^T
        for (const InvWs& w : ws) {
            GemmSpec t;
            t.a = sliced_view(w.pa[slot], m, kLeaf);
            t.b = sliced_view(w.px[slot], kLeaf, kLeaf);
            t.rows = m;
            t.cols = kLeaf;
            t.k = kLeaf;
            t.flags = EPI_VEC4;
            t.c = at(w.l, w.ld, r0, o);
            t.ldc = w.ld;
            g.push_back(t);
        }
        em.gemms(g);
        sl.clear();
        g.clear();
        // by d, so a factor's bits never depend on what else is in the call:
        // below 2048 the digit path stays (8x1024 alone: 528 vs 540 us; the
        // layer step is the same either way)
        const bool dfp = diag_fp32_enabled() && d >= diag_fp32_min_d();
        for (const InvWs& w : ws) sl.push_back(slice_of(w.l, w.ld, r0, o, m, kLeaf, w.pl[slot], SLICE_FULL));
        if (!dfp) em.slices(sl);
        if (k >= 1 && m > 0) em.wait(evU(k - 1));  // BU(k-1) wrote block column k+1
        const bool rest = m > kLeaf;
        const int side = 1 + (k & 1);
        if (rest) {
            em.record(evF);
            em.on(side);
            em.wait(evF);
            side_used[side - 1] = true;
            if (dfp) em.slices(sl);
            const int m2 = m - kLeaf;  // rows below block k+1
            // col: A[r0+128:, k+1] -= L[r0+128:, k] L[k+1, k]^T, then the A panel of k+1
            for (const InvWs& w : ws) {
                const Sliced lp = sliced_view(w.pl[slot], m, kLeaf);
                g.push_back(update(w, rows_of(lp, kLeaf, m2), rows_of(lp, 0, nc), m2, nc, r0 + kLeaf, r0, false));
            }
            em.gemms(g);
            g.clear();
            sl.clear();
            const int ns = (k + 1) % 3;
            for (const InvWs& w : ws) sl.push_back(slice_of(w.a, w.ld, r0 + kLeaf, r0, m2, kLeaf, w.pa[ns], SLICE_FULL));
            em.slices(sl);
            em.record(evA(k + 1));
            // BU: block column k+2 (rows >= k+2) -- BR(k-1) also wrote it
            if (k >= 1) em.wait(evB(k - 1));
            const int nc2 = std::min(kLeaf, m2);
            for (const InvWs& w : ws) {
                const Sliced lb = rows_of(sliced_view(w.pl[slot], m, kLeaf), kLeaf, m2);
                g.push_back(update(w, lb, rows_of(lb, 0, nc2), m2, nc2, r0 + kLeaf, r0 + kLeaf, false));
            }
            em.gemms(g);
            g.clear();
            em.record(evU(k));
            // BR: columns >= k+3, lower
            const int m3 = m2 - kLeaf;
            if (m3 > 0) {
                for (const InvWs& w : ws) {
                    const Sliced lr = rows_of(sliced_view(w.pl[slot], m, kLeaf), 2 * kLeaf, m3);
                    g.push_back(update(w, lr, lr, m3, m3, r0 + 2 * kLeaf, r0 + 2 * kLeaf, true));
                }
                em.gemms(g);
                g.clear();
            }
            em.record(evB(k));
            em.on(0);
        }
        // ---- diagonal block of k+1 (critical)
        if (dfp) {
            em.diag_updates(ws, r0, nc, o);
            continue;
        }
        for (const InvWs& w : ws) {
            const Sliced lp = sliced_view(w.pl[slot], m, kLeaf);
            g.push_back(update(w, rows_of(lp, 0, nc), rows_of(lp, 0, nc), nc, nc, r0, r0, false));
        }
        em.gemms(g);
        g.clear();
    }
    for (int s = 0; s < 2; ++s) {
        if (!side_used[s]) continue;
        em.on(s + 1);
        em.record(evEnd0 + s);
        em.on(0);
        em.wait(evEnd0 + s);
    }
}

// X = L^-1 from the strictly-lower L (w.l) and the leaves' diagonal blocks:
// per node X21 = -X22 (L21 X11); T^T = (L21 X11)^T needs only the left half,
// so it runs on the depth's side stream while the right half is inverted.
void trtri_rec(const std::vector<InvWs>& ws, int o, int n, Emitter& em, int depth = 0) {
    if (n <= kLeaf) return;  // diagonal block inverted by its leaf
    const int n1 = kTile * ((n + 2 * kTile - 1) / (2 * kTile));
    const int n2 = n - n1;
    trtri_rec(ws, o, n1, em, depth + 1);
    std::vector<SliceReq> sl;
    std::vector<GemmSpec> g;
    em.side_begin(depth);
    for (const InvWs& w : ws) {
        sl.push_back(slice_of(w.l, w.ld, o + n1, o, n2, n1, w.side0[depth], SLICE_FULL));
        sl.push_back(slice_of(w.xt, w.ld, o, o, n1, n1, w.side1[depth], SLICE_UPPER_BLOCK));
        GemmSpec s;
        s.a = sliced_view(w.side0[depth], n2, n1);
        s.b = sliced_view(w.side1[depth], n1, n1);
        s.rows = n2;
        s.cols = n1;
        s.k = n1;
        s.k_mode = K_FROM_COL_TILE;
        s.flags = EPI_TRANSPOSE;
        s.c = at(w.t, w.ld, w.t_row[depth], 0);  // T^T [n1 x n2]
        s.ldc = w.ld;
        g.push_back(s);
    }
    em.slices(sl);
    em.gemms(g);
    em.side_end(depth);
    trtri_rec(ws, o + n1, n2, em, depth + 1);
    em.side_join(depth);
    sl.clear();
    g.clear();
    for (const InvWs& w : ws) {
        sl.push_back(slice_of(w.x, w.ld, o + n1, o + n1, n2, n2, w.s0, SLICE_LOWER_BLOCK));
        sl.push_back(slice_of(w.t, w.ld, w.t_row[depth], 0, n1, n2, w.s1, SLICE_FULL));
        GemmSpec s;
        s.a = sliced_view(w.s0, n2, n2);
        s.b = sliced_view(w.s1, n1, n2);
        s.rows = n2;
        s.cols = n1;
        s.k = n2;
        s.k_mode = K_TO_ROW_TILE_END;
        s.alpha = -1.0f;
        s.flags = EPI_ALSO_T | EPI_VEC4;
        s.c = at(w.x, w.ld, o + n1, o);
        s.ldc = w.ld;
        s.c_t = at(w.xt, w.ld, o, o + n1);
        s.ldc_t = w.ld;
        g.push_back(s);
    }
    em.slices(sl);
    em.gemms(g);
}

// X = L^-1 bottom-up: the recursion tree of node splits (n1 = 128 ceil(n/256))
// grouped by height; every node of a height is independent, so each height is
// four batched launches (slices, T^T GEMMs, slices, X21 GEMMs) over all its
// nodes instead of a depth-first chain.  Same arithmetic per node as trtri_rec.
// Scratch: T^T of node (o, n) at rows [o, o + n1) of w.t (disjoint within a
// height); digit blocks packed in s0 / s1 (L21 | X22) and side0/side1 (XT11 | T).
struct TriNode {
    int o, n1, n2;
};

int tri_height(int n, std::vector<std::vector<TriNode>>& by_h, int o) {
    if (n <= kLeaf) return 0;
    const int n1 = kTile * ((n + 2 * kTile - 1) / (2 * kTile));
    const int h = 1 + std::max(tri_height(n1, by_h, o), tri_height(n - n1, by_h, o + n1));
    if (static_cast<int>(by_h.size()) < h) by_h.resize(h);
    by_h[h - 1].push_back(TriNode{o, n1, n - n1});
    return h;
}

void trtri_emit_levels(const std::vector<InvWs>& ws, Emitter& em, const std::vector<std::vector<TriNode>>& by_h,
                       int phases = 3);

// Bottom-up TRTRI of the diagonal range [o, o + n) (its node tree as built by
// tri_height: the whole matrix for (0, d), a subtree otherwise), every level
// one slice + GEMM pair per phase for all nodes and problems.
void trtri_levels(const std::vector<InvWs>& ws, Emitter& em, int o, int n) {
    std::vector<std::vector<TriNode>> by_h;
    tri_height(n, by_h, o);
    trtri_emit_levels(ws, em, by_h);
}

// phases: bit 0 = T^T = (L21 X11)^T into w.t, bit 1 = X21 = -X22 T (and X^T);
// a node's phase 1 needs only L21 and X11, so it can run before X22 exists.
void trtri_emit_levels(const std::vector<InvWs>& ws, Emitter& em, const std::vector<std::vector<TriNode>>& by_h,
                       int phases) {
    for (const auto& level : by_h) {
        std::vector<SliceReq> sl;
        std::vector<GemmSpec> g;
        if (phases & 1) {
        for (const InvWs& w : ws) {
            size_t off0 = 0, off1 = 0;
            for (const TriNode& nd : level) {
                char* a = static_cast<char*>(w.s0) + off0;
                char* b = static_cast<char*>(w.s1) + off1;
                off0 += align256(sliced_bytes(nd.n2, nd.n1));
                off1 += align256(sliced_bytes(nd.n1, nd.n1));
                sl.push_back(slice_of(w.l, w.ld, nd.o + nd.n1, nd.o, nd.n2, nd.n1, a, SLICE_FULL));
                sl.push_back(slice_of(w.xt, w.ld, nd.o, nd.o, nd.n1, nd.n1, b, SLICE_UPPER_BLOCK));
                GemmSpec s;
                s.a = sliced_view(a, nd.n2, nd.n1);
                s.b = sliced_view(b, nd.n1, nd.n1);
                s.rows = nd.n2;
                s.cols = nd.n1;
                s.k = nd.n1;
                s.k_mode = K_FROM_COL_TILE;
                s.flags = EPI_TRANSPOSE;
                s.c = at(w.t, w.ld, nd.o, 0);  // T^T [n1 x n2]
                s.ldc = w.ld;
                g.push_back(s);
            }
        }
        em.slices(sl);
        em.gemms(g);
        sl.clear();
        g.clear();
        }
        if (!(phases & 2)) continue;
        for (const InvWs& w : ws) {
            size_t off0 = 0, off1 = 0;
            for (const TriNode& nd : level) {
                char* a = static_cast<char*>(w.side0[0]) + off0;
                char* b = static_cast<char*>(w.side1[0]) + off1;
                off0 += align256(sliced_bytes(nd.n2, nd.n2));
                off1 += align256(sliced_bytes(nd.n1, nd.n2));
                sl.push_back(slice_of(w.x, w.ld, nd.o + nd.n1, nd.o + nd.n1, nd.n2, nd.n2, a, SLICE_LOWER_BLOCK));
                sl.push_back(slice_of(w.t, w.ld, nd.o, 0, nd.n1, nd.n2, b, SLICE_FULL));
                GemmSpec s;
                s.a = sliced_view(a, nd.n2, nd.n2);
                s.b = sliced_view(b, nd.n1, nd.n2);
                s.rows = nd.n2;
                s.cols = nd.n1;
                s.k = nd.n2;
                s.k_mode = K_TO_ROW_TILE_END;
                s.alpha = -1.0f;
                s.flags = EPI_ALSO_T | EPI_VEC4;
                s.c = at(w.x, w.ld, nd.o + nd.n1, nd.o);
                s.ldc = w.ld;
                s.c_t = at(w.xt, w.ld, nd.o, nd.o + nd.n1);
                s.ldc_t = w.ld;
                g.push_back(s);
            }
        }
        em.slices(sl);
        em.gemms(g);
    }
}

// Two schedules of the same factorisation: the right-looking one (above) has
// the shortest critical path but re-reads / re-writes the trailing matrix once
// per 128-column panel (K = 128 updates); the recursive one (inverse_rec)
// aggregates those updates into large-K GEMMs.  A call is latency-bound while
// its total work per panel of the longest chain, W = sum d^3 / d_max, is small
// (right-looking wins) and throughput-bound beyond (recursive wins).  Measured
// crossover (ms, right-looking / recursive): 3x4096 (W = 3 2^24) 3.17 / 3.37,
// 4x4096 (2^26) 3.78 / 3.75, 1x8192 (2^26) 6.43 / 6.60, 4x4096 + 20x1024
// (1.08 2^26) 4.21 / 3.97, 6x4096 6.03 / 5.07 ... 8x4096 6.80 / 5.67,
// 2x8192 10.8 / 9.2; one BERT-Large layer (0.54 2^26) 2.69 / 3.00.
// PF_INV_RECURSIVE=0/1 forces one.
constexpr double kRecursiveFromW = 67108864.0;  // 2^26

bool early_root_enabled() {  // PF_EARLY_ROOT=0: the root's T = L21 X11 after the factorisation (A/B)
    static const bool on = [] {
        const char* e = std::getenv("PF_EARLY_ROOT");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool early_trtri_enabled() {  // PF_EARLY_TRTRI=0: whole TRTRI after the factorisation (A/B)
    static const bool on = [] {
        const char* e = std::getenv("PF_EARLY_TRTRI");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool trtri_spine_enabled() {  // PF_TRTRI_SPINE=0: right subtree by levels after the factorisation (A/B)
    static const bool on = [] {
        const char* e = std::getenv("PF_TRTRI_SPINE");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool use_recursive_inverse(const std::vector<const pf_inverse_problem*>& probs) {
    static const int forced = [] {
        const char* e = std::getenv("PF_INV_RECURSIVE");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    if (forced >= 0) return forced == 1;
    double w = 0.0, dmax = 1.0;
    for (const pf_inverse_problem* p : probs) {
        const double d = p->d;
        w += d * d * d;
        dmax = std::max(dmax, d);
    }
    return w / dmax > kRecursiveFromW;
}

// PF_DIAG_SPLIT=0: the LAUUM slices X^T with its diagonal (measurement only:
// the d = 4096 residual goes back from ~2e-6 to ~1e-5)
bool diag_split_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PF_DIAG_SPLIT");
        return !(e && e[0] == '0');
    }();
    return on;
}

void damped_inverse_group(const std::vector<const pf_inverse_problem*>& probs, Emitter& em, bool recursive) {
    const int d = probs.front()->d;
    std::vector<InvWs> ws;
    std::vector<Damp2D> damps;
    for (const pf_inverse_problem* p : probs) {
        InvWs w = carve(p->workspace, d);
        w.info = p->d_info;
        damps.push_back(Damp2D{p->m, w.a, p->d_info, d, p->ldm, w.ld, p->damping});
        ws.push_back(w);
    }
    em.damp(damps);
    if (recursive) {
        inverse_rec(ws, 0, d, em);
    } else {
        // TRTRI along the factorisation.  The node tree's right spine (the
        // root, its right child, that node's right child, ...) is what the
        // last panels finish; everything else is done before:
        //   * the whole LEFT subtree of spine node (o, n1 | n2) needs only L
        //     and the leaves of panels < (o + n1)/128: level-batched on a
        //     low-priority side stream right after leaf (o + n1)/128 - 1;
        //   * the node's first phase, T = L21 X11, needs L[o+n1:, o:o+n1]
        //     (final once TRSM((o + n1)/128 - 1) ran, i.e. after leaf
        //     (o + n1)/128) and X11: right after it on the same stream;
        // so the tail after the last leaf is only the spine's X21 = -X22 T,
        // deepest node first (2x4096: 8 level pairs + the root -> 5 pairs).
        // PF_TRTRI_SPINE=0: only the root's left half and T early (the round-1
        // schedule).  Streaming EVERY finished node at its own panel was
        // measured slower (the many small nodes interfere with the chain).
        const int d = ws.front().d;
        struct Spine {
            TriNode node;
            std::vector<std::vector<TriNode>> left;  // levels of its left subtree
        };
        std::vector<Spine> spine;
        for (int o = 0, n = d; n > kLeaf;) {
            const int n1 = kTile * ((n + 2 * kTile - 1) / (2 * kTile));
            Spine sp{TriNode{o, n1, n - n1}, {}};
            tri_height(n1, sp.left, o);
            spine.push_back(std::move(sp));
            if (!trtri_spine_enabled()) break;  // round-1 schedule: the root only
            o += n1;
            n -= n1;
        }
        constexpr int evF = 29, evT = 30, kTrtriStream = 3;
        const bool early = !spine.empty() && early_trtri_enabled();
        cholesky_blocked(ws, em, [&](int k) {
            if (!early) return;
            bool opened = false;
            auto open = [&] {
                if (opened) return;
                opened = true;
                em.record(evF);
                em.on(kTrtriStream);
                em.wait(evF);
            };
            for (const Spine& sp : spine) {
                const int kl = (sp.node.o + sp.node.n1) / kLeaf - 1;
                if (k == kl && !sp.left.empty()) {
                    open();
                    trtri_emit_levels(ws, em, sp.left);
                }
                if (k == kl + 1 && early_root_enabled()) {
                    open();
                    trtri_emit_levels(ws, em, {{sp.node}}, 1);
                }
            }
            if (opened) {
                em.record(evT);
                em.on(0);
            }
        });
        if (early) {
            em.wait(evT);  // level digit slots are reused below
            if (!trtri_spine_enabled()) {  // round-1 schedule: right subtree by levels, then the root
                const Spine& r = spine.front();
                trtri_levels(ws, em, r.node.o + r.node.n1, r.node.n2);
            }
            for (auto it = spine.rbegin(); it != spine.rend(); ++it)
                trtri_emit_levels(ws, em, {{it->node}}, early_root_enabled() ? 2 : 3);
        } else {
            trtri_levels(ws, em, 0, d);
        }
    }
    // ---- LAUUM: M^-1 = X^T X = XT XT^T  (lower tiles, mirrored), with the
    // diagonal of XT split off: XT = D + O, O sliced with a zero diagonal, the
    // D terms added exactly in the epilogue (EPI_DIAG_SPLIT; the rows of XT
    // peak on the diagonal, where the digit form's row-max-relative error
    // would otherwise dominate the residual)
    std::vector<SliceReq> sl;
    std::vector<GemmSpec> g;
    for (std::size_t i = 0; i < ws.size(); ++i) {
        const InvWs& w = ws[i];
        const pf_inverse_problem* p = probs[i];
        const bool split = diag_split_enabled();
        sl.push_back(slice_of(w.xt, w.ld, 0, 0, d, d, w.s0, SLICE_UPPER_BLOCK | (split ? SLICE_ZERO_DIAG : 0)));
        GemmSpec s;
        s.a = sliced_view(w.s0, d, d);
        s.b = s.a;
        s.rows = s.cols = s.k = d;
        s.lower = true;
        s.k_mode = K_FROM_ROW_TILE;
        s.flags = EPI_MIRROR | (split ? EPI_DIAG_SPLIT : 0u);
        s.aux = w.x;  // X = L^-1, lower, ld = w.ld (multiple of 4, 256-B aligned plane)
        s.aux_t = w.xt;
        s.ld_aux = w.ld;
        if (aligned16(p->minv) && p->ldinv % 4 == 0) s.flags |= EPI_VEC4;
        s.c = p->minv;
        s.ldc = p->ldinv;
        g.push_back(s);
    }
    em.slices(sl);
    em.gemms(g);
    sl.clear();
    for (const pf_inverse_problem* p : probs)
        if (p->minv_sliced)
            sl.push_back(SliceReq{p->minv, p->ldinv, SLICE_FULL, sliced_view(p->minv_sliced, d, d)});
    if (!sl.empty()) em.slices(sl);
}

// ------------------------------------------------------------ precondition
// workspace: digit forms of A^-1, B^-1 (when given as fp32), G, U^T; fp32 U^T
struct PrecWs {
    void *ainv, *binv, *g, *ut_s;
    float* ut;
};

size_t precondition_ws_bytes(int d_out, int d_in) {
    return align256(sliced_bytes(d_in, d_in)) + align256(sliced_bytes(d_out, d_out)) +
           align256(sliced_bytes(d_out, d_in)) + align256(sliced_bytes(d_in, d_out)) +
           align256(static_cast<size_t>(d_in) * d_out * 4);
}

PrecWs carve_prec(void* base, int d_out, int d_in) {
    PrecWs w;
    char* p = static_cast<char*>(base);
    w.ainv = p;
    p += align256(sliced_bytes(d_in, d_in));
    w.binv = p;
    p += align256(sliced_bytes(d_out, d_out));
    w.g = p;
    p += align256(sliced_bytes(d_out, d_in));
    w.ut_s = p;
    p += align256(sliced_bytes(d_in, d_out));
    w.ut = reinterpret_cast<float*>(p);
    return w;
}

struct PrecJob {
    pf_precondition_problem p;
    const float* a_plain;  // non-null: slice A^-1 / B^-1 here first
    const float* b_plain;
};

void precondition_group(const std::vector<PrecJob>& jobs, cudaStream_t st) {
    std::vector<SliceReq> sl;
    std::vector<GemmSpec> g1, g2;
    std::vector<PrecWs> ws;
    for (const PrecJob& j : jobs) {
        const auto& p = j.p;
        PrecWs w = carve_prec(p.workspace, p.d_out, p.d_in);
        sl.push_back(SliceReq{p.grad, p.d_in, SLICE_FULL, sliced_view(w.g, p.d_out, p.d_in)});
        if (j.a_plain) {
            sl.push_back(SliceReq{j.a_plain, p.d_in, SLICE_FULL, sliced_view(w.ainv, p.d_in, p.d_in)});
            sl.push_back(SliceReq{j.b_plain, p.d_out, SLICE_FULL, sliced_view(w.binv, p.d_out, p.d_out)});
        }
        ws.push_back(w);
    }
    launch_slices(sl, st);
    sl.clear();
    for (std::size_t i = 0; i < jobs.size(); ++i) {
        const auto& p = jobs[i].p;
        const PrecWs& w = ws[i];
        const Sliced ainv = sliced_view(jobs[i].a_plain ? w.ainv : const_cast<void*>(p.a_inv_sliced),
                                        p.d_in, p.d_in);
        // U^T = A^-1 G^T  ([d_in x d_out], fp32)
        GemmSpec s;
        s.a = ainv;
        s.b = sliced_view(w.g, p.d_out, p.d_in);
        s.rows = p.d_in;
        s.cols = p.d_out;
        s.k = p.d_in;
        s.c = w.ut;
        s.ldc = p.d_out;
        if (aligned16(w.ut) && p.d_out % 4 == 0) s.flags |= EPI_VEC4;
        g1.push_back(s);
        sl.push_back(SliceReq{w.ut, p.d_out, SLICE_FULL, sliced_view(w.ut_s, p.d_in, p.d_out)});
    }
    gemm_oz8(g1, st);
    launch_slices(sl, st);
    for (std::size_t i = 0; i < jobs.size(); ++i) {
        const auto& p = jobs[i].p;
        const PrecWs& w = ws[i];
        const Sliced binv = sliced_view(jobs[i].b_plain ? w.binv : const_cast<void*>(p.b_inv_sliced),
                                        p.d_out, p.d_out);
        // P = B^-1 U ; epilogue W -= eta P (or P itself)
        GemmSpec t;
        t.a = binv;
        t.b = sliced_view(w.ut_s, p.d_in, p.d_out);
        t.rows = p.d_out;
        t.cols = p.d_in;
        t.k = p.d_out;
        float* dst = p.w ? p.w : p.p_out;
        t.alpha = p.w ? -p.eta : 1.0f;
        t.beta = p.w ? 1.0f : 0.0f;
        t.c = dst;
        t.ldc = p.d_in;
        if (aligned16(dst) && p.d_in % 4 == 0) t.flags |= EPI_VEC4;
        g2.push_back(t);
    }
    gemm_oz8(g2, st);
}

// ------------------------------------------------------------ fork / join
// Per-thread, per-device pool of non-blocking side streams and events.  A
// call forks onto them with an event recorded on the caller's stream and
// joins back with one event per side stream: stream-ordered semantics are
// kept and the pattern is legal inside CUDA-graph capture.
struct SidePool {
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> events;  // [0] fork, [1..] joins
};

SidePool& side_pool(std::size_t n) {
    thread_local std::vector<SidePool> pools;
    int dev = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    if (pools.size() <= static_cast<std::size_t>(dev)) pools.resize(dev + 1);
    SidePool& p = pools[dev];
    while (p.streams.size() < n) {
        cudaStream_t s;
        check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
        p.streams.push_back(s);
    }
    while (p.events.size() < n + 1) {
        cudaEvent_t e;
        check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        p.events.push_back(e);
    }
    return p;
}

template <class F>
void run_forked(std::size_t n, cudaStream_t st, F&& body) {
    if (n == 0) return;
    if (n == 1) {
        body(0, st);
        return;
    }
    SidePool& p = side_pool(n - 1);
    check(cudaEventRecord(p.events[0], st), "cudaEventRecord(fork)");
    for (std::size_t g = 1; g < n; ++g) check(cudaStreamWaitEvent(p.streams[g - 1], p.events[0], 0), "fork");
    body(0, st);
    for (std::size_t g = 1; g < n; ++g) {
        body(g, p.streams[g - 1]);
        check(cudaEventRecord(p.events[g], p.streams[g - 1]), "cudaEventRecord(join)");
        check(cudaStreamWaitEvent(st, p.events[g], 0), "join");
    }
}

}  // namespace
}  // namespace pf

// ============================================================== C-ABI
using namespace pf;

extern "C" {

int64_t pf_kernel_launch_count(void) { return g_launches.load(); }

#ifdef PF_GEMM_PROBE
int pf_gemm_probe_read(long long* out) {  // 64 records of 8; returns the record count
    int n = 0;
    if (cudaMemcpyFromSymbol(out, pf::g_gemm_probe, sizeof(long long) * 64 * 16) != cudaSuccess) return -1;
    if (cudaMemcpyFromSymbol(&n, pf::g_gemm_probe_n, sizeof(int)) != cudaSuccess) return -1;
    const int zero = 0;
    cudaMemcpyToSymbol(pf::g_gemm_probe_n, &zero, sizeof(int));
    return n;
}
#endif

#ifdef PF_LEAF_RING
int pf_leaf_ring_read(long long* out) {  // 64 records of 8; returns the record count, resets it
    int n = 0;
    if (cudaMemcpyFromSymbol(out, pf::g_leaf_ring, sizeof(long long) * 64 * 8) != cudaSuccess) return -1;
    if (cudaMemcpyFromSymbol(&n, pf::g_leaf_ring_n, sizeof(int)) != cudaSuccess) return -1;
    const int zero = 0;
    cudaMemcpyToSymbol(pf::g_leaf_ring_n, &zero, sizeof(int));
    return n;
}
#endif

int pf_set_background(int on) {
    const int was = pf::g_background ? 1 : 0;
    pf::g_background = on != 0;
    return was;
}

int pf_device_ok(void) {
    int dev = 0;
    cudaDeviceProp prop{};
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return 0;
    return prop.major == 10 ? 1 : 0;
}

int pf_curvature_syrk_grouped(const pf_syrk_problem* problems, int count, int fill_upper,
                              void* stream) {
    return pf_detail::guard([&] {
        if (count < 0 || (count > 0 && !problems)) throw std::invalid_argument("bad problem list");
        if (count == 0) return 0;
        std::vector<GemmSpec> specs;
        for (int i = 0; i < count; ++i) {
            const pf_syrk_problem& p = problems[i];
            if (p.layout != 0 && p.layout != 1) throw std::invalid_argument("curvature_syrk: bad layout");
            const bool tm = p.layout == 1;  // token-major x [n x d]
            if (p.d < 1 || p.n < 1 || p.ldx < (tm ? p.d : p.n) || p.ldf < p.d || !p.x || !p.f)
                throw ShapeError("curvature_syrk: shape mismatch");
            if (p.ldx % 8 != 0 || !aligned16(p.x))
                throw ShapeError("curvature_syrk: x needs 16-byte rows (ldx % 8 == 0)");
            GemmSpec s;
            s.mn_major = tm;
            s.a_bf16 = s.b_bf16 = p.x;
            s.lda = s.ldb = p.ldx;
            s.rows = s.cols = p.d;
            s.k = p.n;
            s.lower = true;
            s.alpha = p.scale;
            s.beta = p.accumulate ? 1.0f : 0.0f;
            s.flags = fill_upper ? EPI_MIRROR : 0u;
            if (aligned16(p.f) && p.ldf % 4 == 0) s.flags |= EPI_VEC4;
            s.c = p.f;
            s.ldc = p.ldf;
            specs.push_back(s);
        }
        gemm_bf16(specs, static_cast<cudaStream_t>(stream));
        return 0;
    });
}

int pf_curvature_syrk(const void* x_bf16, int d, int n, int ldx, float scale, int accumulate,
                      float* f, int ldf, int fill_upper, void* stream) {
    pf_syrk_problem p{x_bf16, f, d, n, ldx, ldf, scale, accumulate, 0};
    return pf_curvature_syrk_grouped(&p, 1, fill_upper, stream);
}

int pf_slice_bytes(int rows, int k, size_t* bytes) {
    return pf_detail::guard([&] {
        if (rows < 1 || k < 1 || !bytes) throw std::invalid_argument("bad dims");
        *bytes = sliced_bytes(rows, k);
        return 0;
    });
}

int pf_slice(const float* x, int rows, int k, int ld, void* sliced, void* stream) {
    return pf_detail::guard([&] {
        if (rows < 1 || k < 1 || ld < k || !x || !sliced) throw ShapeError("slice: shape mismatch");
        if (!aligned16(sliced)) throw std::invalid_argument("slice: output must be 16-B aligned");
        launch_slices({SliceReq{x, ld, SLICE_FULL, sliced_view(sliced, rows, k)}},
                      static_cast<cudaStream_t>(stream));
        return 0;
    });
}

int pf_damped_inverse_workspace(int d, size_t* bytes) {
    return pf_detail::guard([&] {
        if (d < 1 || !bytes) throw std::invalid_argument("bad d");
        *bytes = inverse_ws_bytes(d);
        return 0;
    });
}

int pf_damped_inverse_batched(const pf_inverse_problem* problems, int count, void* stream) {
    return pf_detail::guard([&] {
        if (count < 0 || (count > 0 && !problems)) throw std::invalid_argument("bad problem list");
        std::vector<const pf_inverse_problem*> order;
        for (int i = 0; i < count; ++i) {
            const pf_inverse_problem& p = problems[i];
            if (p.d < 1 || p.ldm < p.d || p.ldinv < p.d || !p.m || !p.minv || !p.d_info ||
                !p.workspace)
                throw ShapeError("cholesky_spd_inverse: matrix not square / bad arguments");
            if (!aligned16(p.workspace)) throw std::invalid_argument("workspace must be 16-B aligned");
            if (p.minv_sliced && !aligned16(p.minv_sliced))
                throw std::invalid_argument("sliced output must be 16-B aligned");
            order.push_back(&p);
        }
        if (order.empty()) return 0;  // nothing to invert: no launch, no side streams
        // Largest first; equal-d problems share every launch (groups of <= 8,
        // split evenly).  Independent groups run concurrently: the first on
        // `stream`, the others on side streams forked/joined with events, so
        // the short d=1024 chains hide under a d=4096 chain.
        std::stable_sort(order.begin(), order.end(), [](auto* a, auto* b) { return a->d > b->d; });
        // equal-d problems share launches in groups of <= 8 (right-looking: few,
        // latency-bound chains) or <= 4 (recursive: more concurrent chains for
        // a throughput-bound batch; 8x4096 5.37 -> 5.24 ms)
        const bool recursive = use_recursive_inverse(order);
        std::vector<std::vector<const pf_inverse_problem*>> groups;
        for (std::size_t i = 0; i < order.size();) {
            std::size_t j = i;
            while (j < order.size() && order[j]->d == order[i]->d) ++j;
            static const int forced = [] {
                const char* e = std::getenv("PF_INV_GROUP");
                return e ? std::max(1, std::atoi(e)) : 0;
            }();
            // lead-size problems of a right-looking call in groups of
            // PF_INV_GROUP_LEAD (default 1 with the fp32 diagonal update:
            // separate chains on forked streams, 2x4096 + 10x1024 2.394 ->
            // 2.357 ms; with the digit diagonal update shared launches were
            // faster); 0 = groups of <= 8 like the others
            static const int lead_per = [] {
                const char* e = std::getenv("PF_INV_GROUP_LEAD");
                return e ? std::max(0, std::atoi(e)) : diag_fp32_enabled() ? 1 : 0;
            }();
            std::size_t per = forced ? static_cast<std::size_t>(forced) : recursive ? 4 : 8;
            if (lead_per && !recursive && order[i]->d == order.front()->d && order[i]->d >= diag_fp32_min_d())
                per = static_cast<std::size_t>(lead_per);
            // the shorter groups of a right-looking call (they run under the
            // lead chains) in groups of <= PF_INV_GROUP_SIDE (default 4; 0 =
            // <= 8): 2x4096 + 10x1024 2.336 -> 2.326 ms
            static const int side_per = [] {
                const char* e = std::getenv("PF_INV_GROUP_SIDE");
                return e ? std::max(0, std::atoi(e)) : 4;
            }();
            if (side_per && !forced && !recursive && order[i]->d != order.front()->d)
                per = static_cast<std::size_t>(side_per);
            const std::size_t m = j - i, parts = (m + per - 1) / per;
            for (std::size_t q = 0; q < parts; ++q)
                groups.emplace_back(order.begin() + i + m * q / parts, order.begin() + i + m * (q + 1) / parts);
            i = j;
        }
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        {
            g_lead_panels = 0;
            const int lead_d = groups[0].front()->d;
            run_forked(groups.size(), st, [&](std::size_t g, cudaStream_t s) {
                const int d_g = groups[g].front()->d;
                if (g > 0 && d_g < lead_d && g_lead_panels > 0) {
                    static const double mul = [] {
                        const char* e = std::getenv("PF_DELAY_MUL");
                        return e ? std::atof(e) : 1.5;  // round 2 re-tune (2.0: 2.437 ms, 1.5: 2.415)
                    }();
                    const int start = g_lead_panels - static_cast<int>(mul * ((d_g + kLeaf - 1) / kLeaf));
                    if (start > 0)
                        check(cudaStreamWaitEvent(s, pool_event(kMarkGroup, start), 0), "lead mark wait");
                }
                StreamEmitter em(s, static_cast<int>(g), groups[g].front()->d == groups[0].front()->d);
                damped_inverse_group(groups[g], em, recursive);
            });
        }
        return 0;
    });
}

int pf_damped_inverse(const float* m, int d, int ldm, float damping, float* minv, int ldinv,
                      void* minv_sliced, void* workspace, size_t workspace_bytes, int* d_info,
                      void* stream) {
    return pf_detail::guard([&] {
        if (d >= 1 && workspace_bytes < inverse_ws_bytes(d))
            throw std::invalid_argument("workspace too small");
        pf_inverse_problem p{m, minv, minv_sliced, d, ldm, ldinv, damping, workspace, d_info};
        const int rc = pf_damped_inverse_batched(&p, 1, stream);
        if (rc != 0) throw std::invalid_argument(pf_detail::last_error());
        return 0;
    });
}

int pf_cholesky_factor(const float* m, int d, int ldm, float damping, float* l, int ldl, void* workspace,
                       size_t workspace_bytes, int* d_info, void* stream) {
    return pf_detail::guard([&] {
        if (d < 1 || ldm < d || ldl < d || !m || !l || !d_info || !workspace)
            throw ShapeError("cholesky_factor: matrix not square / bad arguments");
        if (workspace_bytes < inverse_ws_bytes(d)) throw std::invalid_argument("workspace too small");
        if (!aligned16(workspace)) throw std::invalid_argument("workspace must be 16-B aligned");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        InvWs w = carve(workspace, d);
        w.info = d_info;
        w.lout = l;
        w.ldl = ldl;
        g_lead_panels = 0;
        StreamEmitter em(st, 0, true);
        em.damp({Damp2D{m, w.a, d_info, d, ldm, w.ld, damping}});
        cholesky_blocked({w}, em);
        launch(assemble_l_kernel, dim3(d), dim3(256), 0, st, w.l, w.ld, l, ldl, d);
        after_launch("assemble_l_kernel");
        return 0;
    });
}

int pf_precondition_workspace(int d_out, int d_in, size_t* bytes) {
    return pf_detail::guard([&] {
        if (d_out < 1 || d_in < 1 || !bytes) throw std::invalid_argument("bad dims");
        *bytes = precondition_ws_bytes(d_out, d_in);
        return 0;
    });
}

static int precondition_plain(const float* b_inv, const float* grad, const float* a_inv, float* w,
                              float* p_out, int d_out, int d_in, float eta, void* workspace,
                              size_t workspace_bytes, void* stream) {
    return pf_detail::guard([&] {
        if (d_out < 1 || d_in < 1 || !b_inv || !grad || !a_inv || (!w && !p_out) || !workspace)
            throw ShapeError("precondition: shape mismatch");
        if (workspace_bytes < precondition_ws_bytes(d_out, d_in))
            throw std::invalid_argument("workspace too small");
        if (!aligned16(workspace)) throw std::invalid_argument("workspace must be 16-B aligned");
        PrecJob j{};
        j.p.grad = grad;
        j.p.w = w;
        j.p.p_out = p_out;
        j.p.d_out = d_out;
        j.p.d_in = d_in;
        j.p.eta = eta;
        j.p.workspace = workspace;
        j.a_plain = a_inv;
        j.b_plain = b_inv;
        precondition_group({j}, static_cast<cudaStream_t>(stream));
        return 0;
    });
}

int pf_precondition(const float* b_inv, const float* grad, const float* a_inv, float* p_out,
                    int d_out, int d_in, void* workspace, size_t workspace_bytes, void* stream) {
    return precondition_plain(b_inv, grad, a_inv, nullptr, p_out, d_out, d_in, 0.0f, workspace,
                              workspace_bytes, stream);
}

int pf_precondition_update(const float* b_inv, const float* grad, const float* a_inv, float* w,
                           int d_out, int d_in, float eta, void* workspace,
                           size_t workspace_bytes, void* stream) {
    return precondition_plain(b_inv, grad, a_inv, w, nullptr, d_out, d_in, eta, workspace,
                              workspace_bytes, stream);
}

int pf_precondition_update_sliced(const pf_precondition_problem* problems, int count,
                                  void* stream) {
    return pf_detail::guard([&] {
        if (count < 0 || (count > 0 && !problems)) throw std::invalid_argument("bad problem list");
        std::vector<PrecJob> v;
        for (int i = 0; i < count; ++i) {
            const auto& p = problems[i];
            if (p.d_out < 1 || p.d_in < 1 || !p.grad || (!p.w && !p.p_out) || !p.workspace ||
                !p.a_inv_sliced || !p.b_inv_sliced)
                throw ShapeError("precondition: shape mismatch");
            v.push_back(PrecJob{p, nullptr, nullptr});
        }
        for (std::size_t i = 0; i < v.size(); i += kMaxProbs) {
            std::vector<PrecJob> chunk(v.begin() + i, v.begin() + std::min(v.size(), i + kMaxProbs));
            precondition_group(chunk, static_cast<cudaStream_t>(stream));
        }
        return 0;
    });
}

int pf_f32_to_bf16(const float* x, int64_t n, void* out, void* stream) {
    return pf_detail::guard([&] {
        if (n < 0 || !x || !out) throw std::invalid_argument("bad convert");
        const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
        if (blocks > 0) {
            launch(f32_to_bf16_kernel, dim3(blocks), dim3(256), 0, static_cast<cudaStream_t>(stream), x, n,
                   static_cast<__nv_bfloat16*>(out));
            after_launch("f32_to_bf16_kernel");
        }
        return 0;
    });
}

}  // extern "C"
