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

template <typename... KArgs, typename... Args>
void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
            Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
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

struct SliceReq {
    const float* src;
    int ld;
    int mode;
    Sliced dst;
};

void launch_slices(const std::vector<SliceReq>& reqs, cudaStream_t st) {
    for (std::size_t i = 0; i < reqs.size(); i += kMaxSliceJobs) {
        SliceBatch b{};
        const int cnt = static_cast<int>(std::min<std::size_t>(kMaxSliceJobs, reqs.size() - i));
        int rows = 1;
        for (int j = 0; j < cnt; ++j) {
            const SliceReq& r = reqs[i + j];
            b.j[j] = SliceJob{r.src, r.dst.rows, r.dst.k, r.ld, r.mode, r.dst.planes,
                              r.dst.plane_stride, r.dst.kpad, r.dst.exps, r.dst.sqnorm};
            rows = std::max(rows, r.dst.rows);
        }
        launch(slice_kernel, dim3((rows + 7) / 8, cnt), dim3(256), 0, st, b);
        after_launch("slice_kernel");
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
};

template <int kFmt>
void launch_gemms(const std::vector<GemmSpec>& specs, cudaStream_t stream) {
    using T = GemmTraits<kFmt>;
    auto kernel = umma_gemm_kernel<kFmt>;
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
            const GemmSpec& s = specs[i];
            const bool shared_ab = kFmt == kBF16 ? (s.a_bf16 == s.b_bf16 && s.lda == s.ldb)
                                                 : (s.a.planes == s.b.planes);
            const int need = T::kPlanes * (shared_ab ? 1 : 2);
            if (maps + need > kMaxMaps) break;
            GemmDesc& d = batch.probs[probs];
            auto put_maps = [&](bool is_a) {
                const int first = maps;
                if constexpr (kFmt == kBF16) {
                    encode(&batch.maps[maps++], is_a ? s.a_bf16 : s.b_bf16, true,
                           is_a ? s.rows : s.cols, s.k, static_cast<size_t>(is_a ? s.lda : s.ldb) * 2);
                } else {
                    const Sliced& o = is_a ? s.a : s.b;
                    for (int pl = 0; pl < kDigits; ++pl)
                        encode(&batch.maps[maps++], o.planes + pl * o.plane_stride, false, o.rows,
                               o.k, static_cast<size_t>(o.kpad));
                }
                return first;
            };
            d.a_map = put_maps(true);
            d.b_map = shared_ab ? d.a_map : put_maps(false);
            if (kFmt == kOZ8 && shared_ab) d.flags |= EPI_EXACT_DIAG;
            d.rows = s.rows;
            d.cols = s.cols;
            d.k = s.k;
            d.tiles_m = (s.rows + kTile - 1) / kTile;
            d.tiles_n = (s.cols + kTile - 1) / kTile;
            d.lower = s.lower ? 1 : 0;
            d.tile_begin = tiles;
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
            tiles += s.lower ? d.tiles_m * (d.tiles_m + 1) / 2 : d.tiles_m * d.tiles_n;
            ++probs;
            ++i;
        }
        batch.n_probs = probs;
        batch.total_tiles = tiles;
        if (tiles == 0) continue;
        launch(kernel, dim3(tiles), dim3(128), T::kSmemBytes, stream, batch);
        after_launch("umma_gemm_kernel");
    }
}

void gemm_bf16(const std::vector<GemmSpec>& s, cudaStream_t st) { launch_gemms<kBF16>(s, st); }
void gemm_oz8(const std::vector<GemmSpec>& s, cudaStream_t st) { launch_gemms<kOZ8>(s, st); }

// ------------------------------------------------------------ small kernels
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

// dst = M + damping * I  (lower triangle incl. diagonal; the rest never read)
__global__ void damp_kernel(const __grid_constant__ DampBatch b) {
    const Damp2D& s = b.e[blockIdx.y];
    ptx::grid_dep_wait();
    ptx::grid_dep_launch();
    if (blockIdx.x == 0 && threadIdx.x == 0) *s.info = 0;
    const int64_t total = static_cast<int64_t>(s.d) * s.d;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(idx / s.d), c = static_cast<int>(idx % s.d);
        if (c > r) continue;
        float v = s.src[static_cast<int64_t>(r) * s.ld_src + c];
        if (r == c) v += s.damping;
        s.dst[static_cast<int64_t>(r) * s.ld_dst + c] = v;
    }
}

__global__ void f32_to_bf16_kernel(const float* x, int64_t n, __nv_bfloat16* out) {
    ptx::grid_dep_wait();
    ptx::grid_dep_launch();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __float2bfloat16_rn(x[i]);
}

// ------------------------------------------------------------ damped inverse
// Workspace of one factor (ld = round_up(d, 4)):
//   fp32  A (damped factor, updated in place), L (panel blocks L21),
//         X = L^-1 (lower), XT = L^-T (upper), T (temporary)
//   digit form  two operand slots S0, S1 sized for d x d
struct InvWs {
    int d = 0, ld = 0;
    float *a, *l, *x, *xt, *t;
    void* s0;
    void* s1;
    int* info = nullptr;
};

size_t inverse_ws_bytes(int d) {
    const size_t plane = align256(static_cast<size_t>(round_up(d, 4)) * d * sizeof(float));
    return 5 * plane + 2 * align256(sliced_bytes(d, d));
}

InvWs carve(void* base, int d) {
    InvWs w;
    w.d = d;
    w.ld = round_up(d, 4);
    const size_t plane = align256(static_cast<size_t>(w.ld) * d * sizeof(float));
    char* p = static_cast<char*>(base);
    float** f[5] = {&w.a, &w.l, &w.x, &w.xt, &w.t};
    for (int i = 0; i < 5; ++i) *f[i] = reinterpret_cast<float*>(p + i * plane);
    w.s0 = p + 5 * plane;
    w.s1 = p + 5 * plane + align256(sliced_bytes(d, d));
    return w;
}

float* at(float* base, int ld, int r, int c) { return base + static_cast<size_t>(r) * ld + c; }

void launch_leaves(const std::vector<InvWs>& ws, int o, int n, cudaStream_t st) {
    static std::once_flag once;
    std::call_once(once, [] {
        check(cudaFuncSetAttribute(leaf_chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kLeafSmemBytes),
              "cudaFuncSetAttribute(leaf)");
    });
    for (std::size_t i = 0; i < ws.size(); i += kMaxLeafBatch) {
        LeafBatch b{};
        const int cnt = static_cast<int>(std::min<std::size_t>(kMaxLeafBatch, ws.size() - i));
        for (int j = 0; j < cnt; ++j) {
            const InvWs& w = ws[i + j];
            b.e[j] = LeafArgs{at(w.a, w.ld, o, o), at(w.x, w.ld, o, o), at(w.xt, w.ld, o, o),
                              w.info, w.ld, n, o};
        }
        launch(leaf_chol_inv_kernel, dim3(cnt), dim3(kLeafThreads), kLeafSmemBytes, st, b);
        after_launch("leaf_chol_inv_kernel");
    }
}

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
void inverse_rec(const std::vector<InvWs>& ws, int o, int n, cudaStream_t st) {
    if (n <= kLeaf) {
        launch_leaves(ws, o, n, st);
        return;
    }
    const int n1 = kTile * ((n + 2 * kTile - 1) / (2 * kTile));
    const int n2 = n - n1;
    inverse_rec(ws, o, n1, st);

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
    launch_slices(sl, st);
    gemm_oz8(g, st);
    // ---- A22 -= L21 L21^T
    sl.clear();
    g.clear();
    for (const InvWs& w : ws) {
        sl.push_back(slice_of(w.l, w.ld, o + n1, o, n2, n1, w.s0, SLICE_FULL));
        GemmSpec s;
        s.a = sliced_view(w.s0, n2, n1);
        s.b = s.a;
        s.rows = s.cols = n2;
        s.k = n1;
        s.lower = true;
        s.alpha = -1.0f;
        s.beta = 1.0f;
        s.flags = EPI_VEC4;
        s.c = at(w.a, w.ld, o + n1, o + n1);
        s.ldc = w.ld;
        g.push_back(s);
    }
    launch_slices(sl, st);
    gemm_oz8(g, st);

    inverse_rec(ws, o + n1, n2, st);

    // ---- T^T = (L21 X11)^T : B operand rows = XT11 (upper block-triangular)
    sl.clear();
    g.clear();
    for (const InvWs& w : ws) {
        sl.push_back(slice_of(w.l, w.ld, o + n1, o, n2, n1, w.s0, SLICE_FULL));
        sl.push_back(slice_of(w.xt, w.ld, o, o, n1, n1, w.s1, SLICE_UPPER_BLOCK));
        GemmSpec s;
        s.a = sliced_view(w.s0, n2, n1);
        s.b = sliced_view(w.s1, n1, n1);
        s.rows = n2;
        s.cols = n1;
        s.k = n1;
        s.k_mode = K_FROM_COL_TILE;
        s.flags = EPI_TRANSPOSE;
        s.c = w.t;  // T^T [n1 x n2], ld = w.ld
        s.ldc = w.ld;
        g.push_back(s);
    }
    launch_slices(sl, st);
    gemm_oz8(g, st);
    // ---- X21 = -X22 T  (B operand rows = T^T), also stored as XT12
    sl.clear();
    g.clear();
    for (const InvWs& w : ws) {
        sl.push_back(slice_of(w.x, w.ld, o + n1, o + n1, n2, n2, w.s0, SLICE_LOWER_BLOCK));
        sl.push_back(slice_of(w.t, w.ld, 0, 0, n1, n2, w.s1, SLICE_FULL));
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
    launch_slices(sl, st);
    gemm_oz8(g, st);
}

void damped_inverse_group(const std::vector<const pf_inverse_problem*>& probs, cudaStream_t st) {
    const int d = probs.front()->d;
    std::vector<InvWs> ws;
    DampBatch db{};
    for (std::size_t i = 0; i < probs.size(); ++i) {
        const pf_inverse_problem* p = probs[i];
        InvWs w = carve(p->workspace, d);
        w.info = p->d_info;
        db.e[i] = Damp2D{p->m, w.a, p->d_info, d, p->ldm, w.ld, p->damping};
        ws.push_back(w);
    }
    const int blocks = std::min((d * d + 255) / 256, 148 * 8);
    launch(damp_kernel, dim3(blocks, static_cast<unsigned>(probs.size())), dim3(256), 0, st, db);
    after_launch("damp_kernel");
    inverse_rec(ws, 0, d, st);
    // ---- LAUUM: M^-1 = X^T X = XT XT^T  (lower tiles, mirrored)
    std::vector<SliceReq> sl;
    std::vector<GemmSpec> g;
    for (std::size_t i = 0; i < ws.size(); ++i) {
        const InvWs& w = ws[i];
        const pf_inverse_problem* p = probs[i];
        sl.push_back(slice_of(w.xt, w.ld, 0, 0, d, d, w.s0, SLICE_UPPER_BLOCK));
        GemmSpec s;
        s.a = sliced_view(w.s0, d, d);
        s.b = s.a;
        s.rows = s.cols = s.k = d;
        s.lower = true;
        s.k_mode = K_FROM_ROW_TILE;
        s.flags = EPI_MIRROR;
        if (aligned16(p->minv) && p->ldinv % 4 == 0) s.flags |= EPI_VEC4;
        s.c = p->minv;
        s.ldc = p->ldinv;
        g.push_back(s);
    }
    launch_slices(sl, st);
    gemm_oz8(g, st);
    sl.clear();
    for (const pf_inverse_problem* p : probs)
        if (p->minv_sliced)
            sl.push_back(SliceReq{p->minv, p->ldinv, SLICE_FULL, sliced_view(p->minv_sliced, d, d)});
    launch_slices(sl, st);
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
int pf_gemm_probe_read(long long* out) {
    return cudaMemcpyFromSymbol(out, pf::g_gemm_probe, sizeof(long long) * 16) == cudaSuccess ? 0 : 3;
}
#endif

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
        std::vector<GemmSpec> specs;
        for (int i = 0; i < count; ++i) {
            const pf_syrk_problem& p = problems[i];
            if (p.d < 1 || p.n < 1 || p.ldx < p.n || p.ldf < p.d || !p.x || !p.f)
                throw ShapeError("curvature_syrk: shape mismatch");
            if (p.ldx % 8 != 0 || !aligned16(p.x))
                throw ShapeError("curvature_syrk: x needs 16-byte rows (ldx % 8 == 0)");
            GemmSpec s;
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
    pf_syrk_problem p{x_bf16, f, d, n, ldx, ldf, scale, accumulate};
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
        // Largest first; equal-d problems share every launch (groups of <= 8,
        // split evenly).  Independent groups run concurrently: the first on
        // `stream`, the others on side streams forked/joined with events, so
        // the short d=1024 chains hide under a d=4096 chain.
        std::stable_sort(order.begin(), order.end(), [](auto* a, auto* b) { return a->d > b->d; });
        std::vector<std::vector<const pf_inverse_problem*>> groups;
        for (std::size_t i = 0; i < order.size();) {
            std::size_t j = i;
            while (j < order.size() && order[j]->d == order[i]->d) ++j;
            const std::size_t m = j - i, parts = (m + 7) / 8;
            for (std::size_t q = 0; q < parts; ++q)
                groups.emplace_back(order.begin() + i + m * q / parts, order.begin() + i + m * (q + 1) / parts);
            i = j;
        }
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        run_forked(groups.size(), st, [&](std::size_t g, cudaStream_t s) { damped_inverse_group(groups[g], s); });
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
