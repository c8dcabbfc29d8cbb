// Host launchers and the C-ABI (include/pf_kfac.h) of the K-FAC hot path:
//   curvature SYRK (bf16 tcgen05), damped inverse (SIMT panels + 3xTF32
//   tcgen05 recursion), precondition + fused update (3xTF32 tcgen05).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
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
#include "umma_gemm.cuh"

namespace pf {
namespace {

std::atomic<int64_t> g_launches{0};

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void after_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    check(cudaGetLastError(), what);
}

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

// A K-major operand: `rows` rows of `k` elements, row pitch `ld` elements.
// Planes: hi (or the only plane) and, for 3xTF32, lo.
struct Operand {
    const void* hi = nullptr;
    const void* lo = nullptr;
    int rows = 0, k = 0, ld = 0;
    bool bf16 = false;
};

void encode(CUtensorMap* m, const void* ptr, const Operand& op) {
    const size_t es = op.bf16 ? 2 : 4;
    if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0 || (op.ld * es) % 16 != 0)
        throw std::invalid_argument("TMA operand needs 16-byte aligned base and row pitch");
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(op.k), static_cast<cuuint64_t>(op.rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(op.ld) * es};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / es), 128};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = encoder()(
        m, op.bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
        const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

struct GemmSpec {
    Operand a, b;
    int rows = 0, cols = 0, k = 0;
    bool lower = false;
    int k_mode = K_FULL;
    float alpha = 1.0f, beta = 0.0f;
    uint32_t flags = 0;
    float* c = nullptr;
    float* c_lo = nullptr;
    float* c_t = nullptr;
    float* c_t_lo = nullptr;
    int ldc = 0, ldc_t = 0;
};

template <int kFmt, int kPlanes, int kStages>
void launch_gemms(const std::vector<GemmSpec>& specs, cudaStream_t stream) {
    using T = GemmTraits<kFmt, kPlanes, kStages>;
    auto kernel = umma_gemm_kernel<kFmt, kPlanes, kStages>;
    static std::once_flag attr_once;
    std::call_once(attr_once, [&] {
        check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   T::kSmemBytes),
              "cudaFuncSetAttribute(gemm)");
    });
    std::size_t i = 0;
    while (i < specs.size()) {
        GemmBatch batch;
        std::memset(&batch, 0, sizeof(batch));
        int maps = 0, probs = 0, tiles = 0;
        while (i < specs.size() && probs < kMaxProbs) {
            const GemmSpec& s = specs[i];
            const bool shared_ab = s.a.hi == s.b.hi && s.a.rows == s.b.rows && s.a.k == s.b.k &&
                                   s.a.ld == s.b.ld && s.a.lo == s.b.lo;
            const int need = kPlanes * (shared_ab ? 1 : 2);
            if (maps + need > kMaxMaps) break;
            GemmDesc& d = batch.probs[probs];
            d.a_map = maps;
            encode(&batch.maps[maps++], s.a.hi, s.a);
            if (kPlanes == 2) encode(&batch.maps[maps++], s.a.lo, s.a);
            if (shared_ab) {
                d.b_map = d.a_map;
            } else {
                d.b_map = maps;
                encode(&batch.maps[maps++], s.b.hi, s.b);
                if (kPlanes == 2) encode(&batch.maps[maps++], s.b.lo, s.b);
            }
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
            d.flags = s.flags;
            d.c = s.c;
            d.c_lo = s.c_lo;
            d.c_t = s.c_t;
            d.c_t_lo = s.c_t_lo;
            d.ldc = s.ldc;
            d.ldc_t = s.ldc_t;
            tiles += s.lower ? d.tiles_m * (d.tiles_m + 1) / 2 : d.tiles_m * d.tiles_n;
            ++probs;
            ++i;
        }
        batch.n_probs = probs;
        batch.total_tiles = tiles;
        if (tiles == 0) continue;
        kernel<<<tiles, 128, T::kSmemBytes, stream>>>(batch);
        after_launch("umma_gemm_kernel");
    }
}

void gemm_bf16(const std::vector<GemmSpec>& s, cudaStream_t st) { launch_gemms<1, 1, 3>(s, st); }
void gemm_tf32x3(const std::vector<GemmSpec>& s, cudaStream_t st) { launch_gemms<2, 2, 3>(s, st); }

// ------------------------------------------------------------ small kernels
struct Split2D {
    const float* src;
    float* hi;
    float* lo;
    int rows, cols, ld_src, ld_dst;
    float diag_add;  // added on the diagonal before splitting (damping)
};
constexpr int kMaxSplit = 16;
struct SplitBatch {
    Split2D e[kMaxSplit];
    int count;
};

__global__ void split_kernel(const __grid_constant__ SplitBatch b) {
    const Split2D& s = b.e[blockIdx.y];
    const int64_t total = static_cast<int64_t>(s.rows) * s.cols;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(idx / s.cols), c = static_cast<int>(idx % s.cols);
        float v = s.src[static_cast<int64_t>(r) * s.ld_src + c];
        if (r == c) v += s.diag_add;
        const float h = ptx::tf32_round(v);
        s.hi[static_cast<int64_t>(r) * s.ld_dst + c] = h;
        s.lo[static_cast<int64_t>(r) * s.ld_dst + c] = ptx::tf32_round(v - h);
    }
}

void launch_split(const std::vector<Split2D>& items, cudaStream_t st) {
    for (std::size_t i = 0; i < items.size(); i += kMaxSplit) {
        SplitBatch b{};
        b.count = static_cast<int>(std::min<std::size_t>(kMaxSplit, items.size() - i));
        int64_t biggest = 1;
        for (int j = 0; j < b.count; ++j) {
            b.e[j] = items[i + j];
            biggest = std::max<int64_t>(biggest, static_cast<int64_t>(b.e[j].rows) * b.e[j].cols);
        }
        const int blocks = static_cast<int>(std::min<int64_t>((biggest + 255) / 256, 148 * 8));
        split_kernel<<<dim3(blocks, b.count), 256, 0, st>>>(b);
        after_launch("split_kernel");
    }
}

__global__ void f32_to_bf16_kernel(const float* x, int64_t n, __nv_bfloat16* out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __float2bfloat16_rn(x[i]);
}

// ------------------------------------------------------------ damped inverse
inline int round4(int x) { return (x + 3) & ~3; }
inline size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// Workspace of one factor: five hi/lo pairs, each ldw x d fp32.
struct InvWs {
    int d = 0, ldw = 0;
    float *a[2], *l[2], *x[2], *xt[2], *t[2];
    int* info = nullptr;
};

size_t inverse_ws_bytes(int d) {
    const size_t plane = align256(static_cast<size_t>(round4(d)) * d * sizeof(float));
    return 10 * plane;
}

InvWs carve(void* base, int d) {
    InvWs w;
    w.d = d;
    w.ldw = round4(d);
    const size_t plane = align256(static_cast<size_t>(w.ldw) * d * sizeof(float));
    char* p = static_cast<char*>(base);
    float** slots[10] = {&w.a[0], &w.a[1], &w.l[0], &w.l[1], &w.x[0],
                         &w.x[1], &w.xt[0], &w.xt[1], &w.t[0], &w.t[1]};
    for (int i = 0; i < 10; ++i) *slots[i] = reinterpret_cast<float*>(p + i * plane);
    return w;
}

Operand sub(float* const pair[2], int ld, int r0, int c0, int rows, int k) {
    Operand o;
    o.hi = pair[0] + static_cast<size_t>(r0) * ld + c0;
    o.lo = pair[1] + static_cast<size_t>(r0) * ld + c0;
    o.rows = rows;
    o.k = k;
    o.ld = ld;
    return o;
}

void launch_leaves(const std::vector<InvWs>& ws, int o, int n, cudaStream_t st) {
    static std::once_flag once;
    std::call_once(once, [] {
        check(cudaFuncSetAttribute(leaf_chol_inv_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kLeafSmemBytes),
              "cudaFuncSetAttribute(leaf)");
    });
    for (std::size_t i = 0; i < ws.size(); i += kMaxLeafBatch) {
        LeafBatch b{};
        const int cnt = static_cast<int>(std::min<std::size_t>(kMaxLeafBatch, ws.size() - i));
        for (int j = 0; j < cnt; ++j) {
            const InvWs& w = ws[i + j];
            const size_t off = static_cast<size_t>(o) * w.ldw + o;
            b.e[j] = LeafArgs{w.a[0] + off, w.a[1] + off, w.x[0] + off, w.x[1] + off,
                              w.xt[0] + off, w.xt[1] + off, w.info, w.ldw, n, o};
        }
        leaf_chol_inv_kernel<<<cnt, kLeafThreads, kLeafSmemBytes, st>>>(b);
        after_launch("leaf_chol_inv_kernel");
    }
}

// Recursive blocked Cholesky + triangular inverse on the diagonal block
// [o, o+n) of every workspace (all of equal d): on return X = L^-1 and
// XT = L^-T hold that block, ready for the LAUUM product.
void inverse_rec(const std::vector<InvWs>& ws, int o, int n, cudaStream_t st) {
    if (n <= kLeaf) {
        launch_leaves(ws, o, n, st);
        return;
    }
    const int n1 = kTile * ((n + 2 * kTile - 1) / (2 * kTile));
    const int n2 = n - n1;
    inverse_rec(ws, o, n1, st);
    std::vector<GemmSpec> g1, g2;
    for (const InvWs& w : ws) {
        const int ld = w.ldw;
        // L21 = A21 * X11^T                                     (TRSM as GEMM)
        GemmSpec s;
        s.a = sub(w.a, ld, o + n1, o, n2, n1);
        s.b = sub(w.x, ld, o, o, n1, n1);
        s.rows = n2;
        s.cols = n1;
        s.k = n1;
        s.k_mode = K_TO_COL_TILE_END;
        s.flags = EPI_SPLIT;
        s.c = w.l[0] + static_cast<size_t>(o + n1) * ld + o;
        s.c_lo = w.l[1] + static_cast<size_t>(o + n1) * ld + o;
        s.ldc = ld;
        g1.push_back(s);
        // A22 -= L21 * L21^T                                    (SYRK, lower)
        GemmSpec u;
        u.a = sub(w.l, ld, o + n1, o, n2, n1);
        u.b = u.a;
        u.rows = u.cols = n2;
        u.k = n1;
        u.lower = true;
        u.alpha = -1.0f;
        u.beta = 1.0f;
        u.flags = EPI_SPLIT | EPI_READ_SPLIT;
        u.c = w.a[0] + static_cast<size_t>(o + n1) * ld + o + n1;
        u.c_lo = w.a[1] + static_cast<size_t>(o + n1) * ld + o + n1;
        u.ldc = ld;
        g2.push_back(u);
    }
    gemm_tf32x3(g1, st);
    gemm_tf32x3(g2, st);
    inverse_rec(ws, o + n1, n2, st);
    std::vector<GemmSpec> g3, g4;
    for (const InvWs& w : ws) {
        const int ld = w.ldw;
        // T^T = (L21 * X11)^T   (B operand = X11^T rows = XT11)
        GemmSpec s;
        s.a = sub(w.l, ld, o + n1, o, n2, n1);
        s.b = sub(w.xt, ld, o, o, n1, n1);
        s.rows = n2;
        s.cols = n1;
        s.k = n1;
        s.k_mode = K_FROM_COL_TILE;
        s.flags = EPI_SPLIT | EPI_TRANSPOSE;
        s.c = w.t[0];
        s.c_lo = w.t[1];
        s.ldc = ld;
        g3.push_back(s);
        // X21 = -X22 * T, also stored transposed into XT12
        GemmSpec x;
        x.a = sub(w.x, ld, o + n1, o + n1, n2, n2);
        x.b = sub(w.t, ld, 0, 0, n1, n2);
        x.rows = n2;
        x.cols = n1;
        x.k = n2;
        x.k_mode = K_TO_ROW_TILE_END;
        x.alpha = -1.0f;
        x.flags = EPI_SPLIT | EPI_ALSO_T;
        x.c = w.x[0] + static_cast<size_t>(o + n1) * ld + o;
        x.c_lo = w.x[1] + static_cast<size_t>(o + n1) * ld + o;
        x.c_t = w.xt[0] + static_cast<size_t>(o) * ld + o + n1;
        x.c_t_lo = w.xt[1] + static_cast<size_t>(o) * ld + o + n1;
        x.ldc = ld;
        x.ldc_t = ld;
        g4.push_back(x);
    }
    gemm_tf32x3(g3, st);
    gemm_tf32x3(g4, st);
}

void damped_inverse_group(const std::vector<const pf_inverse_problem*>& probs, cudaStream_t st) {
    const int d = probs.front()->d;
    std::vector<InvWs> ws;
    std::vector<Split2D> prep;
    for (const pf_inverse_problem* p : probs) {
        InvWs w = carve(p->workspace, d);
        w.info = p->d_info;
        check(cudaMemsetAsync(p->d_info, 0, sizeof(int), st), "memset(info)");
        prep.push_back(Split2D{p->m, w.a[0], w.a[1], d, d, p->ldm, w.ldw, p->damping});
        ws.push_back(w);
    }
    launch_split(prep, st);  // A = split(M + lambda I)
    inverse_rec(ws, 0, d, st);
    // LAUUM: M^-1 = X^T X = XT * XT^T  (lower tiles, mirrored)
    std::vector<GemmSpec> g;
    for (std::size_t i = 0; i < ws.size(); ++i) {
        const InvWs& w = ws[i];
        const pf_inverse_problem* p = probs[i];
        GemmSpec s;
        s.a = sub(const_cast<InvWs&>(w).xt, w.ldw, 0, 0, d, d);
        s.b = s.a;
        s.rows = s.cols = s.k = d;
        s.lower = true;
        s.k_mode = K_FROM_ROW_TILE;
        s.flags = EPI_MIRROR;
        if (p->minv_lo) {
            s.flags |= EPI_SPLIT;
        } else if (reinterpret_cast<uintptr_t>(p->minv) % 16 == 0 && p->ldinv % 4 == 0) {
            s.flags |= EPI_VEC4;
        }
        s.c = p->minv;
        s.c_lo = p->minv_lo;
        s.ldc = p->ldinv;
        g.push_back(s);
    }
    gemm_tf32x3(g, st);
}

// ------------------------------------------------------------ precondition
struct PrecWs {
    float *ainv[2], *binv[2], *g[2], *ut[2];
    int ldi, ldo;
};

size_t precondition_ws_bytes(int d_out, int d_in) {
    const size_t ldi = round4(d_in), ldo = round4(d_out);
    return 2 * (align256(ldi * d_in * 4) + align256(ldo * d_out * 4) + align256(ldi * d_out * 4) +
                align256(ldo * d_in * 4));
}

PrecWs carve_prec(void* base, int d_out, int d_in) {
    PrecWs w;
    w.ldi = round4(d_in);
    w.ldo = round4(d_out);
    char* p = static_cast<char*>(base);
    auto take = [&](size_t bytes) {
        float* f = reinterpret_cast<float*>(p);
        p += align256(bytes);
        return f;
    };
    for (int h = 0; h < 2; ++h) w.ainv[h] = take(static_cast<size_t>(w.ldi) * d_in * 4);
    for (int h = 0; h < 2; ++h) w.binv[h] = take(static_cast<size_t>(w.ldo) * d_out * 4);
    for (int h = 0; h < 2; ++h) w.g[h] = take(static_cast<size_t>(w.ldi) * d_out * 4);
    for (int h = 0; h < 2; ++h) w.ut[h] = take(static_cast<size_t>(w.ldo) * d_in * 4);
    return w;
}

// problems whose inverses are plain fp32 get them split into the workspace
void precondition_group(const std::vector<pf_precondition_problem>& probs, bool split_inverses,
                        const std::vector<const float*>& a_plain,
                        const std::vector<const float*>& b_plain, cudaStream_t st) {
    std::vector<Split2D> splits;
    std::vector<PrecWs> ws;
    for (std::size_t i = 0; i < probs.size(); ++i) {
        const auto& p = probs[i];
        PrecWs w = carve_prec(p.workspace, p.d_out, p.d_in);
        splits.push_back(Split2D{p.grad, w.g[0], w.g[1], p.d_out, p.d_in, p.d_in, w.ldi, 0.0f});
        if (split_inverses) {
            splits.push_back(
                Split2D{a_plain[i], w.ainv[0], w.ainv[1], p.d_in, p.d_in, p.d_in, w.ldi, 0.0f});
            splits.push_back(
                Split2D{b_plain[i], w.binv[0], w.binv[1], p.d_out, p.d_out, p.d_out, w.ldo, 0.0f});
        }
        ws.push_back(w);
    }
    launch_split(splits, st);
    std::vector<GemmSpec> g1, g2;
    for (std::size_t i = 0; i < probs.size(); ++i) {
        const auto& p = probs[i];
        PrecWs& w = ws[i];
        Operand ainv, binv;
        if (split_inverses) {
            ainv = Operand{w.ainv[0], w.ainv[1], p.d_in, p.d_in, w.ldi, false};
            binv = Operand{w.binv[0], w.binv[1], p.d_out, p.d_out, w.ldo, false};
        } else {
            ainv = Operand{p.a_inv_hi, p.a_inv_lo, p.d_in, p.d_in, p.d_in, false};
            binv = Operand{p.b_inv_hi, p.b_inv_lo, p.d_out, p.d_out, p.d_out, false};
        }
        // U^T = A^-1 G^T   ( [d_in x d_out] )
        GemmSpec s;
        s.a = ainv;
        s.b = Operand{w.g[0], w.g[1], p.d_out, p.d_in, w.ldi, false};
        s.rows = p.d_in;
        s.cols = p.d_out;
        s.k = p.d_in;
        s.flags = EPI_SPLIT;
        s.c = w.ut[0];
        s.c_lo = w.ut[1];
        s.ldc = w.ldo;
        g1.push_back(s);
        // P = B^-1 U ; epilogue W -= eta P  (or P itself)
        GemmSpec t;
        t.a = binv;
        t.b = Operand{w.ut[0], w.ut[1], p.d_in, p.d_out, w.ldo, false};
        t.rows = p.d_out;
        t.cols = p.d_in;
        t.k = p.d_out;
        float* dst = p.w ? p.w : p.p_out;
        t.alpha = p.w ? -p.eta : 1.0f;
        t.beta = p.w ? 1.0f : 0.0f;
        t.c = dst;
        t.ldc = p.d_in;
        if (reinterpret_cast<uintptr_t>(dst) % 16 == 0 && p.d_in % 4 == 0) t.flags |= EPI_VEC4;
        g2.push_back(t);
    }
    gemm_tf32x3(g1, st);
    gemm_tf32x3(g2, st);
}

bool aligned16(const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; }

}  // namespace
}  // namespace pf

// ============================================================== C-ABI
using namespace pf;

extern "C" {

int64_t pf_kernel_launch_count(void) { return g_launches.load(); }

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
                throw std::invalid_argument("pf_curvature_syrk: shape mismatch");
            if (p.ldx % 8 != 0 || !aligned16(p.x))
                throw std::invalid_argument("pf_curvature_syrk: x needs 16-B rows (ldx % 8 == 0)");
            GemmSpec s;
            s.a = Operand{p.x, nullptr, p.d, p.n, p.ldx, true};
            s.b = s.a;
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
                throw std::invalid_argument("cholesky_spd_inverse: bad arguments");
            if (!aligned16(p.workspace)) throw std::invalid_argument("workspace must be 16-B aligned");
            if (p.minv_lo && (p.ldinv % 4 != 0 || !aligned16(p.minv) || !aligned16(p.minv_lo)))
                throw std::invalid_argument("split inverse output needs 16-B rows");
            order.push_back(&p);
        }
        std::stable_sort(order.begin(), order.end(),
                         [](auto* a, auto* b) { return a->d < b->d; });
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        for (std::size_t i = 0; i < order.size();) {
            std::size_t j = i;
            while (j < order.size() && order[j]->d == order[i]->d && j - i < 16) ++j;
            damped_inverse_group({order.begin() + i, order.begin() + j}, st);
            i = j;
        }
        return 0;
    });
}

int pf_damped_inverse(const float* m, int d, int ldm, float damping, float* minv, float* minv_lo,
                      int ldinv, void* workspace, size_t workspace_bytes, int* d_info,
                      void* stream) {
    return pf_detail::guard([&] {
        if (d >= 1 && workspace_bytes < inverse_ws_bytes(d))
            throw std::invalid_argument("workspace too small");
        pf_inverse_problem p{m, minv, minv_lo, d, ldm, ldinv, damping, workspace, d_info};
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

static int precondition_plain(const float* b_inv, const float* grad, const float* a_inv,
                              float* w, float* p_out, int d_out, int d_in, float eta,
                              void* workspace, size_t workspace_bytes, void* stream) {
    return pf_detail::guard([&] {
        if (d_out < 1 || d_in < 1 || !b_inv || !grad || !a_inv || (!w && !p_out) || !workspace)
            throw std::invalid_argument("precondition: shape mismatch");
        if (workspace_bytes < precondition_ws_bytes(d_out, d_in))
            throw std::invalid_argument("workspace too small");
        if (!aligned16(workspace)) throw std::invalid_argument("workspace must be 16-B aligned");
        pf_precondition_problem p{};
        p.grad = grad;
        p.w = w;
        p.p_out = p_out;
        p.d_out = d_out;
        p.d_in = d_in;
        p.eta = eta;
        p.workspace = workspace;
        precondition_group({p}, true, {a_inv}, {b_inv}, static_cast<cudaStream_t>(stream));
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

int pf_precondition_update_split(const pf_precondition_problem* problems, int count,
                                 void* stream) {
    return pf_detail::guard([&] {
        std::vector<pf_precondition_problem> v;
        for (int i = 0; i < count; ++i) {
            const auto& p = problems[i];
            if (p.d_out < 1 || p.d_in < 1 || !p.grad || (!p.w && !p.p_out) || !p.workspace ||
                !p.a_inv_hi || !p.a_inv_lo || !p.b_inv_hi || !p.b_inv_lo)
                throw std::invalid_argument("precondition: shape mismatch");
            if (p.d_in % 4 != 0 || p.d_out % 4 != 0)
                throw std::invalid_argument("split inverses need d % 4 == 0");
            v.push_back(p);
        }
        for (std::size_t i = 0; i < v.size(); i += kMaxProbs) {
            std::vector<pf_precondition_problem> chunk(
                v.begin() + i, v.begin() + std::min(v.size(), i + kMaxProbs));
            precondition_group(chunk, false, {}, {}, static_cast<cudaStream_t>(stream));
        }
        return 0;
    });
}

int pf_split_tf32(const float* x, int64_t n, float* hi, float* lo, void* stream) {
    return pf_detail::guard([&] {
        if (n < 0 || n > INT32_MAX || !x || !hi || !lo) throw std::invalid_argument("bad split");
        launch_split({Split2D{x, hi, lo, 1, static_cast<int>(n), static_cast<int>(n),
                              static_cast<int>(n), 0.0f}},
                     static_cast<cudaStream_t>(stream));
        return 0;
    });
}

int pf_f32_to_bf16(const float* x, int64_t n, void* out, void* stream) {
    return pf_detail::guard([&] {
        if (n < 0 || !x || !out) throw std::invalid_argument("bad convert");
        const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
        if (blocks > 0) {
            f32_to_bf16_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
                x, n, static_cast<__nv_bfloat16*>(out));
            after_launch("f32_to_bf16_kernel");
        }
        return 0;
    });
}

}  // extern "C"
