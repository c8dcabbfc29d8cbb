// Critical-chain step of the right-looking damped inverse (kfac_ops.cu,
// cholesky_blocked), one launch per 128-column panel k >= 1:
//
//   chain_leaf_kernel<kCl>   one cluster of kCl CTAs per problem:
//     1. L_t = A[k, k-1] X_{k-1}^T          (the one L tile the next diagonal
//                                           block needs; rows split over the
//                                           cluster, fp32 SIMT, K = 128)
//     2. A[k, k] -= L_t L_t^T  (lower)      (rows split over the cluster; L_t
//                                           rows exchanged through DSMEM)
//     3. CTA 0: leaf(k) on the updated block (leaf.cuh): X_k = chol(A_kk)^-1
//
// This replaces the four dependent launches that used to sit between two
// leaves (slice X, TRSM of the whole column, slice L, one-tile diagonal
// update; ~17 us per panel on B200) with one short prologue: the full-column
// TRSM and its digit slices now run on the side streams, off the chain, and
// compute their own copy of this tile for the stored L (both copies are
// fp32-accurate; the factorisation only ever mixes them at rounding level).
//
// Arithmetic: plain fp32 FMA in ascending k, like LAPACK's SGEMM/SSYRK block
// updates (reference proj/src/kfac/matrix.cpp:117-134 updates in place with
// the same products).
#pragma once

#include <cooperative_groups.h>

#include "leaf.cuh"

namespace pf {

#ifdef PF_CHAIN_PROBE
// globaltimer stamps (ns) of CTA 0 per launch: entry, after griddepcontrol.wait,
// operands staged, step 1 + sync, gather + sync, step 2 + sync, leaf done
__device__ long long g_chain_probe[64 * 8];
__device__ int g_chain_probe_n;
__device__ __forceinline__ long long chain_gt() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define PF_CSTAMP(i) \
    if (threadIdx.x == 0 && rank == 0 && blockIdx.x == 0) st[i] = chain_gt()
#else
#define PF_CSTAMP(i)
#endif

struct ChainArgs {
    const float* xprev;  // X_{k-1}: 128 x 128 lower block of L^-1 (ld = leaf.ld)
    const float* arow;   // A[k, k-1]: leaf.n x 128 (ld = leaf.ld), fully updated by panels < k-1
    float* akk;          // A[k, k] (updated by panels < k-1; step 2 finishes it in place)
    LeafArgs leaf;       // block k (leaf.a == akk)
};

struct ChainBatch {
    ChainArgs e[kMaxLeafBatch];
};

constexpr int kChainPitch = 132;  // float4-aligned rows, banks skewed by 4 per row

template <int kCl>
constexpr int chain_smem_bytes() {
    constexpr int rows = kLeaf / kCl;
    constexpr int steps = (2 * kLeaf * kChainPitch + 2 * rows * kChainPitch) * 4;
    return steps > kLeafSmemBytes ? steps : kLeafSmemBytes;
}

// Step 1 / step 2 register tile: kRT rows x 4 columns per thread.
template <int kCl>
__global__ void __launch_bounds__(kLeafThreads, 1) chain_leaf_kernel(const __grid_constant__ ChainBatch batch) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) float sm[];
    constexpr int R = kLeaf / kCl;           // rows per CTA
    constexpr int kRT = R / 8;               // rows per thread (8 row groups x 32 column groups)
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    const ChainArgs& P = batch.e[blockIdx.x / kCl];
    const int n = P.leaf.n, ld = P.leaf.ld;
    const int tid = threadIdx.x;
    float* XT = sm;                          // [128][pitch]: X_{k-1}^T, then L_t^T (all rows)
    float* Ar = XT + kLeaf * kChainPitch;    // [128][pitch]: (reuse) unused rows
    float* Ak = Ar;                          // [R][pitch]: my rows of A[k, k-1]
    float* Lr = Ar + R * kChainPitch;        // [R][pitch]: my rows of L_t (read remotely)
    (void)Ar;
    const int g0 = rank * R;                 // first global row of this CTA
    const int ti = tid >> 5, tj = tid & 31;  // row group (warp), column group (lane)

#ifdef PF_CHAIN_PROBE
    long long st[8];
#endif
    PF_CSTAMP(0);
    ptx::grid_dep_wait();  // PDL: X_{k-1} comes from the previous chain step
    PF_CSTAMP(1);
    // ---- stage X_{k-1}^T (XT[c][j] = X[j][c]; the leaf wrote zeros above the diagonal)
    for (int idx = tid; idx < kLeaf * kLeaf / 4; idx += kLeafThreads) {
        const int j = idx & 127, c = 4 * (idx >> 7);
        const float4 v = __ldcg(reinterpret_cast<const float4*>(P.xprev + static_cast<size_t>(j) * ld + c));
        XT[(c + 0) * kChainPitch + j] = v.x;
        XT[(c + 1) * kChainPitch + j] = v.y;
        XT[(c + 2) * kChainPitch + j] = v.z;
        XT[(c + 3) * kChainPitch + j] = v.w;
    }
    for (int idx = tid; idx < R * kLeaf / 4; idx += kLeafThreads) {
        const int i = idx >> 5, c = 4 * (idx & 31);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (g0 + i < n) v = __ldcg(reinterpret_cast<const float4*>(P.arow + static_cast<size_t>(g0 + i) * ld + c));
        *reinterpret_cast<float4*>(Ak + i * kChainPitch + c) = v;
    }
    __syncthreads();
    PF_CSTAMP(2);
    // ---- step 1: L_t[g0 + i][j] = sum_{c <= j} A[i][c] X[j][c]
    {
        float acc[kRT][4];
#pragma unroll
        for (int u = 0; u < kRT; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[u][q] = 0.0f;
        const int cmax = 4 * tj + 4;  // X lower: X[j][c] = 0 for c > j
#pragma unroll 4
        for (int c = 0; c < cmax; ++c) {
            const float4 x = *reinterpret_cast<const float4*>(XT + c * kChainPitch + 4 * tj);
#pragma unroll
            for (int u = 0; u < kRT; ++u) {
                const float a = Ak[(kRT * ti + u) * kChainPitch + c];
                acc[u][0] = fmaf(a, x.x, acc[u][0]);
                acc[u][1] = fmaf(a, x.y, acc[u][1]);
                acc[u][2] = fmaf(a, x.z, acc[u][2]);
                acc[u][3] = fmaf(a, x.w, acc[u][3]);
            }
        }
#pragma unroll
        for (int u = 0; u < kRT; ++u)
            *reinterpret_cast<float4*>(Lr + (kRT * ti + u) * kChainPitch + 4 * tj) =
                make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
    }
    cluster.sync();  // every CTA's L_t rows are visible cluster-wide; X^T no longer needed
    PF_CSTAMP(3);
    // ---- gather L_t^T rows 0 .. g0 + R - 1 (what my diagonal rows need) into XT
    const int need = g0 + R;
    for (int idx = tid; idx < need * (kLeaf / 4); idx += kLeafThreads) {
        const int j = idx % need, c = 4 * (idx / need);
        const float* src = cluster.map_shared_rank(Lr, j / R) + (j % R) * kChainPitch + c;
        const float4 v = *reinterpret_cast<const float4*>(src);
        XT[(c + 0) * kChainPitch + j] = v.x;
        XT[(c + 1) * kChainPitch + j] = v.y;
        XT[(c + 2) * kChainPitch + j] = v.z;
        XT[(c + 3) * kChainPitch + j] = v.w;
    }
    cluster.sync();  // no remote reads past this point (CTA 0 may reuse its shared memory)
    PF_CSTAMP(4);
    // ---- step 2: A[k][k][g0 + i][j] -= sum_c L_t[g0 + i][c] L_t[j][c],  j <= g0 + i
    if (4 * tj <= g0 + R - 1) {
        float acc[kRT][4];
#pragma unroll
        for (int u = 0; u < kRT; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[u][q] = 0.0f;
#pragma unroll 4
        for (int c = 0; c < kLeaf; ++c) {
            const float4 b = *reinterpret_cast<const float4*>(XT + c * kChainPitch + 4 * tj);
#pragma unroll
            for (int u = 0; u < kRT; ++u) {
                const float a = Lr[(kRT * ti + u) * kChainPitch + c];
                acc[u][0] = fmaf(a, b.x, acc[u][0]);
                acc[u][1] = fmaf(a, b.y, acc[u][1]);
                acc[u][2] = fmaf(a, b.z, acc[u][2]);
                acc[u][3] = fmaf(a, b.w, acc[u][3]);
            }
        }
#pragma unroll
        for (int u = 0; u < kRT; ++u) {
            const int g = g0 + kRT * ti + u;
            if (g >= n) continue;
            float* dst = P.akk + static_cast<size_t>(g) * ld;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = 4 * tj + q;
                if (j <= g) dst[j] = __ldcg(dst + j) - acc[u][q];
            }
        }
    }
    __threadfence();
    cluster.sync();  // the updated diagonal block is complete (global, L2)
    PF_CSTAMP(5);
    if (rank != 0) return;
    leaf_body(P.leaf, sm, true);
#ifdef PF_CHAIN_PROBE
    PF_CSTAMP(6);
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const int slot = atomicAdd(&g_chain_probe_n, 1);
        if (slot < 64)
            for (int i = 0; i < 7; ++i) g_chain_probe[slot * 8 + i] = st[i];
    }
#endif  // (griddepcontrol.wait again is a no-op; it triggers the next step before its store)
}

}  // namespace pf
