// Diagonal-block kernel of the damped inverse: for one 128x128 diagonal block
// A_kk (already holding all trailing updates) compute
//     L_kk = chol(A_kk)          and          X_kk = L_kk^-1
// on the SIMT cores, entirely in shared memory (fp32 storage, every dot
// product accumulated in fp64 and rounded once), and write X_kk (lower,
// explicit zeros above) and X_kk^T (upper, zeros below).
//
// Follows the reference arithmetic (proj/src/kfac/matrix.cpp:117-153):
// pivot test `!(diag > 0) || !isfinite(diag)` -> 1-based failing column in
// *info; L^-1 by forward substitution.  Organisation (B200-first): four
// 32-wide panels; each panel is factored by ONE WARP in registers (lane i
// owns row i, column broadcasts via shuffles) together with its 32x32
// triangular inverse; the panel solve and the trailing update are small
// register-tiled smem GEMMs over all 16 warps.
#pragma once

#include <climits>
#include <cstdint>

#include "ptx.cuh"

namespace pf {

constexpr int kLeaf = 128;
constexpr int kLeafPitch = 129;  // +1 pad: column walks hit 32 distinct banks
constexpr int kLeafThreads = 512;
constexpr int kMaxLeafBatch = 32;
constexpr int kLeafSmemBytes = 2 * kLeaf * kLeafPitch * 4 + 16;

struct LeafArgs {
    const float* a;
    float* x;
    float* xt;
    int* info;
    int ld;    // shared leading dimension of a / x / xt
    int n;     // block size (<= 128; the tail block of a non-multiple-of-128 d)
    int col0;  // global column of the block (for info)
};

struct LeafBatch {
    LeafArgs e[kMaxLeafBatch];
};

// One small product over shared memory, all threads cooperating:
//   C[i][j] = beta*C[i][j] + alpha * sum_k A[i*ars + k*aks] * B[j*bcs + k*bks]
// i < M, j < N (multiples of 32), 4x4 register micro-tiles with strided rows
// and columns (rows ti + s*M/4) so lane-consecutive tiles hit distinct banks.
// `lower` skips outputs with j > i.  Results are staged in registers and
// written after a barrier, so C may alias A or B (in-place panel solves).
struct SmemGemm {
    const float* a;
    int ars, aks;
    const float* b;
    int bcs, bks;
    float* c;
    int M, N, K;
    float alpha, beta;
    int lower;
};

template <int kMaxPerThread>
__device__ void smem_gemm(const SmemGemm* probs, int count) {
    int total = 0;
    for (int q = 0; q < count; ++q) total += (probs[q].M / 4) * (probs[q].N / 4);
    double acc[kMaxPerThread][4][4];
    int where[kMaxPerThread][3];
#pragma unroll
    for (int s = 0; s < kMaxPerThread; ++s) {
        where[s][0] = -1;
        const int t = threadIdx.x + s * kLeafThreads;
        if (t >= total) continue;
        int q = 0, base = 0;
        while (t - base >= (probs[q].M / 4) * (probs[q].N / 4)) {
            base += (probs[q].M / 4) * (probs[q].N / 4);
            ++q;
        }
        const SmemGemm& P = probs[q];
        const int nt = P.N / 4;
        const int ti = (t - base) / nt, tj = (t - base) % nt;
        const int mstep = P.M / 4, nstep = P.N / 4;
        where[s][0] = q;
        where[s][1] = ti;
        where[s][2] = tj;
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[s][r][c] = 0.0f;
        for (int k = 0; k < P.K; ++k) {
            double av[4], bv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) av[r] = P.a[(ti + r * mstep) * P.ars + k * P.aks];
#pragma unroll
            for (int c = 0; c < 4; ++c) bv[c] = P.b[(tj + c * nstep) * P.bcs + k * P.bks];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[s][r][c] = fma(av[r], bv[c], acc[s][r][c]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kMaxPerThread; ++s) {
        const int q = where[s][0];
        if (q < 0) continue;
        const SmemGemm& P = probs[q];
        const int mstep = P.M / 4, nstep = P.N / 4;
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int i = where[s][1] + r * mstep;
                const int j = where[s][2] + c * nstep;
                if (P.lower && j > i) continue;
                float* dst = P.c + i * kLeafPitch + j;
                const double old = P.beta != 0.0f ? static_cast<double>(P.beta) * *dst : 0.0;
                *dst = static_cast<float>(old + static_cast<double>(P.alpha) * acc[s][r][c]);
            }
    }
    __syncthreads();
}

// Warp 0: Cholesky of the 32x32 block at (c0, c0) of Ls in registers, then
// its inverse into Xs (full 32x32 with zeros above the diagonal).
__device__ void panel_chol_inv32(float* Ls, float* Xs, int c0, int col_base, int n, int* bad) {
    const int lane = threadIdx.x & 31;
    double a[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = (j <= lane) ? Ls[(c0 + lane) * kLeafPitch + c0 + j] : 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        double piv = __shfl_sync(0xffffffffu, a[k], k);
        if (!(piv > 0.0) || !isfinite(piv)) {
            if (lane == 0 && c0 + k < n) atomicMin(bad, col_base + c0 + k + 1);
            piv = 1.0;  // keep going; the caller reports the failure
        }
        const double lkk = sqrt(piv);
        if (lane == k) a[k] = lkk;
        if (lane > k) a[k] = a[k] / lkk;
#pragma unroll
        for (int j = k + 1; j < 32; ++j) {
            const double ljk = __shfl_sync(0xffffffffu, a[k], j);
            if (lane >= j) a[j] = fma(-a[k], ljk, a[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j)
        Ls[(c0 + lane) * kLeafPitch + c0 + j] = (j <= lane) ? static_cast<float>(a[j]) : 0.0f;
    __syncwarp();
    // column `lane` of L^-1 by forward substitution (reference matrix.cpp:145-153)
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < i; ++k) s = fma(static_cast<double>(Ls[(c0 + i) * kLeafPitch + c0 + k]), x[k], s);
        const double lii = Ls[(c0 + i) * kLeafPitch + c0 + i];
        x[i] = (i == lane) ? 1.0 / lii : (i > lane ? -s / lii : 0.0);
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) Xs[(c0 + i) * kLeafPitch + c0 + lane] = static_cast<float>(x[i]);
}

__global__ void __launch_bounds__(kLeafThreads, 1) leaf_chol_inv_kernel(const __grid_constant__ LeafBatch batch) {
    extern __shared__ float leaf_smem[];
    float* Ls = leaf_smem;
    float* Xs = leaf_smem + kLeaf * kLeafPitch;
    int* bad = reinterpret_cast<int*>(Xs + kLeaf * kLeafPitch);
    const LeafArgs& A = batch.e[blockIdx.x];
    const int n = A.n;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;

    if (tid == 0) *bad = INT_MAX;
    // load lower triangle of A (hi + lo); pad beyond n with the identity
    for (int idx = tid; idx < kLeaf * kLeaf; idx += kLeafThreads) {
        const int r = idx / kLeaf, c = idx % kLeaf;
        float v;
        if (r < n && c < n)
            v = (c <= r) ? A.a[(size_t)r * A.ld + c] : 0.0f;
        else
            v = (r == c) ? 1.0f : 0.0f;
        Ls[r * kLeafPitch + c] = v;
        Xs[r * kLeafPitch + c] = 0.0f;
    }
    __syncthreads();

    // ---- blocked right-looking Cholesky, 32-wide panels
    for (int p = 0; p < 4; ++p) {
        const int c0 = 32 * p;
        if (warp == 0) panel_chol_inv32(Ls, Xs, c0, A.col0, n, bad);
        __syncthreads();
        if (p == 3) break;
        const int m = kLeaf - c0 - 32;  // rows below the panel
        // panel solve  L[i, p] = A[i, p] * Linv_pp^T     (in place)
        {
            SmemGemm g{Ls + (c0 + 32) * kLeafPitch + c0, kLeafPitch, 1,
                       Xs + c0 * kLeafPitch + c0,        kLeafPitch, 1,
                       Ls + (c0 + 32) * kLeafPitch + c0, m, 32, 32, 1.0f, 0.0f, 0};
            smem_gemm<1>(&g, 1);
        }
        // trailing update  A[i, j] -= L[i, p] L[j, p]^T   (lower part)
        {
            SmemGemm g{Ls + (c0 + 32) * kLeafPitch + c0, kLeafPitch, 1,
                       Ls + (c0 + 32) * kLeafPitch + c0, kLeafPitch, 1,
                       Ls + (c0 + 32) * kLeafPitch + c0 + 32, m, m, 32, -1.0f, 1.0f, 1};
            smem_gemm<2>(&g, 1);
        }
    }

    // ---- triangular inverse of the off-diagonal 32-blocks, by block diagonal:
    //   X[bi,bj] = -Linv_bi * ( sum_{k=bj}^{bi-1} L[bi,k] X[k,bj] )
    // The temporary sum is staged in the (unused) upper triangle of Ls.
    for (int dgap = 1; dgap < 4; ++dgap) {
        SmemGemm g[3];
        int cnt = 0;
        for (int bj = 0; bj + dgap < 4; ++bj) {
            const int bi = bj + dgap;
            // T = L[bi, bj..bi-1] * X[bj..bi-1, bj]   (NN: B indexed [k][j])
            g[cnt++] = SmemGemm{Ls + (32 * bi) * kLeafPitch + 32 * bj, kLeafPitch, 1,
                                Xs + (32 * bj) * kLeafPitch + 32 * bj, 1, kLeafPitch,
                                Ls + (32 * bj) * kLeafPitch + 32 * bi, 32, 32, 32 * dgap,
                                1.0f, 0.0f, 0};
        }
        smem_gemm<1>(g, cnt);
        cnt = 0;
        for (int bj = 0; bj + dgap < 4; ++bj) {
            const int bi = bj + dgap;
            g[cnt++] = SmemGemm{Xs + (32 * bi) * kLeafPitch + 32 * bi, kLeafPitch, 1,
                                Ls + (32 * bj) * kLeafPitch + 32 * bi, 1, kLeafPitch,
                                Xs + (32 * bi) * kLeafPitch + 32 * bj, 32, 32, 32,
                                -1.0f, 0.0f, 0};
        }
        smem_gemm<1>(g, cnt);
    }

    // ---- store X (lower, zeros above) and X^T (upper, zeros below)
    for (int idx = tid; idx < n * n; idx += kLeafThreads) {
        const int r = idx / n, c = idx % n;
        A.x[(size_t)r * A.ld + c] = (c <= r) ? Xs[r * kLeafPitch + c] : 0.0f;
        A.xt[(size_t)r * A.ld + c] = (r <= c) ? Xs[c * kLeafPitch + r] : 0.0f;
    }
    if (tid == 0 && *bad != INT_MAX) {
        // keep the smallest failing column across blocks (0 = success)
        int old = *A.info;
        while (old == 0 || *bad < old) {
            const int seen = atomicCAS(A.info, old, *bad);
            if (seen == old) break;
            old = seen;
        }
    }
}

}  // namespace pf
