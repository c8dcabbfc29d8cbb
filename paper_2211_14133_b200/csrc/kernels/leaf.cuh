// Diagonal-block kernel of the damped inverse: for one 128x128 diagonal block
// A_kk (already holding all trailing updates) compute
//     L_kk = chol(A_kk)          and          X_kk = L_kk^-1
// on the SIMT cores, entirely in shared memory, and write X_kk (lower,
// explicit zeros above) and X_kk^T (upper, zeros below).
//
// Follows the reference arithmetic (proj/src/kfac/matrix.cpp:117-153):
// pivot test `!(diag > 0) || !isfinite(diag)` -> 1-based failing column in
// *info; L^-1 by forward substitution.  Organisation (B200-first), fp32 like
// LAPACK's SPOTRF/STRTRI block steps:
//   * four 32-wide panels; the 32x32 diagonal block of each is factored by
//     ONE WARP in registers (lane i owns row i).  The column being
//     eliminated is always register a[0]: after each step the row is rotated
//     left, so every register index is a compile-time constant while the
//     32-step loop stays a loop (a fully unrolled version stalled on
//     instruction fetch: it ran once per panel, ~20K instructions);
//   * the panel's 32x32 triangular inverse: one lane per column;
//   * panel solve, trailing update and the off-diagonal blocks of L^-1 are
//     4x4 register-tiled shared-memory products over all 8 warps.
#pragma once

#include <climits>
#include <cstdint>

#include "ptx.cuh"

namespace pf {

constexpr int kLeaf = 128;
constexpr int kLeafPitch = 129;  // +1 pad: column walks hit 32 distinct banks
constexpr int kLeafThreads = 256;
constexpr int kLeafWarps = kLeafThreads / 32;
constexpr int kMaxLeafBatch = 32;
constexpr int kLeafSmemBytes = 2 * kLeaf * kLeafPitch * 4 + kLeaf * 4 + 16;

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

// C[i][j] = alpha * sum_k A[i][k] B[k][j]  (+ C[i][j] if accumulate) over an
// M x N block (multiples of 4), 4x4 fp32 micro-tiles with strided rows/cols
// (row ti + r*M/4) so lane-consecutive tiles hit distinct banks.  A(i,k) at
// a[i*ars + k*aks], B(k,j) at b[k*bks + j*bcs], C(i,j) at c[i*kLeafPitch + j].
// `lower`: only j <= i is written.  Caller guarantees C does not alias A/B.
__device__ __forceinline__ void leaf_mm(const float* a, int ars, int aks, const float* b, int bks,
                                        int bcs, float* c, int M, int N, int K, float alpha,
                                        bool accumulate, bool lower, int tid, int nthreads) {
    const int mt = M / 4, nt = N / 4;
    for (int t = tid; t < mt * nt; t += nthreads) {
        const int ti = t / nt, tj = t % nt;
        float acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[r][q] = 0.0f;
        const float* ap = a + ti * ars;
        const float* bp = b + tj * bcs;
#pragma unroll 4
        for (int k = 0; k < K; ++k) {
            float av[4], bv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) av[r] = ap[r * mt * ars + k * aks];
#pragma unroll
            for (int q = 0; q < 4; ++q) bv[q] = bp[k * bks + q * nt * bcs];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[r][q] = fmaf(av[r], bv[q], acc[r][q]);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int i = ti + r * mt, j = tj + q * nt;
                if (lower && j > i) continue;
                float* dst = c + i * kLeafPitch + j;
                *dst = accumulate ? fmaf(alpha, acc[r][q], *dst) : alpha * acc[r][q];
            }
    }
}

// One warp: Cholesky of the 32x32 block at (c0, c0) of Ls (in place, zeros
// above the diagonal), then its inverse into Xs (zeros above the diagonal).
__device__ __forceinline__ void panel_chol_inv32(float* Ls, float* Xs, float* rdiag, int c0,
                                                 int col_base, int n, int* bad) {
    const int lane = threadIdx.x & 31;
    float* row = Ls + (c0 + lane) * kLeafPitch + c0;
    float a[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = row[j];
#pragma unroll 1
    for (int k = 0; k < 32; ++k) {
        // a[0] holds column k of this lane's row (rotated k times)
        float piv = __shfl_sync(0xffffffffu, a[0], k);
        if (!(piv > 0.0f) || !isfinite(piv)) {
            if (lane == 0 && c0 + k < n) *bad = min(*bad, col_base + c0 + k + 1);  // one warp: no race
            piv = 1.0f;  // keep going; the caller reports the failure
        }
        const float rl = rsqrtf(piv);
        const float l = lane > k ? a[0] * rl : (lane == k ? piv * rl : 0.0f);
        row[k] = l;  // L[lane][c0+k] (0 above the diagonal)
        if (lane == k) rdiag[c0 + k] = rl;
        // all shuffles first (independent), then the dependent FMAs
        float lj[32];
#pragma unroll
        for (int j = 1; j < 32; ++j) lj[j] = __shfl_sync(0xffffffffu, l, (k + j) & 31);
#pragma unroll
        for (int j = 1; j < 32; ++j)
            if (lane >= k + j) a[j] = fmaf(-l, lj[j], a[j]);
#pragma unroll
        for (int j = 0; j < 31; ++j) a[j] = a[j + 1];
        a[31] = 0.0f;
    }
    __syncwarp();
    // column `lane` of L^-1 by forward substitution (reference matrix.cpp:145-153),
    // column-oriented: every index is a compile-time constant
    float x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? 1.0f : 0.0f;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        x[i] *= rdiag[c0 + i];
#pragma unroll
        for (int r = i + 1; r < 32; ++r) x[r] = fmaf(-Ls[(c0 + r) * kLeafPitch + c0 + i], x[i], x[r]);
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) Xs[(c0 + i) * kLeafPitch + c0 + lane] = x[i];
}

__global__ void __launch_bounds__(kLeafThreads, 1) leaf_chol_inv_kernel(const __grid_constant__ LeafBatch batch) {
    extern __shared__ float leaf_smem[];
    float* Ls = leaf_smem;
    float* Xs = leaf_smem + kLeaf * kLeafPitch;
    float* rdiag = Xs + kLeaf * kLeafPitch;  // 1 / L[k][k]
    int* bad = reinterpret_cast<int*>(rdiag + kLeaf);
    const LeafArgs& A = batch.e[blockIdx.x];
    const int n = A.n;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    if (tid == 0) *bad = INT_MAX;
    // load the lower triangle of A; pad beyond n with the identity.  Full
    // blocks (n == 128, 16-byte aligned rows) use float4 loads, all in flight.
    const bool vec = n == kLeaf && (A.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(A.a) & 15) == 0);
    if (vec) {
        constexpr int kPer = kLeaf * kLeaf / 4 / kLeafThreads;  // 16 float4 per thread
        float4 v[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int idx = tid + q * kLeafThreads;
            const int r = idx / (kLeaf / 4), c = 4 * (idx % (kLeaf / 4));
            v[q] = (c <= r) ? *reinterpret_cast<const float4*>(A.a + (size_t)r * A.ld + c)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int idx = tid + q * kLeafThreads;
            const int r = idx / (kLeaf / 4), c = 4 * (idx % (kLeaf / 4));
            float* dst = Ls + r * kLeafPitch + c;
            dst[0] = c <= r ? v[q].x : 0.f;
            dst[1] = c + 1 <= r ? v[q].y : 0.f;
            dst[2] = c + 2 <= r ? v[q].z : 0.f;
            dst[3] = c + 3 <= r ? v[q].w : 0.f;
            float* xz = Xs + r * kLeafPitch + c;
            xz[0] = xz[1] = xz[2] = xz[3] = 0.f;
        }
    } else {
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
    }
    __syncthreads();

    // ---- blocked right-looking Cholesky, 32-wide panels
    for (int p = 0; p < 4; ++p) {
        const int c0 = 32 * p;
        if (warp == 0) panel_chol_inv32(Ls, Xs, rdiag, c0, A.col0, n, bad);
        __syncthreads();
        if (p == 3) break;
        // panel solve  L[i, p] = A[i, p] Linv_pp^T  (in place; a warp owns a row
        // and reads all of it before writing it)
        for (int i = c0 + 32 + warp; i < kLeaf; i += kLeafWarps) {
            float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
            for (int k = 0; k < 32; k += 2) {
                s0 = fmaf(Ls[i * kLeafPitch + c0 + k], Xs[(c0 + lane) * kLeafPitch + c0 + k], s0);
                s1 = fmaf(Ls[i * kLeafPitch + c0 + k + 1], Xs[(c0 + lane) * kLeafPitch + c0 + k + 1], s1);
            }
            __syncwarp();
            Ls[i * kLeafPitch + c0 + lane] = s0 + s1;
        }
        __syncthreads();
        // trailing update  A[i, j] -= L[i, p] L[j, p]^T   (lower part)
        const int m = kLeaf - c0 - 32;
        const float* lp = Ls + (c0 + 32) * kLeafPitch + c0;
        leaf_mm(lp, kLeafPitch, 1, lp, 1, kLeafPitch, Ls + (c0 + 32) * kLeafPitch + c0 + 32, m, m, 32,
                -1.0f, true, true, tid, kLeafThreads);
        __syncthreads();
    }

    // ---- off-diagonal 32-blocks of L^-1, by block diagonal:
    //   X[bi,bj] = -Linv_bi * ( sum_{k=bj}^{bi-1} L[bi,k] X[k,bj] )
    // The temporary sum T(bi,bj) is staged in the (unused) upper block (bj,bi) of Ls.
    for (int dgap = 1; dgap < 4; ++dgap) {
        const int pairs = 4 - dgap;
        // one 64-thread group per block pair (64 micro-tiles of 4x4 each)
        const int q = tid / 64, qt = tid % 64;
        const int bj = q, bi = q + dgap;
        if (q < pairs)  // T = L[bi, bj..bi-1] * X[bj..bi-1, bj]
            leaf_mm(Ls + (32 * bi) * kLeafPitch + 32 * bj, kLeafPitch, 1,
                    Xs + (32 * bj) * kLeafPitch + 32 * bj, kLeafPitch, 1,
                    Ls + (32 * bj) * kLeafPitch + 32 * bi, 32, 32, 32 * dgap, 1.0f, false, false,
                    qt, 64);
        __syncthreads();
        if (q < pairs)  // X[bi, bj] = -Linv_bi T
            leaf_mm(Xs + (32 * bi) * kLeafPitch + 32 * bi, kLeafPitch, 1,
                    Ls + (32 * bj) * kLeafPitch + 32 * bi, kLeafPitch, 1,
                    Xs + (32 * bi) * kLeafPitch + 32 * bj, 32, 32, 32, -1.0f, false, false, qt, 64);
        __syncthreads();
    }

    // ---- store X (lower, zeros above) and X^T (upper, zeros below)
    if (vec && (reinterpret_cast<uintptr_t>(A.x) & 15) == 0 && (reinterpret_cast<uintptr_t>(A.xt) & 15) == 0) {
        for (int idx = tid; idx < kLeaf * kLeaf / 4; idx += kLeafThreads) {
            const int r = idx / (kLeaf / 4), c = 4 * (idx % (kLeaf / 4));
            float4 lo, up;
            lo.x = c <= r ? Xs[r * kLeafPitch + c] : 0.f;
            lo.y = c + 1 <= r ? Xs[r * kLeafPitch + c + 1] : 0.f;
            lo.z = c + 2 <= r ? Xs[r * kLeafPitch + c + 2] : 0.f;
            lo.w = c + 3 <= r ? Xs[r * kLeafPitch + c + 3] : 0.f;
            up.x = r <= c ? Xs[c * kLeafPitch + r] : 0.f;
            up.y = r <= c + 1 ? Xs[(c + 1) * kLeafPitch + r] : 0.f;
            up.z = r <= c + 2 ? Xs[(c + 2) * kLeafPitch + r] : 0.f;
            up.w = r <= c + 3 ? Xs[(c + 3) * kLeafPitch + r] : 0.f;
            *reinterpret_cast<float4*>(A.x + (size_t)r * A.ld + c) = lo;
            *reinterpret_cast<float4*>(A.xt + (size_t)r * A.ld + c) = up;
        }
    } else {
        for (int idx = tid; idx < n * n; idx += kLeafThreads) {
            const int r = idx / n, c = idx % n;
            A.x[(size_t)r * A.ld + c] = (c <= r) ? Xs[r * kLeafPitch + c] : 0.0f;
            A.xt[(size_t)r * A.ld + c] = (r <= c) ? Xs[c * kLeafPitch + r] : 0.0f;
        }
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
