// Diagonal-block kernel of the damped inverse, on the SIMT cores in shared
// memory (fp32, like LAPACK's SPOTRF/STRTRI block steps):
//
//   leaf_chol_inv_kernel   one 128x128 block A_kk (already holding every
//                          trailing update):  L = chol(A_kk),  X = L^-1;
//                          writes X (lower, zeros above) and X^T (upper).
//
// Follows the reference arithmetic (proj/src/kfac/matrix.cpp:117-153):
// pivot test `!(diag > 0) || !isfinite(diag)` -> 1-based failing column in
// *info; L^-1 by forward substitution.
//
// The leaf sits on the sequential chain of the factorisation (d/128 leaves
// one after another), so it is organised for latency, as a pipeline over four
// 32-wide panels p with three barrier-separated phases each:
//   A  warp 0: Cholesky of the 32x32 diagonal block in registers (lane i owns
//      row i, fully unrolled, the pivot chain runs through a separate
//      diagonal register so it never waits on the row-update shuffles);
//      warps 1-7 meanwhile finish the previous panel's trailing update and
//      compute T_p = L[p, 0:p] X[0:p, 0:p] (block-row forward substitution);
//   B  panel solve (TRSM), one thread per row below the panel, reading the
//      transposed diagonal block with float4 broadcasts; the last warp
//      inverts the diagonal block (X_pp) concurrently;
//   C  trailing update of the NEXT panel's block column only (all that the
//      next Cholesky needs) and X[p, 0:p] = -X_pp T_p.
// All products are 4x4 register tiles fed by float4 shared-memory reads of
// k-major copies (PT_p = panel transposed, LB / XTd = diagonal blocks
// transposed), skipping the structurally-zero triangles.
#pragma once

#include <cfloat>
#include <climits>
#include <cstdint>
#include <utility>

#include "ptx.cuh"

namespace pf {

#ifdef PF_LEAF_PROBE
__device__ long long* g_probe;
#define PF_STAMP(i)                                                      \
    do {                                                                 \
        __syncthreads();                                                 \
        if (threadIdx.x == 0 && blockIdx.x == 0) g_probe[i] = clock64(); \
    } while (0)
// no barrier: the calling thread's own progress (tid = thread that stamps)
#define PF_STAMP_T(i, tid)                                                  \
    do {                                                                    \
        if (threadIdx.x == (tid) && blockIdx.x == 0) g_probe[i] = clock64(); \
    } while (0)
#else
#define PF_STAMP(i) \
    do {            \
    } while (0)
#define PF_STAMP_T(i, tid) \
    do {                   \
    } while (0)
#endif

#ifdef PF_LEAF_RING
// in-situ probe (-DPF_LEAF_RING): CTA 0 of every leaf launch records
// {globaltimer at entry, after griddepcontrol.wait, after the load, at the
// end; clock64 at entry and end} into a 64-entry ring
__device__ long long g_leaf_ring[64 * 8];
__device__ int g_leaf_ring_n;
__device__ __forceinline__ long long leaf_gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

constexpr int kLeaf = 128;
constexpr int kLeafThreads = 256;
constexpr int kLeafWarps = kLeafThreads / 32;
constexpr int kMaxLeafBatch = 32;
// shared-memory layout (floats; every array 16-byte aligned)
constexpr int kLeafPitch = 129;   // Ls: active trailing matrix (column walks conflict-free)
constexpr int kXPitch = 132;      // Xs, PT: float4 rows
constexpr int kSmallPitch = 36;   // LB (shifted columns of L_pp), XTd (X_pp transposed)
// Tb: T_1, T_2, T_3 (32 x 32bi, pitch 32bi + 4), accumulated panel by panel
__host__ __device__ constexpr int t_pitch(int bi) { return 32 * bi + 4; }
__host__ __device__ constexpr int t_offset(int bi) { return bi == 1 ? 0 : bi == 2 ? 32 * t_pitch(1) : 32 * (t_pitch(1) + t_pitch(2)); }
constexpr int kLsFloats = kLeaf * kLeafPitch + 4 - (kLeaf * kLeafPitch) % 4;
constexpr int kXsFloats = kLeaf * kXPitch;
constexpr int kPTFloats = 32 * kXPitch;
constexpr int kSmallFloats = 32 * kSmallPitch;
constexpr int kTbFloats = 32 * (t_pitch(1) + t_pitch(2) + t_pitch(3));
constexpr int kLeafSmemFloats =
    kLsFloats + kXsFloats + 3 * kPTFloats + 2 * kSmallFloats + kTbFloats + 64 + kLeaf + 4;
constexpr int kLeafSmemBytes = kLeafSmemFloats * 4;

struct LeafArgs {
    const float* a;
    float* x;
    float* xt;
    int* info;
    int ld;    // shared leading dimension of a / x / xt
    int n;     // block size (<= 128; the tail block of a non-multiple-of-128 d)
    int col0;  // global column of the block (for info)
    float* l = nullptr;  // optional: the block's Cholesky factor L_kk (lower part only; pf_cholesky_factor)
    int ldl = 0;
    // optional: published (set to 1, release) once X is in global memory, before
    // X^T is stored; reset at the start.  The slice of X_kk on the right-looking
    // chain waits on it instead of on this launch's completion.
    int* ready = nullptr;
};

struct LeafBatch {
    LeafArgs e[kMaxLeafBatch];
};

// acc[u][q] += sum_{k0 <= k < k1} a4(k)[u] * b4(k)[q], a4(k) / b4(k) the
// float4 at a + k*as / b + k*bs (k ascending, as in the reference loops).
__device__ __forceinline__ void outer4(float (&acc)[4][4], const float* a, int as, const float* b,
                                       int bs, int k0, int k1) {
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
        const float4 av = *reinterpret_cast<const float4*>(a + k * as);
        const float4 bv = *reinterpret_cast<const float4*>(b + k * bs);
        const float ar[4] = {av.x, av.y, av.z, av.w};
        const float br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[u][q] = fmaf(ar[u], br[q], acc[u][q]);
    }
}

__device__ __forceinline__ void zero4x4(float (&acc)[4][4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[u][q] = 0.0f;
}

// t -> (i, j) with i >= j, t = i(i+1)/2 + j
__device__ __forceinline__ void lower_pair(int t, int& i, int& j) {
    int m = static_cast<int>((sqrtf(8.0f * static_cast<float>(t) + 1.0f) - 1.0f) * 0.5f);
    while ((m + 1) * (m + 2) / 2 <= t) ++m;
    while (m * (m + 1) / 2 > t) --m;
    i = m;
    j = t - m * (m + 1) / 2;
}

// ---- phase A, warp 0: Cholesky of the 32x32 diagonal block at (c0, c0) of Ls.
// Lane i owns row i.  The three 32-step loops of the leaf (chol32, trsm_row,
// inv32) are ROLLED: the leaf's code must stay inside the SM's 32 KB L1.5
// instruction cache (fully unrolled the leaf was 126 KB of SASS and ran 30 %
// slower in cycles whenever a concurrent GEMM loaded L2, instruction fetch
// from L2 being on its critical path).  Rolling keeps every register index
// static by ROTATING the row: at pivot k, a[0] holds column k and the update
// of column k + m writes a[m - 1], so the array shifts by one per step at no
// extra cost (the FMA's destination is the shifted slot).  The arithmetic is
// the reference order, operation for operation: a[j] -= l_i l_j per pivot,
// pivots by rsqrt (the unrolled form produced the same bits).
//
// Writes LB[k][m] = L[k + 1 + m][k] (column k below the diagonal, shifted to
// start at m = 0, zero-padded to 32: aligned float4 rows for the TRSM and the
// inverse), rdiag[c0 + k] = 1 / L[k][k] and, kWithL, ldiag[k] = L[k][k].
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Steps per rolled loop of chol32 / trsm_row / inv32 (the width shrinks by
// kPhase from one loop to the next).
#ifndef PF_LEAF_PHASE
#define PF_LEAF_PHASE 8
#endif
constexpr int kPhase = PF_LEAF_PHASE;
#ifndef PF_LEAF_UNROLL
#define PF_LEAF_UNROLL 2
#endif
constexpr int kLeafUnroll = PF_LEAF_UNROLL;

// First W floats of an LB row (aligned float4 loads).
template <int W>
__device__ __forceinline__ void lb_load(const float* lb, float4 (&v)[W / 4]) {
#pragma unroll
    for (int q = 0; q < W / 4; ++q) v[q] = *reinterpret_cast<const float4*>(lb + 4 * q);
}

// One rotated elimination step on an array of width W:
// a[m] = a[m + 1] + s * lv[m] for m < W - 1 (lv = the first W floats of an LB row).
template <int W>
__device__ __forceinline__ void rot_step(float (&a)[32], float s, const float4 (&v)[W / 4]) {
#pragma unroll
    for (int q = 0; q < W / 4; ++q) {
        const float lv[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (4 * q + e < W - 1) a[4 * q + e] = fmaf(s, lv[e], a[4 * q + e + 1]);
    }
}

// The 32 steps of each loop run as 32 / kPhase rolled loops of kPhase steps
// over a shrinking width (32, 28, ..., 4): after step k only 32 - k - 1
// entries are live, so each loop touches at most kPhase - 1 dead ones (544
// FMAs per row for kPhase = 4, against 496 unrolled or 992 fully rolled) and
// the code stays a few short loop bodies.
//
// chol32: the pivot chain is software-pipelined across iterations -- the
// next pivot (shuffle of the updated diagonal + rsqrt) is issued as soon as
// this pivot's l is known, and the next column's value reaches a[0] through
// one shuffle instead of the shared-memory round trip the rest of the row
// update takes.  Same operations in the same order as the plain loop.
template <bool kWithL, int W>
__device__ __forceinline__ void chol32_steps(float (&a)[32], float& dii, float& piv, float& rl, float& mypiv,
                                             int k0, float* LB, float* rdiag, float* ldiag, int c0) {
    const int lane = threadIdx.x & 31;
#pragma unroll(kLeafUnroll)
    for (int k = k0; k < k0 + kPhase; ++k) {
        const float l = lane > k ? a[0] * rl : (lane == k ? piv * rl : 0.0f);
        dii = fmaf(-l, l, dii);
        // lanes > k publish their l at lane - k - 1; lanes <= k zero the tail
        // of the row (index 31 - k + lane: the same expression mod 32)
        LB[k * kSmallPitch + ((lane - k - 1) & 31)] = lane > k ? l : 0.0f;
        // the next pivot: lane k + 1's diagonal is final once its l is known
        const float piv_n = __shfl_sync(0xffffffffu, dii, (k + 1) & 31);
        const float l_k1 = __shfl_sync(0xffffffffu, l, (k + 1) & 31);  // L[k + 1][k] = LB[k][0]
        if (lane == k) {
            mypiv = piv;  // checked after the loop
            rdiag[c0 + k] = rl;
            if (kWithL) ldiag[k] = l;
        }
        const float rl_n = rsqrt_ftz(piv_n);
        const float a0 = fmaf(-l, l_k1, a[1]);
        __syncwarp();
        float4 v[W / 4];
        lb_load<W>(LB + k * kSmallPitch, v);
        rot_step<W>(a, -l, v);
        a[0] = a0;
        piv = piv_n;
        rl = rl_n;
    }
}

template <bool kWithL>
__device__ __forceinline__ void chol32(const float* Ls, float* LB, float* rdiag, float* ldiag, int c0, int n,
                                       int col_base, int* bad) {
    const int lane = threadIdx.x & 31;
    const float* row = Ls + (c0 + lane) * kLeafPitch + c0;
    float a[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = row[j];
    float dii = row[lane];  // == a[lane], kept apart so the pivot chain is short
    float piv = __shfl_sync(0xffffffffu, dii, 0);  // warp-uniform
    float rl = rsqrt_ftz(piv);
    float mypiv = 1.0f;
    [&]<int... P>(std::integer_sequence<int, P...>) {
        (chol32_steps<kWithL, 32 - kPhase * P>(a, dii, piv, rl, mypiv, kPhase * P, LB, rdiag, ldiag, c0), ...);
    }(std::make_integer_sequence<int, 32 / kPhase>{});
    // a failed pivot (<= 0, inf, NaN) propagated NaN / inf through the block;
    // the first one (1-based column) goes to *bad, the caller raises on it
    const unsigned failed = __ballot_sync(0xffffffffu, !(mypiv > 0.0f && mypiv <= FLT_MAX) && c0 + lane < n);
    if (lane == 0 && failed) *bad = min(*bad, col_base + c0 + __ffs(failed));
}

// ---- phase B: row r of the panel solve  L[r, p] = A[r, p] L_pp^-T  by
// forward substitution (x_j final -> eliminate it from the later entries;
// reference matrix.cpp order), result stored transposed: PTp[k][r].  Rotated
// like chol32; the next step's LB row and 1/L_jj are loaded one step ahead.
template <int W>
__device__ __forceinline__ void trsm_steps(float (&x)[32], int j0, const float* LB, const float* rdiag,
                                           float* PTp, int c0, int r) {
    float4 nv[W / 4];
    lb_load<W>(LB + j0 * kSmallPitch, nv);
    float rd_n = rdiag[c0 + j0];
#pragma unroll(kLeafUnroll)
    for (int j = j0; j < j0 + kPhase; ++j) {
        float4 v[W / 4];
#pragma unroll
        for (int q = 0; q < W / 4; ++q) v[q] = nv[q];
        const float rd = rd_n;
        if (j + 1 < j0 + kPhase) {
            lb_load<W>(LB + (j + 1) * kSmallPitch, nv);
            rd_n = rdiag[c0 + j + 1];
        }
        const float xj = x[0] * rd;
        PTp[j * kXPitch + r] = xj;
        rot_step<W>(x, -xj, v);
    }
}

__device__ __forceinline__ void trsm_row(const float* Ls, const float* LB, const float* rdiag, float* PTp,
                                         int c0, int r) {
    const float* row = Ls + r * kLeafPitch + c0;
    float x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = row[j];
    [&]<int... P>(std::integer_sequence<int, P...>) {
        (trsm_steps<32 - kPhase * P>(x, kPhase * P, LB, rdiag, PTp, c0, r), ...);
    }(std::make_integer_sequence<int, 32 / kPhase>{});
}

// ---- phase B, one warp: X_pp = L_pp^-1 (lane c computes column c, reference
// matrix.cpp:145-153); into Xs (zeros above the diagonal) and XTd[c][i] = X[i][c].
template <int W>
__device__ __forceinline__ void inv32_steps(float (&x)[32], int i0, const float* LB, const float* rdiag,
                                            float* Xs, float* XTd, int c0) {
    const int lane = threadIdx.x & 31;
    float4 nv[W / 4];
    lb_load<W>(LB + i0 * kSmallPitch, nv);
    float rd_n = rdiag[c0 + i0];
#pragma unroll(kLeafUnroll)
    for (int i = i0; i < i0 + kPhase; ++i) {
        float4 v[W / 4];
#pragma unroll
        for (int q = 0; q < W / 4; ++q) v[q] = nv[q];
        const float rd = rd_n;
        if (i + 1 < i0 + kPhase) {
            lb_load<W>(LB + (i + 1) * kSmallPitch, nv);
            rd_n = rdiag[c0 + i + 1];
        }
        const float xi = x[0] * rd;
        Xs[(c0 + i) * kXPitch + c0 + lane] = xi;
        XTd[lane * kSmallPitch + i] = xi;
        rot_step<W>(x, -xi, v);  // fmaf(-xi, L, x) == fmaf(-L, xi, x) exactly
    }
}

__device__ __forceinline__ void inv32(const float* LB, const float* rdiag, float* Xs, float* XTd, int c0) {
    const int lane = threadIdx.x & 31;
    float x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? 1.0f : 0.0f;
    [&]<int... P>(std::integer_sequence<int, P...>) {
        (inv32_steps<32 - kPhase * P>(x, kPhase * P, LB, rdiag, Xs, XTd, c0), ...);
    }(std::make_integer_sequence<int, 32 / kPhase>{});
}

// trailing-update tile: Ls[r][c] -= sum_k L[r][k] L[c][k] over panel PTp, for
// the 4x4 tile at (r0, cc), lower part only
__device__ __forceinline__ void trail_tile(float* Ls, const float* PTp, int r0, int cc) {
    float acc[4][4];
    zero4x4(acc);
    outer4(acc, PTp + r0, kXPitch, PTp + cc, kXPitch, 0, 32);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (cc + q <= r0 + u) {
                float* d = Ls + (r0 + u) * kLeafPitch + cc + q;
                *d = fmaf(-1.0f, acc[u][q], *d);
            }
}

// Contribution of panel q to T_bi (bi > q), tile (ti in [0,8), tj in [0, 8(q+1))):
//   T_bi[i][j] += sum_{k in panel q, k >= 4tj} L[32bi+i][k] X[k][j]
// The first panel that reaches column j initialises the tile; later panels
// continue the same fmaf chain (k ascending), so the result is bit-identical
// to one pass over k in [4tj, 32bi).
__device__ __forceinline__ void tpanel_tile(const float* PT, const float* Xs, float* Tb, int bi, int q, int ti,
                                            int tj) {
    float* T = Tb + t_offset(bi);
    const int tp = t_pitch(bi);
    float acc[4][4];
    const int kstart = 4 * tj;
    if (kstart / 32 == q) {
        zero4x4(acc);
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float4 v = *reinterpret_cast<const float4*>(T + (4 * ti + u) * tp + 4 * tj);
            acc[u][0] = v.x;
            acc[u][1] = v.y;
            acc[u][2] = v.z;
            acc[u][3] = v.w;
        }
    }
    outer4(acc, PT + q * kPTFloats + 32 * bi + 4 * ti, kXPitch, Xs + (32 * q) * kXPitch + 4 * tj, kXPitch,
           max(kstart - 32 * q, 0), 32);
#pragma unroll
    for (int u = 0; u < 4; ++u)
        *reinterpret_cast<float4*>(T + (4 * ti + u) * tp + 4 * tj) = make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
}

// X[32p+i][j] = -sum_{k <= i} X_pp[i][k] T[k][j]  for the 4x4 tile (ti, tj)
__device__ __forceinline__ void xprod_tile(const float* XTd, const float* Tb, float* Xs, int p, int ti, int tj) {
    float acc[4][4];
    zero4x4(acc);
    outer4(acc, XTd + 4 * ti, kSmallPitch, Tb + t_offset(p) + 4 * tj, t_pitch(p), 0, 4 * ti + 4);
#pragma unroll
    for (int u = 0; u < 4; ++u)
        *reinterpret_cast<float4*>(Xs + (32 * p + 4 * ti + u) * kXPitch + 4 * tj) =
            make_float4(-acc[u][0], -acc[u][1], -acc[u][2], -acc[u][3]);
}

// ---- global <-> shared (256 threads)
// dst = lower triangle of the n x n block at src (zeros above, identity beyond n)
__device__ __forceinline__ void load_lower(float* dst, const float* src, int ld, int n) {
    const int tid = threadIdx.x;
    const bool vec = n == kLeaf && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
    if (vec) {
        constexpr int kPer = kLeaf * kLeaf / 4 / kLeafThreads;  // 16 float4 per thread
        float4 v[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int idx = tid + q * kLeafThreads;
            const int r = idx / (kLeaf / 4), c = 4 * (idx % (kLeaf / 4));
            v[q] = (c <= r) ? __ldcg(reinterpret_cast<const float4*>(src + (size_t)r * ld + c))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int idx = tid + q * kLeafThreads;
            const int r = idx / (kLeaf / 4), c = 4 * (idx % (kLeaf / 4));
            float* d = dst + r * kLeafPitch + c;
            d[0] = c <= r ? v[q].x : 0.f;
            d[1] = c + 1 <= r ? v[q].y : 0.f;
            d[2] = c + 2 <= r ? v[q].z : 0.f;
            d[3] = c + 3 <= r ? v[q].w : 0.f;
        }
    } else {
        for (int idx = tid; idx < kLeaf * kLeaf; idx += kLeafThreads) {
            const int r = idx / kLeaf, c = idx % kLeaf;
            float v;
            if (r < n && c < n)
                v = (c <= r) ? __ldcg(src + (size_t)r * ld + c) : 0.0f;
            else
                v = (r == c) ? 1.0f : 0.0f;
            dst[r * kLeafPitch + c] = v;
        }
    }
}

// vectorised full-block load split in two: issue (registers) and commit (smem)
constexpr int kLoadPer = kLeaf * kLeaf / 4 / kLeafThreads;  // 16 float4 per thread
__device__ __forceinline__ void load_lower_issue(const float* src, int ld, float4 (&v)[kLoadPer]) {
#pragma unroll
    for (int q = 0; q < kLoadPer; ++q) {
        const int idx = threadIdx.x + q * kLeafThreads;
        const int r = idx / (kLeaf / 4), c = 4 * (idx % (kLeaf / 4));
        v[q] = (c <= r) ? __ldcg(reinterpret_cast<const float4*>(src + (size_t)r * ld + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}
__device__ __forceinline__ void load_lower_commit(float* dst, const float4 (&v)[kLoadPer]) {
#pragma unroll
    for (int q = 0; q < kLoadPer; ++q) {
        const int idx = threadIdx.x + q * kLeafThreads;
        const int r = idx / (kLeaf / 4), c = 4 * (idx % (kLeaf / 4));
        float* d = dst + r * kLeafPitch + c;
        d[0] = c <= r ? v[q].x : 0.f;
        d[1] = c + 1 <= r ? v[q].y : 0.f;
        d[2] = c + 2 <= r ? v[q].z : 0.f;
        d[3] = c + 3 <= r ? v[q].w : 0.f;
    }
}

// zero the strictly-upper 32x32 blocks of Xs (never written otherwise)
__device__ __forceinline__ void zero_upper_blocks(float* Xs) {
    for (int idx = threadIdx.x; idx < kLeaf * kLeaf / 4; idx += kLeafThreads) {
        const int r = idx / (kLeaf / 4), c = 4 * (idx % (kLeaf / 4));
        if (c >= 32 * (r / 32 + 1))
            *reinterpret_cast<float4*>(Xs + r * kXPitch + c) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// x = X (lower, zeros above) and xt = X^T for the n x n block
// `tbuf` (pitch kLeafPitch, 128 rows) is scratch: the active-matrix buffer,
// free once the factorisation is done.  Every thread must call this.
__device__ __forceinline__ void store_x(const float* Xs, float* tbuf, float* x, float* xt, int ld, int n,
                                        int* ready = nullptr) {
    const int tid = threadIdx.x;
    auto publish = [&] {  // every thread's X stores, then one release of the flag
        if (!ready) return;
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicExch(ready, 1);
        }
    };
    const bool vec = n == kLeaf && (ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(xt) & 15) == 0);
    if (vec) {
        // shared-memory reads of a batch first, then its global stores
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            float4 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = tid + (8 * b + q) * kLeafThreads;
                const int r = idx / (kLeaf / 4), c = 4 * (idx % (kLeaf / 4));
                v[q] = *reinterpret_cast<const float4*>(Xs + r * kXPitch + c);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = tid + (8 * b + q) * kLeafThreads;
                const int r = idx / (kLeaf / 4), c = 4 * (idx % (kLeaf / 4));
                *reinterpret_cast<float4*>(x + (size_t)r * ld + c) = v[q];
            }
        }
        publish();
        // X^T: transpose into the (now free) pitch-129 buffer, then store its rows
        for (int idx = tid; idx < kLeaf * kLeaf; idx += kLeafThreads) {
            const int r = idx / kLeaf, c = idx % kLeaf;  // lanes: consecutive c
            tbuf[c * kLeafPitch + r] = Xs[r * kXPitch + c];
        }
        __syncthreads();
#pragma unroll 4
        for (int idx = tid; idx < kLeaf * kLeaf; idx += kLeafThreads) {
            const int r = idx / kLeaf, c = idx % kLeaf;
            xt[(size_t)r * ld + c] = tbuf[r * kLeafPitch + c];
        }
    } else {
        for (int idx = tid; idx < n * n; idx += kLeafThreads) {
            const int r = idx / n, c = idx % n;
            x[(size_t)r * ld + c] = Xs[r * kXPitch + c];
            xt[(size_t)r * ld + c] = Xs[c * kXPitch + r];
        }
        publish();
    }
}

__device__ __forceinline__ void report_bad(int* info, int bad) {
    if (bad == INT_MAX) return;
    // keep the smallest failing column across blocks (0 = success)
    int old = *info;
    while (old == 0 || bad < old) {
        const int seen = atomicCAS(info, old, bad);
        if (seen == old) break;
        old = seen;
    }
}

// pf_cholesky_factor: the 32x32 diagonal block c0 of L from LB / ldiag
// (L[i][j] = LB[j][i - j - 1] below the diagonal, ldiag[j] on it)
__device__ __forceinline__ void store_l_diag(const float* LB, const float* ldiag, const LeafArgs& A, int c0) {
    for (int idx = threadIdx.x; idx < 32 * 32; idx += kLeafThreads) {
        const int i = idx >> 5, j = idx & 31;
        if (j <= i && c0 + i < A.n)
            A.l[static_cast<size_t>(c0 + i) * A.ldl + c0 + j] = i == j ? ldiag[j] : LB[j * kSmallPitch + i - j - 1];
    }
}
// ... and the panels below the diagonal blocks, PT_p[k][r] = L[r][32p + k]
__device__ __forceinline__ void store_l_panels(const float* PT, const LeafArgs& A) {
    for (int p = 0; p < 3; ++p)
        for (int idx = threadIdx.x; idx < 32 * kLeaf; idx += kLeafThreads) {
            const int r = idx >> 5, k = idx & 31;
            if (r >= 32 * (p + 1) && r < A.n)
                A.l[static_cast<size_t>(r) * A.ldl + 32 * p + k] = PT[p * kPTFloats + k * kXPitch + r];
        }
}

// Helper warps of a phase: warps in [first, last] whose scheduler (warp % 4)
// is not in `sched_mask`, so the critical warps keep their issue slots.
// Returns the warp's rank among them and their count.
__device__ __forceinline__ bool helper_warp(int warp, unsigned sched_mask) {
    return !((sched_mask >> (warp & 3)) & 1u);
}
__device__ __forceinline__ int helper_rank(int warp, unsigned sched_mask, int& count, int first, int last) {
    int rank = 0;
    count = 0;
#pragma unroll
    for (int w = 0; w < kLeafWarps; ++w) {
        if (w > last) break;
        const bool ok = w >= first && helper_warp(w, sched_mask);
        if (ok && w < warp) ++rank;
        count += ok ? 1 : 0;
    }
    return rank;
}

// The whole leaf for one block, 256 threads, `leaf_smem` = kLeafSmemBytes of
// 16-byte aligned shared memory.  `pdl`: called from a PDL-launched kernel.
template <bool kWithL>
__device__ __forceinline__ void leaf_body(const LeafArgs& A, float* leaf_smem, bool pdl) {
    float* Ls = leaf_smem;
    float* Xs = Ls + kLsFloats;
    float* PT = Xs + kXsFloats;  // panels 0..2, transposed
    float* LB = PT + 3 * kPTFloats;  // chol32's shifted columns of L_pp
    float* XTd = LB + kSmallFloats;
    float* Tb = XTd + kSmallFloats;
    float* ldiag = Tb + kTbFloats;  // kWithL: the diagonal of L_pp (64 floats reserved)
    float* rdiag = ldiag + 64;
    int* bad = reinterpret_cast<int*>(rdiag + kLeaf);
    const int tid = threadIdx.x;
    const int warp = tid >> 5;

    PF_STAMP(0);
#ifdef PF_LEAF_RING
    long long r_t0 = leaf_gtimer(), r_c0 = clock64(), r_t1 = 0, r_t2 = 0;
#endif
    if (tid == 0) {
        *bad = INT_MAX;
        if (A.ready) atomicExch(A.ready, 0);  // performed at L2 before any reader can start (below)
    }
    if (pdl) ptx::grid_dep_wait();  // PDL: A is produced by the previous launch
#ifdef PF_LEAF_RING
    r_t1 = leaf_gtimer();
#endif
    const bool vec = A.n == kLeaf && (A.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(A.a) & 15) == 0);
    if (vec) {
        float4 v[kLoadPer];
        load_lower_issue(A.a, A.ld, v);  // global loads in flight ...
        zero_upper_blocks(Xs);           // ... while the upper blocks of X are cleared
        load_lower_commit(Ls, v);
    } else {
        zero_upper_blocks(Xs);
        load_lower(Ls, A.a, A.ld, A.n);
    }
    __syncthreads();
    PF_STAMP(2);
#ifdef PF_LEAF_RING
    r_t2 = leaf_gtimer();
#endif

#pragma unroll 1
    for (int p = 0; p < 4; ++p) {
        const int c0 = 32 * p;
        // ---- A: chol(p) || rest of U(p-1) + T_p
        if (warp == 0) {
            chol32<kWithL>(Ls, LB, rdiag, ldiag, c0, A.n, A.col0, bad);
            PF_STAMP_T(20 + p, 0);
        } else if (p > 0 && helper_warp(warp, 1u)) {
            // rest of U(p-1) + panel p-1's contribution to T_p (the later T_bi
            // get theirs on the idle warps of phase B), on the warps that do
            // not share warp 0's scheduler (warp w issues on scheduler w % 4)
            const int base = 8 * (p + 1), m = 32 - base;  // tile rows/cols [base, 32), lower
            const int nrest = m * (m + 1) / 2;
            const int per = 64 * p;                       // tiles of one T_bi slice (8 x 8p)
            int nh;
            const int h = helper_rank(warp, 1u, nh, 1, kLeafWarps - 1);
            for (int t = h * 32 + (tid & 31); t < nrest + per; t += nh * 32) {
                if (t < nrest) {
                    int i, j;
                    lower_pair(t, i, j);
                    trail_tile(Ls, PT + (p - 1) * kPTFloats, 4 * (base + i), 4 * (base + j));
                } else {
                    const int v = t - nrest;
                    tpanel_tile(PT, Xs, Tb, p, p - 1, v / (8 * p), v % (8 * p));
                }
            }
            PF_STAMP_T(24 + p, 32);
        }
        __syncthreads();
        PF_STAMP(3 + 3 * p);
        if constexpr (kWithL) store_l_diag(LB, ldiag, A, c0);  // LB stays untouched until the next phase A
        if (p == 3) break;
        // ---- B: TRSM of the rows below || X_pp
        const int below = kLeaf - c0 - 32;
        if (tid < below) {
            trsm_row(Ls, LB, rdiag, PT + p * kPTFloats, c0, c0 + 32 + tid);
        } else if (warp == kLeafWarps - 1) {
            inv32(LB, rdiag, Xs, XTd, c0);
        } else if (p > 0) {  // warps between: panel p-1's contribution to T_{p+1} .. T_3
            // (keeping them off the schedulers of the TRSM / X_pp warps was
            // measured slower: too few warps left for this work at p = 1)
            const int first = (below + 31) / 32 * 32;  // first thread of the free warps
            const int per = 64 * p, n = per * (3 - p);
            for (int t = tid - first; t >= 0 && t < n; t += (kLeafWarps - 1) * 32 - first) {
                const int bi = p + 1 + t / per, v = t % per;
                tpanel_tile(PT, Xs, Tb, bi, p - 1, v / (8 * p), v % (8 * p));
            }
        }
        __syncthreads();
        PF_STAMP(4 + 3 * p);
        // ---- C: U(p) on block column p+1 || X[p, 0:p] = -X_pp T_p
        {
            const int base = 8 * (p + 1), rows = 32 - base;
            const int nu = rows * 8, nx = 64 * p;
            for (int t = tid; t < nu + nx; t += kLeafThreads) {
                if (t < nu) {
                    const int tr = base + t / 8, tc = base + t % 8;
                    if (tc <= tr) trail_tile(Ls, PT + p * kPTFloats, 4 * tr, 4 * tc);
                } else {
                    const int u = t - nu;
                    xprod_tile(XTd, Tb, Xs, p, u / (8 * p), u % (8 * p));
                }
            }
        }
        __syncthreads();
        PF_STAMP(5 + 3 * p);
    }
    // ---- tail: X_33, then X[3, 0:3] = -X_33 T_3
    if (warp == 0) inv32(LB, rdiag, Xs, XTd, 96);
    __syncthreads();
    PF_STAMP(13);
    for (int t = tid; t < 192; t += kLeafThreads) xprod_tile(XTd, Tb, Xs, 3, t / 24, t % 24);
    __syncthreads();
    PF_STAMP(14);
    if constexpr (kWithL) store_l_panels(PT, A);
#ifdef PF_LEAF_RING
    const long long r_t3 = leaf_gtimer();
#endif
    if (pdl) ptx::grid_dep_launch();
    store_x(Xs, Ls, A.x, A.xt, A.ld, A.n, A.ready);
    PF_STAMP(19);
#ifdef PF_LEAF_RING
    __syncthreads();
    if (tid == 0 && blockIdx.x == 0) {
        const int i = atomicAdd(&g_leaf_ring_n, 1) & 63;
        long long* rec = g_leaf_ring + 8 * i;
        rec[0] = r_t0; rec[1] = r_t1; rec[2] = r_t2; rec[3] = leaf_gtimer();
        rec[4] = r_c0; rec[5] = clock64(); rec[6] = r_t3; rec[7] = A.col0;
    }
#endif
    if (tid == 0) report_bad(A.info, *bad);
}

// kWithL: the leaves of pf_cholesky_factor also write their block of L (a
// separate instantiation, so the inverse's leaf keeps its register budget)
template <bool kWithL>
__global__ void __launch_bounds__(kLeafThreads, 1) leaf_chol_inv_kernel(const __grid_constant__ LeafBatch batch) {
    extern __shared__ __align__(16) float leaf_smem[];
    leaf_body<kWithL>(batch.e[blockIdx.x], leaf_smem, true);
}

}  // namespace pf
