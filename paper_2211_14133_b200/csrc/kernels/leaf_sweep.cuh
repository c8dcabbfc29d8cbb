// Diagonal-block kernel of the damped inverse, single-sweep form:
//
//   leaf_sweep_kernel   one 128x128 block A_kk (already holding every trailing
//                       update):  L = chol(A_kk),  X = L^-1;  writes X (lower,
//                       zeros above) and X^T (upper) -- the same contract as
//                       leaf_chol_inv_kernel (leaf.cuh), which it replaces on
//                       the critical chain.
//
// Arithmetic (reference proj/src/kfac/matrix.cpp:117-153): right-looking
// Cholesky with the forward substitution for L^-1 carried along, one pivot j
// at a time:
//     v_j    = rl_j = 1/sqrt(c_jj)                      (= x_jj)
//     v_i    = l_ij = c_ij rl_j                 i > j   (column j of L)
//     c_ik  -= v_i v_k                          j < k <= i   (trailing update)
//     x_jr   = b_jr rl_j,  b_ir -= v_i x_jr     r < j < i    (forward subst.)
// where B starts as I, so column j of B is born as b_ij = -v_i rl_j, and row j
// of B scaled by rl_j is row j of X = L^-1.  Pivot test as the reference
// (`!(diag > 0) || !isfinite`), 1-based failing column into *info.
//
// Layout (256 threads, 2 per row, 64 registers each): thread (r, q) holds
//   * while r > j: the A-part of row r, columns k = 2m+q (k <= r), and
//   * once r <= j: column r of B, rows i = 2m+q (i > j),
// so one register array and one FMA loop serve both parts -- every thread does
// c[m] -= mult * v[2m+q] with mult = v_r (A-part) or x_jr (B-part), the same
// v vector, read as float4 from shared memory.  The two ranges never overlap
// (k <= r < i), so turning row j into column j of B only has to clear the
// few slots the warp-wide loop bound scribbled on.  Every 16 pivots the array
// rotates down by 8 slots (indices <= j are dead for both parts), so inside
// the 16-pivot unrolled body every register index is static; v is stored
// rotated the same way.  Warps are paired on a scheduler short-row with
// long-row (virtual warp 7 - s beside s) to balance the triangle.
//
// One barrier per pivot: during phase j every thread applies pivot j, and the
// owners of column j+1 (and of the diagonal c_{j+1,j+1}, kept one step ahead
// in `dg`) FIRST form v^(j+1) -- the only values the next phase waits for.
// The X rows leave through a shared-memory staging array, stored coalesced
// (X and X^T) at the end.
#pragma once

#include <cfloat>
#include <climits>
#include <cstdint>

#include "leaf.cuh"

namespace pf {

constexpr int kSweepThreads = 256;
constexpr int kVsPitch = 68;  // per-q row of a v buffer: 64 slots, float4-aligned, banks skewed by 4
constexpr int kXsPitch = 129; // X staging: row and column walks conflict-free
constexpr int kSweepVsFloats = 2 * 2 * kVsPitch;
constexpr int kSweepSmemFloats = kSweepVsFloats + kLeaf + kLeaf * kXsPitch + 4;
constexpr int kSweepSmemBytes = kSweepSmemFloats * 4;

// 1/sqrt(p) to ~0.5 ulp: hardware estimate plus one Newton step
__device__ __forceinline__ float rsqrt_nr(float p) {
    const float y = rsqrtf(p);
    const float h = 0.5f * p * y;
    return fmaf(fmaf(-h, y, 0.5f), y, y);
}

// Per-thread constants of the sweep (hoisted out of the phases).
struct SweepThread {
    int row, q, lane, vw;
    int arow_off;  // float offset of v_row's per-q row: (row & 1) * kVsPitch + (row >> 1)
};

// Phase j = 16 it + R.  `vb`: v^(j), `vn`: v^(j+1), both stored with slot
// m <-> index 2(base + m) + q (base = 8 it; 8 (it + 1) for vn when R = 15).
// `ng`: groups of 8 slots the warp updates this iteration (warp-uniform).
// The critical section is branch-free (every thread computes, owners store)
// so the compiler can interleave its latency chain with the bulk FMAs.
template <int R>
__device__ __forceinline__ void sweep_phase(float (&c)[64], const int it, const SweepThread& t, const int ng,
                                            const float* __restrict__ vb, float* __restrict__ vn,
                                            float* __restrict__ dg, float* __restrict__ xs, int& bad, const int n) {
    const int j = 16 * it + R;
    const int base = 8 * it;
    constexpr int kS0 = R >> 1;        // slot of index j (the lowest live index)
    constexpr int kS1 = (R + 1) >> 1;  // slot of index j + 1
    constexpr int kS2 = (R + 2) >> 1;  // slot of index j + 2
    constexpr int kNext = (R == 15) ? 8 : 0;
    constexpr int kQ1 = (R + 1) & 1, kQ0 = R & 1, kQ2 = R & 1;  // (j+1)&1, j&1, (j+2)&1
    const bool isA = t.row > j;
    const float a_row = vb[max(t.arow_off - base, (t.row & 1) * kVsPitch)];  // v_row (A rows)
    // ---- critical: v^(j+1) (column j+1 of L and rl_{j+1}) and dg[j+2]
    if (j + 1 < kLeaf) {
        const float vj1 = vb[kQ1 * kVsPitch + kS1];
        const float p = fmaf(-vj1, vj1, dg[j + 1]);
        const float rl = rsqrt_nr(p);
        const float v = t.row == j + 1 ? rl : fmaf(-a_row, vj1, c[kS1]) * rl;  // == this phase's update, scaled
        const bool own = t.q == kQ1 && isA;
        if (t.row == j + 1 && t.q == kQ1 && !(p > 0.0f && p <= FLT_MAX) && j + 1 < n) bad = min(bad, j + 2);
        if (own) vn[t.arow_off - base - kNext] = v;
        const float d2 = fmaf(-a_row, a_row, c[kS2]);
        if (j + 2 < kLeaf && t.row == j + 2 && t.q == kQ2) dg[j + 2] = d2;
    }
    // ---- row j turns into column j of B: clear what the warp-wide bound
    // wrote above the diagonal (indices j .. 16 vw + 15 = slots kS0 .. 7), b_jj = 1
    if (t.vw == it) {
        if (t.row == j) {
#pragma unroll
            for (int s = kS0; s < 8; ++s) c[s] = 0.0f;
            if (t.q == kQ0) c[kS0] = 1.0f;
        }
    }
    const float rlj = vb[kQ0 * kVsPitch + kS0];                                 // v^(j)_j = rl_j
    const float bj = __shfl_sync(0xffffffffu, c[kS0], (t.lane & ~1) | kQ0);     // b_{j,row}
    const float x = bj * rlj;                                                   // x_{j,row}
    if (!isA && t.q == 0) xs[j * kXsPitch + t.row] = x;
    const float mult = isA ? a_row : x;
    // slots >= 8 in the warp that is converting hold indices past its own rows:
    // only its B columns own them there
    const float mult_hi = (isA && t.vw == it) ? 0.0f : mult;
    // ---- bulk: c[m] -= mult * v[2(base+m)+q] over the warp's live slots
    const float4* v4 = reinterpret_cast<const float4*>(vb + t.q * kVsPitch);
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        if (g > 0 && g >= ng) break;
        const float4 u = v4[2 * g], w = v4[2 * g + 1];
        const float mg = g == 0 ? mult : mult_hi;
        c[8 * g + 0] = fmaf(-mg, u.x, c[8 * g + 0]);
        c[8 * g + 1] = fmaf(-mg, u.y, c[8 * g + 1]);
        c[8 * g + 2] = fmaf(-mg, u.z, c[8 * g + 2]);
        c[8 * g + 3] = fmaf(-mg, u.w, c[8 * g + 3]);
        c[8 * g + 4] = fmaf(-mg, w.x, c[8 * g + 4]);
        c[8 * g + 5] = fmaf(-mg, w.y, c[8 * g + 5]);
        c[8 * g + 6] = fmaf(-mg, w.z, c[8 * g + 6]);
        c[8 * g + 7] = fmaf(-mg, w.w, c[8 * g + 7]);
    }
    __syncthreads();
}

__device__ __forceinline__ void sweep_body(const LeafArgs& A, float* smem, bool pdl) {
    float* vs = smem;                 // [2][2][kVsPitch]
    float* dg = vs + kSweepVsFloats;  // [128]
    float* xs = dg + kLeaf;           // [128][kXsPitch]
    int* badp = reinterpret_cast<int*>(xs + kLeaf * kXsPitch);
    const int tid = threadIdx.x;
    const int lane = tid & 31, w = tid >> 5;
    const int vw = w < 4 ? w : 11 - w;  // scheduler s runs virtual warps s and 7 - s
    const int row = 16 * vw + (lane >> 1), q = lane & 1;
    const SweepThread th{row, q, lane, vw, (row & 1) * kVsPitch + (row >> 1)};
    const int n = A.n;

    if (tid == 0) *badp = INT_MAX;
    for (int i = tid; i < kSweepVsFloats; i += kSweepThreads) vs[i] = 0.0f;
    if (pdl) ptx::grid_dep_wait();  // PDL: A is produced by the previous launch
    float c[64];
    if (n == kLeaf) {
        const float* src = A.a + static_cast<size_t>(row) * A.ld + q;
#pragma unroll
        for (int m = 0; m < 64; ++m) c[m] = (2 * m + q <= row) ? __ldcg(src + 2 * m) : 0.0f;
    } else {
#pragma unroll
        for (int m = 0; m < 64; ++m) {
            const int k = 2 * m + q;
            float v = 0.0f;
            if (row < n && k <= row) v = __ldcg(A.a + static_cast<size_t>(row) * A.ld + k);
            else if (row >= n && k == row) v = 1.0f;
            c[m] = v;
        }
    }
    int bad = INT_MAX;  // 1-based failing column within the block (this thread's pivots)
    // ---- pivot 0 (prologue): v^(0) and dg[1]
    if (row == 0 && q == 0) dg[0] = c[0];
    if (row == 1 && q == 1) dg[1] = c[0];
    __syncthreads();
    if (q == 0) {
        const float p = dg[0];
        const float rl = rsqrt_nr(p);
        if (row == 0 && !(p > 0.0f && p <= FLT_MAX)) bad = 1;
        vs[(row >> 1) + (row & 1) * kVsPitch] = row == 0 ? rl : c[0] * rl;
    }
    __syncthreads();

    float* v0 = vs;
    float* v1 = vs + 2 * kVsPitch;
    for (int it = 0; it < 8; ++it) {
        const int hi = vw > it ? 8 * (vw - it) + 7 : 63 - 8 * it;  // last live slot, warp-uniform
        const int ng = hi / 8 + 1;
        sweep_phase<0>(c, it, th, ng, v0, v1, dg, xs, bad, n);
        sweep_phase<1>(c, it, th, ng, v1, v0, dg, xs, bad, n);
        sweep_phase<2>(c, it, th, ng, v0, v1, dg, xs, bad, n);
        sweep_phase<3>(c, it, th, ng, v1, v0, dg, xs, bad, n);
        sweep_phase<4>(c, it, th, ng, v0, v1, dg, xs, bad, n);
        sweep_phase<5>(c, it, th, ng, v1, v0, dg, xs, bad, n);
        sweep_phase<6>(c, it, th, ng, v0, v1, dg, xs, bad, n);
        sweep_phase<7>(c, it, th, ng, v1, v0, dg, xs, bad, n);
        sweep_phase<8>(c, it, th, ng, v0, v1, dg, xs, bad, n);
        sweep_phase<9>(c, it, th, ng, v1, v0, dg, xs, bad, n);
        sweep_phase<10>(c, it, th, ng, v0, v1, dg, xs, bad, n);
        sweep_phase<11>(c, it, th, ng, v1, v0, dg, xs, bad, n);
        sweep_phase<12>(c, it, th, ng, v0, v1, dg, xs, bad, n);
        sweep_phase<13>(c, it, th, ng, v1, v0, dg, xs, bad, n);
        sweep_phase<14>(c, it, th, ng, v0, v1, dg, xs, bad, n);
        sweep_phase<15>(c, it, th, ng, v1, v0, dg, xs, bad, n);
#pragma unroll
        for (int m = 0; m < 56; ++m) c[m] = c[m + 8];
#pragma unroll
        for (int m = 56; m < 64; ++m) c[m] = 0.0f;
    }
    if (bad != INT_MAX) atomicMin(badp, bad);
    if (pdl) ptx::grid_dep_launch();
    __syncthreads();
    // ---- store X (lower, zeros above) and X^T
    const int ld = A.ld;
    if (n == kLeaf) {
#pragma unroll 8
        for (int idx = tid; idx < kLeaf * kLeaf; idx += kSweepThreads) {
            const int r = idx >> 7, cc = idx & 127;
            A.x[static_cast<size_t>(r) * ld + cc] = cc <= r ? xs[r * kXsPitch + cc] : 0.0f;
        }
#pragma unroll 8
        for (int idx = tid; idx < kLeaf * kLeaf; idx += kSweepThreads) {
            const int r = idx >> 7, cc = idx & 127;  // X^T[r][cc] = X[cc][r]
            A.xt[static_cast<size_t>(r) * ld + cc] = r <= cc ? xs[cc * kXsPitch + r] : 0.0f;
        }
    } else {
        for (int idx = tid; idx < n * n; idx += kSweepThreads) {
            const int r = idx / n, cc = idx % n;
            A.x[static_cast<size_t>(r) * ld + cc] = cc <= r ? xs[r * kXsPitch + cc] : 0.0f;
            A.xt[static_cast<size_t>(r) * ld + cc] = r <= cc ? xs[cc * kXsPitch + r] : 0.0f;
        }
    }
    if (tid == 0 && *badp != INT_MAX) report_bad(A.info, A.col0 + *badp);
}

__global__ void __launch_bounds__(kSweepThreads, 1) leaf_sweep_kernel(const __grid_constant__ LeafBatch batch) {
    extern __shared__ __align__(16) float sweep_smem[];
    sweep_body(batch.e[blockIdx.x], sweep_smem, true);
}

}  // namespace pf
