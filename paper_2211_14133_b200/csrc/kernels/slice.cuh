// Operand preparation for the fp32-accurate int8 tensor-core GEMM (kOZ8):
// every row of an fp32 matrix is written as
//     x = 2^e * (q0 2^-7 + q1 2^-14 + q2 2^-21 + q3 2^-28),   q_s in [-127, 127]
// with one power-of-two scale per row (max|x| in [2^(e-1), 2^e)).  All digit
// extractions are exact fp32 operations (power-of-two scaling and removal of
// the integer part), so the only error is the last digit's rounding:
// |x - x~| <= 2^(e-29) <= 2^-28 max|row|.
//
// Layout of a sliced operand (one allocation): 4 int8 planes of rows x kpad
// bytes (kpad = k rounded up to 16 for TMA row pitch), then rows int32
// exponents, then rows fp64 squared norms of the REPRESENTED row
// sum_k x~_k^2 * 2^-2e over the valid range.  The GEMM writes the diagonal of
// a same-operand product (X X^T) from these: the omitted digit product
// (q2*q2, weight 2^-42) is >= 0 on the diagonal, so dropping it there would be
// a bias that grows linearly with k; off the diagonal it is an unbiased
// 2^-28-level error.  Columns outside a row's valid (block-triangular) range are
// neither read nor written: the GEMM's k-range never loads them.
#pragma once

#include "ptx.cuh"

#include <cstdint>

namespace pf {

enum SliceMode : int {
    SLICE_FULL = 0,
    SLICE_LOWER_BLOCK = 1,  // row r valid for k < (r/128 + 1) * 128
    SLICE_UPPER_BLOCK = 2,  // row r valid for k >= (r/128) * 128
    SLICE_ZERO_DIAG = 4,    // flag: element (r, r) sliced as 0 (the LAUUM's diagonal
                            // split: the diagonal enters the GEMM epilogue exactly)
};

struct SliceJob {
    const float* src;
    int rows, k, ld;
    int mode;
    int8_t* planes;
    int64_t plane_stride;  // bytes between digit planes
    int kpad;
    int* exps;
    double* sqnorm;
    // optional: the rows are published by their producer with this flag (set
    // to 1) before the producer's launch completes (the leaf's X, ahead of its
    // X^T store); slice_short waits on it instead of on the launch and joins
    // the launch at its end, so its own completion still implies the producer's
    const int* ready = nullptr;
};

constexpr int kMaxSliceJobs = 32;
struct SliceBatch {
    SliceJob j[kMaxSliceJobs];
};

__device__ __forceinline__ void valid_range(const SliceJob& J, int r, int& lo, int& hi) {
    lo = 0;
    hi = J.k;
    const int m = J.mode & 3;
    if (m == SLICE_LOWER_BLOCK) hi = min(J.k, (r / 128 + 1) * 128);
    if (m == SLICE_UPPER_BLOCK) lo = (r / 128) * 128;
}

// SLICE_ZERO_DIAG: zero the component of the float4 at columns [c, c + 4) that
// lies on the diagonal of row r (the row max and norm see the zeroed row).
__device__ __forceinline__ float4 zap_diag(float4 v, const SliceJob& J, int r, int c) {
    if ((J.mode & SLICE_ZERO_DIAG) && r >= c && r < c + 4) {
        const int w = r - c;
        if (w == 0) v.x = 0.0f;
        if (w == 1) v.y = 0.0f;
        if (w == 2) v.z = 0.0f;
        if (w == 3) v.w = 0.0f;
    }
    return v;
}
__device__ __forceinline__ float zap_diag1(float x, const SliceJob& J, int r, int c) {
    return ((J.mode & SLICE_ZERO_DIAG) && r == c) ? 0.0f : x;
}

// Row scale 2^(28-e) as one exact multiplier (0 = out of the normal range:
// fall back to ldexpf per element).
__device__ __forceinline__ float digit_scale(int e) {
    const int k = 28 - e;
    return (k >= -126 && k <= 127) ? __int_as_float((k + 127) << 23) : 0.0f;
}

// Digits of x (row exponent e, sc = digit_scale(e)), in integer arithmetic:
// A = |x| 2^(28-e) < 2^28 (exact scaling); with I = trunc(A), R = rint(A)
//   q0 = I >> 21, q1 = (I >> 14) & 127, q2 = (I >> 7) & 127,
//   q3 = min(R - (I & ~127), 127),   all carrying the sign of x
// -- the same digits as truncating t = x 2^(7-e) digit by digit and rounding
// the last (ties-to-even parity of R equals that of t's last digit), with two
// float->int conversions instead of eight.  Returns |Q| = |x~| 2^(28-e).
__device__ __forceinline__ int slice_digits(float x, int e, float sc, int8_t (&q)[4]) {
    const float a = fabsf(sc != 0.0f ? x * sc : ldexpf(x, 28 - e));
    const int I = __float2int_rz(a);
    const int R = __float2int_rn(a);
    const int hi = I & ~127;
    const int d3 = min(R - hi, 127);
    const int neg = x < 0.0f ? -1 : 0;
    q[0] = static_cast<int8_t>(((I >> 21) ^ neg) - neg);
    q[1] = static_cast<int8_t>((((I >> 14) & 127) ^ neg) - neg);
    q[2] = static_cast<int8_t>((((I >> 7) & 127) ^ neg) - neg);
    q[3] = static_cast<int8_t>((d3 ^ neg) - neg);
    return hi + d3;
}

// Exact sum of Q^2 (< 2^69 for rows up to 8192): 128-bit integer, so the
// squared norm is independent of the summation order (every kernel that
// slices a row -- warp, block or persistent task -- writes the same bits).
struct SqAcc {
    unsigned long long lo = 0, hi = 0;
    __device__ __forceinline__ void add(int qv) {
        const unsigned long long v = static_cast<unsigned long long>(static_cast<long long>(qv) * qv);
        lo += v;
        hi += lo < v ? 1ull : 0ull;
    }
    __device__ __forceinline__ void add_u64(unsigned long long v) {
        lo += v;
        hi += lo < v ? 1ull : 0ull;
    }
    __device__ __forceinline__ void add(const SqAcc& o) {
        lo += o.lo;
        hi += o.hi + (lo < o.lo ? 1ull : 0ull);
    }
    __device__ __forceinline__ void warp_reduce() {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            SqAcc t;
            t.lo = __shfl_xor_sync(0xffffffffu, lo, o);
            t.hi = __shfl_xor_sync(0xffffffffu, hi, o);
            add(t);
        }
    }
    // sum x~^2 2^-2e = sum Q^2 2^-56
    __device__ __forceinline__ double value() const {
        return (static_cast<double>(hi) * 0x1p64 + static_cast<double>(lo)) * 0x1p-56;
    }
};

// Row scale 2^(28-e) as two exact power-of-two factors (each in the normal
// range for every finite-row exponent), so no per-element ldexpf branch.
struct RowScale {
    float s1, s2;
};
__device__ __forceinline__ RowScale row_scale2(int e) {
    const int k = 28 - e, k1 = k / 2, k2 = k - k1;
    return RowScale{__int_as_float((k1 + 127) << 23), __int_as_float((k2 + 127) << 23)};
}

// Four consecutive elements -> the four digit-plane words (byte w of plane
// word p = digit p of element w) and the exact sum of their Q^2.  Same digits
// as slice_digits: magnitudes from I = trunc(A), R = rint(A) packed into one
// word per element, sign applied bytewise without carries ((0x80 - m) ^ 0x80
// = -m mod 256 for m <= 127), then a 4x4 byte transpose (8 PRMT).  ~20
// instructions per element instead of ~60.
__device__ __forceinline__ void slice4(const float4 v, RowScale rs, uint32_t (&P)[4], unsigned long long& sq) {
    const float xs[4] = {v.x, v.y, v.z, v.w};
    uint32_t W[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const float a = fabsf(xs[w] * rs.s1 * rs.s2);  // |x| 2^(28-e) < 2^28, exact
        const uint32_t I = static_cast<uint32_t>(__float2int_rz(a));
        const uint32_t R = static_cast<uint32_t>(__float2int_rn(a));
        const uint32_t hi = I & ~127u;
        const uint32_t d3 = min(R - hi, 127u);
        sq += static_cast<unsigned long long>(hi + d3) * (hi + d3);
        const uint32_t m = (I >> 21) | ((I >> 6) & 0x7F00u) | ((I << 9) & 0x7F0000u) | (d3 << 24);
        const uint32_t neg = (0x80808080u - m) ^ 0x80808080u;
        W[w] = xs[w] < 0.0f ? neg : m;
    }
    const uint32_t t0 = __byte_perm(W[0], W[1], 0x5140), t1 = __byte_perm(W[0], W[1], 0x7362);
    const uint32_t t2 = __byte_perm(W[2], W[3], 0x5140), t3 = __byte_perm(W[2], W[3], 0x7362);
    P[0] = __byte_perm(t0, t2, 0x5410);
    P[1] = __byte_perm(t0, t2, 0x7632);
    P[2] = __byte_perm(t1, t3, 0x5410);
    P[3] = __byte_perm(t1, t3, 0x7632);
}

// One warp slices row r of job J.  Rows whose valid range is 16-byte aligned
// move 4 elements per lane per access (float4 in, char4 out) with 4 accesses
// in flight per lane.  Loads bypass L1 (ld.global.cg): in the persistent
// inversion kernel the rows were written by other SMs moments earlier.
// kV: float4 per lane held in registers by the one-pass path (rows up to
// 128 kV elements); longer rows take two passes.
template <int kV = 8>
__device__ __forceinline__ void slice_row(const SliceJob& J, int r, int lane) {
    int lo, hi;
    valid_range(J, r, lo, hi);
    const float* row = J.src + static_cast<int64_t>(r) * J.ld;
    int8_t* p0 = J.planes + static_cast<int64_t>(r) * J.kpad;
    const bool vec = ((reinterpret_cast<uintptr_t>(row + lo) & 15) == 0) && ((hi - lo) % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(p0 + lo) & 3) == 0) && (J.plane_stride % 4 == 0);
    float m = 0.0f;
    if (vec && hi - lo <= 128 * kV) {
        // short row (every inversion operand up to d = 1024): ONE pass over
        // global memory, the row stays in registers between max and digits
        const float4* r4 = reinterpret_cast<const float4*>(row + lo);
        const int n4 = (hi - lo) / 4;
        float4 v[kV];
#pragma unroll
        for (int u = 0; u < kV; ++u)
            v[u] = (lane + 32 * u < n4) ? zap_diag(__ldcg(r4 + lane + 32 * u), J, r, lo + 4 * (lane + 32 * u))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < kV; ++u)
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        int e = 0;
        if (m > 0.0f) frexpf(m, &e);
        if (lane == 0) J.exps[r] = e;
        const float sc = digit_scale(e);
        const RowScale rs = row_scale2(e);
        (void)sc;
        SqAcc sq;
        unsigned long long sq64 = 0;  // <= 16 float4 per lane: < 2^62
#pragma unroll
        for (int u = 0; u < kV; ++u) {
            const int c = lane + 32 * u;
            if (c >= n4) continue;
            uint32_t packed[4];
            slice4(v[u], rs, packed, sq64);
#pragma unroll
            for (int pl = 0; pl < 4; ++pl)
                *reinterpret_cast<uint32_t*>(p0 + lo + 4 * c + pl * J.plane_stride) = packed[pl];
        }
        sq.add_u64(sq64);
        sq.warp_reduce();
        if (lane == 0) J.sqnorm[r] = sq.value();
        return;
    }
    if (vec) {
        const float4* r4 = reinterpret_cast<const float4*>(row + lo);
        const int n4 = (hi - lo) / 4;
        int c = lane;
        for (; c + 96 < n4; c += 128) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = zap_diag(__ldcg(r4 + c + 32 * u), J, r, lo + 4 * (c + 32 * u));
#pragma unroll
            for (int u = 0; u < 4; ++u)
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
        }
        for (; c < n4; c += 32) {
            const float4 v = zap_diag(__ldcg(r4 + c), J, r, lo + 4 * c);
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
    } else {
        for (int c = lo + lane; c < hi; c += 32) m = fmaxf(m, fabsf(zap_diag1(__ldcg(row + c), J, r, c)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    int e = 0;
    if (m > 0.0f) {
        int ex;
        frexpf(m, &ex);  // m = f * 2^ex, f in [0.5, 1)
        e = ex;          // so max|row| < 2^e
    }
    if (lane == 0) J.exps[r] = e;
    const float sc = digit_scale(e);
    const RowScale rs = row_scale2(e);
    SqAcc sq;
    if (vec) {
        const float4* r4 = reinterpret_cast<const float4*>(row + lo);
        const int n4 = (hi - lo) / 4;
        for (int c = lane; c < n4; c += 32) {
            const float4 v = zap_diag(__ldcg(r4 + c), J, r, lo + 4 * c);
            uint32_t packed[4];
            unsigned long long sq64 = 0;
            slice4(v, rs, packed, sq64);
            sq.add_u64(sq64);
#pragma unroll
            for (int pl = 0; pl < 4; ++pl)
                *reinterpret_cast<uint32_t*>(p0 + lo + 4 * c + pl * J.plane_stride) = packed[pl];
        }
    } else {
        for (int c = lo + lane; c < hi; c += 32) {
            int8_t q[4];
            sq.add(slice_digits(zap_diag1(__ldcg(row + c), J, r, c), e, sc, q));
#pragma unroll
            for (int pl = 0; pl < 4; ++pl) p0[c + pl * J.plane_stride] = q[pl];
        }
    }
    sq.warp_reduce();
    if (lane == 0) J.sqnorm[r] = sq.value();
}

// Long rows (1024 < valid length <= 8192, 16-byte aligned): one 256-thread
// block per row, each thread holding up to 8 float4 in registers, so the row
// is read from global memory ONCE with 8 loads in flight per thread (the
// warp-per-row path above reads long rows twice with one load in flight).
constexpr int kLongThreads = 256;
constexpr int kLongVec = 8;  // float4 per thread -> rows up to 8192

template <int kThreads = kLongThreads>
__device__ __forceinline__ bool long_row_ok(const SliceJob& J, int r, int& lo, int& hi) {
    valid_range(J, r, lo, hi);
    const float* row = J.src + static_cast<int64_t>(r) * J.ld;
    int8_t* p0 = J.planes + static_cast<int64_t>(r) * J.kpad;
    return ((reinterpret_cast<uintptr_t>(row + lo) & 15) == 0) && ((hi - lo) % 4 == 0) &&
           ((reinterpret_cast<uintptr_t>(p0 + lo) & 3) == 0) && (J.plane_stride % 4 == 0) &&
           hi - lo <= 4 * kThreads * kLongVec;
}

// kThreads per row: 128 for rows up to 4096 (8 float4 per thread: the per-row
// reductions amortised over twice the elements), 256 up to 8192.
template <int kThreads>
__global__ void __launch_bounds__(kThreads) slice_long_kernel(const __grid_constant__ SliceBatch b) {
    const SliceJob& J = b.j[blockIdx.y];
    const int r = blockIdx.x;
    ptx::grid_dep_wait();
    ptx::grid_dep_launch();
    if (r >= J.rows) return;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int lo, hi;
    if (!long_row_ok<kThreads>(J, r, lo, hi)) {  // unaligned / over-long rows: warp path
        if (warp == 0) slice_row(J, r, lane);
        return;
    }
    __shared__ float red_m[kThreads / 32];
    __shared__ SqAcc red_s[kThreads / 32];
    const float4* r4 = reinterpret_cast<const float4*>(J.src + static_cast<int64_t>(r) * J.ld + lo);
    int8_t* p0 = J.planes + static_cast<int64_t>(r) * J.kpad + lo;
    const int n4 = (hi - lo) / 4;
    float4 v[kLongVec];
#pragma unroll
    for (int u = 0; u < kLongVec; ++u)
        v[u] = (t + kThreads * u < n4) ? zap_diag(__ldcg(r4 + t + kThreads * u), J, r, lo + 4 * (t + kThreads * u))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
    float m = 0.0f;
#pragma unroll
    for (int u = 0; u < kLongVec; ++u)
        m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red_m[warp] = m;
    __syncthreads();
    m = red_m[0];
#pragma unroll
    for (int w = 1; w < kThreads / 32; ++w) m = fmaxf(m, red_m[w]);
    int e = 0;
    if (m > 0.0f) frexpf(m, &e);
    if (t == 0) J.exps[r] = e;
    const RowScale rs = row_scale2(e);
    SqAcc sq;
    unsigned long long sq64 = 0;  // <= 8 float4 per thread: < 2^61
#pragma unroll
    for (int u = 0; u < kLongVec; ++u) {
        const int c = t + kThreads * u;
        if (c >= n4) continue;
        uint32_t packed[4];
        slice4(v[u], rs, packed, sq64);
#pragma unroll
        for (int pl = 0; pl < 4; ++pl) *reinterpret_cast<uint32_t*>(p0 + 4 * c + pl * J.plane_stride) = packed[pl];
    }
    sq.add_u64(sq64);
    sq.warp_reduce();
    if (lane == 0) red_s[warp] = sq;
    __syncthreads();
    if (t == 0) {
        SqAcc tot;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) tot.add(red_s[w]);
        J.sqnorm[r] = tot.value();
    }
}

// Short rows (<= 256 floats, every job 16-byte aligned: checked by the
// caller): eight lanes per row, 32 rows per 256-thread block, so the per-row
// reductions take 3 shuffle steps over up to 8 float4 per lane instead of 5
// over one (the 128-wide panel operands of the right-looking inversion).
// Template: kLanes lanes per row holding up to kV float4 each (8 x 8: rows
// <= 256; a 16 x 16 form for rows <= 1024 measured slower than a warp per
// row: 110 registers).
template <int kLanes, int kV>
__global__ void __launch_bounds__(256) slice_short_kernel(const __grid_constant__ SliceBatch b) {
    const SliceJob& J = b.j[blockIdx.y];
    const int g = threadIdx.x & (kLanes - 1);                              // lane within the row group
    const int r = blockIdx.x * (256 / kLanes) + threadIdx.x / kLanes;  // row
    if (J.ready) {
        if (threadIdx.x == 0)
            while (ptx::ld_acquire_gpu(J.ready) == 0) __nanosleep(64);
        __syncthreads();
    } else {
        ptx::grid_dep_wait();
    }
    ptx::grid_dep_launch();
    const bool live = r < J.rows;
    int lo = 0, hi = 0;
    if (live) valid_range(J, r, lo, hi);
    const int n4 = live ? (hi - lo) / 4 : 0;
    const float4* r4 = reinterpret_cast<const float4*>(J.src + static_cast<int64_t>(live ? r : 0) * J.ld + lo);
    float4 v[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u)
        v[u] = (g + kLanes * u < n4) ? zap_diag(__ldcg(r4 + g + kLanes * u), J, r, lo + 4 * (g + kLanes * u))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
    float m = 0.0f;
#pragma unroll
    for (int u = 0; u < kV; ++u)
        m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
#pragma unroll
    for (int o = kLanes / 2; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    int e = 0;
    if (m > 0.0f) frexpf(m, &e);
    const RowScale rs = row_scale2(e);
    int8_t* p0 = J.planes + static_cast<int64_t>(live ? r : 0) * J.kpad + lo;
    unsigned long long sq64 = 0;
#pragma unroll
    for (int u = 0; u < kV; ++u) {
        const int c = g + kLanes * u;
        if (c >= n4) continue;
        uint32_t packed[4];
        slice4(v[u], rs, packed, sq64);
#pragma unroll
        for (int pl = 0; pl < 4; ++pl) *reinterpret_cast<uint32_t*>(p0 + 4 * c + pl * J.plane_stride) = packed[pl];
    }
    SqAcc sq;
    sq.add_u64(sq64);
#pragma unroll
    for (int o = kLanes / 2; o > 0; o >>= 1) {
        SqAcc t;
        t.lo = __shfl_xor_sync(0xffffffffu, sq.lo, o);
        t.hi = __shfl_xor_sync(0xffffffffu, sq.hi, o);
        sq.add(t);
    }
    if (live && g == 0) {
        J.exps[r] = e;
        J.sqnorm[r] = sq.value();
    }
    if (J.ready) ptx::grid_dep_wait();  // complete only after the producer's launch
}

// one warp per row; grid (ceil(rows / 8), jobs)
template <int kV>
__global__ void __launch_bounds__(256) slice_kernel(const __grid_constant__ SliceBatch b) {
    const SliceJob& J = b.j[blockIdx.y];
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
    ptx::grid_dep_wait();  // PDL: the rows are produced by the previous launch
    ptx::grid_dep_launch();
    if (r >= J.rows) return;
    slice_row<kV>(J, r, threadIdx.x & 31);
}

}  // namespace pf
