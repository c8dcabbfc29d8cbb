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
};

constexpr int kMaxSliceJobs = 32;
struct SliceBatch {
    SliceJob j[kMaxSliceJobs];
};

__device__ __forceinline__ void valid_range(const SliceJob& J, int r, int& lo, int& hi) {
    lo = 0;
    hi = J.k;
    if (J.mode == SLICE_LOWER_BLOCK) hi = min(J.k, (r / 128 + 1) * 128);
    if (J.mode == SLICE_UPPER_BLOCK) lo = (r / 128) * 128;
}

__device__ __forceinline__ void slice_digits(float x, int e, int8_t (&q)[4], double& rep) {
    float t = ldexpf(x, 7 - e);  // x * 2^-e * 2^7, |t| < 128 (exact: power-of-two scaling)
    const float q0 = truncf(t);
    t = (t - q0) * 128.0f;
    const float q1 = truncf(t);
    t = (t - q1) * 128.0f;
    const float q2 = truncf(t);
    t = (t - q2) * 128.0f;
    const float q3 = fminf(fmaxf(rintf(t), -127.0f), 127.0f);
    q[0] = static_cast<int8_t>(q0);
    q[1] = static_cast<int8_t>(q1);
    q[2] = static_cast<int8_t>(q2);
    q[3] = static_cast<int8_t>(q3);
    rep = static_cast<double>(q0) * 0x1p-7 + static_cast<double>(q1) * 0x1p-14 +
          static_cast<double>(q2) * 0x1p-21 + static_cast<double>(q3) * 0x1p-28;
}

// One warp slices row r of job J.  Rows whose valid range is 16-byte aligned
// move 4 elements per lane per access (float4 in, char4 out) with 4 accesses
// in flight per lane.  Loads bypass L1 (ld.global.cg): in the persistent
// inversion kernel the rows were written by other SMs moments earlier.
__device__ __forceinline__ void slice_row(const SliceJob& J, int r, int lane) {
    int lo, hi;
    valid_range(J, r, lo, hi);
    const float* row = J.src + static_cast<int64_t>(r) * J.ld;
    int8_t* p0 = J.planes + static_cast<int64_t>(r) * J.kpad;
    const bool vec = ((reinterpret_cast<uintptr_t>(row + lo) & 15) == 0) && ((hi - lo) % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(p0 + lo) & 3) == 0) && (J.plane_stride % 4 == 0);
    float m = 0.0f;
    if (vec && hi - lo <= 1024) {
        // short row (every inversion operand up to d = 1024): ONE pass over
        // global memory, the row stays in registers between max and digits
        const float4* r4 = reinterpret_cast<const float4*>(row + lo);
        const int n4 = (hi - lo) / 4;
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (lane + 32 * u < n4) ? __ldcg(r4 + lane + 32 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u)
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        int e = 0;
        if (m > 0.0f) frexpf(m, &e);
        if (lane == 0) J.exps[r] = e;
        double sq = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int c = lane + 32 * u;
            if (c >= n4) continue;
            const float xs[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
            uint32_t packed[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                int8_t q[4];
                double rep;
                slice_digits(xs[w], e, q, rep);
                sq = fma(rep, rep, sq);
#pragma unroll
                for (int pl = 0; pl < 4; ++pl)
                    packed[pl] |= static_cast<uint32_t>(static_cast<uint8_t>(q[pl])) << (8 * w);
            }
#pragma unroll
            for (int pl = 0; pl < 4; ++pl)
                *reinterpret_cast<uint32_t*>(p0 + lo + 4 * c + pl * J.plane_stride) = packed[pl];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) J.sqnorm[r] = sq;
        return;
    }
    if (vec) {
        const float4* r4 = reinterpret_cast<const float4*>(row + lo);
        const int n4 = (hi - lo) / 4;
        int c = lane;
        for (; c + 96 < n4; c += 128) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcg(r4 + c + 32 * u);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
        }
        for (; c < n4; c += 32) {
            const float4 v = __ldcg(r4 + c);
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
    } else {
        for (int c = lo + lane; c < hi; c += 32) m = fmaxf(m, fabsf(__ldcg(row + c)));
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
    double sq = 0.0;
    if (vec) {
        const float4* r4 = reinterpret_cast<const float4*>(row + lo);
        const int n4 = (hi - lo) / 4;
        for (int c = lane; c < n4; c += 32) {
            const float4 v = __ldcg(r4 + c);
            const float xs[4] = {v.x, v.y, v.z, v.w};
            uint32_t packed[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                int8_t q[4];
                double rep;
                slice_digits(xs[u], e, q, rep);
                sq = fma(rep, rep, sq);
#pragma unroll
                for (int pl = 0; pl < 4; ++pl)
                    packed[pl] |= static_cast<uint32_t>(static_cast<uint8_t>(q[pl])) << (8 * u);
            }
#pragma unroll
            for (int pl = 0; pl < 4; ++pl)
                *reinterpret_cast<uint32_t*>(p0 + lo + 4 * c + pl * J.plane_stride) = packed[pl];
        }
    } else {
        for (int c = lo + lane; c < hi; c += 32) {
            int8_t q[4];
            double rep;
            slice_digits(__ldcg(row + c), e, q, rep);
            sq = fma(rep, rep, sq);
#pragma unroll
            for (int pl = 0; pl < 4; ++pl) p0[c + pl * J.plane_stride] = q[pl];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) J.sqnorm[r] = sq;
}

// one warp per row; grid (ceil(rows / 8), jobs)
__global__ void __launch_bounds__(256) slice_kernel(const __grid_constant__ SliceBatch b) {
    const SliceJob& J = b.j[blockIdx.y];
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
    ptx::grid_dep_wait();  // PDL: the rows are produced by the previous launch
    ptx::grid_dep_launch();
    if (r >= J.rows) return;
    slice_row(J, r, threadIdx.x & 31);
}

}  // namespace pf
