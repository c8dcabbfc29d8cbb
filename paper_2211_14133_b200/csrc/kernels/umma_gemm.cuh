// Grouped "TN" tensor-core GEMM for sm_100a: C = alpha * A * B^T (+ beta * C)
// with A [rows x k] and B [cols x k] both K-major (K contiguous).  One kernel
// template serves every K-FAC hot op:
//
//   kFmt = kBF16   curvature SYRK: A = B = X (bf16 [d x n_tokens]), lower tiles
//                  only, mirrored store -> full symmetric fp32 factor.
//                  kind::f16, 1 operand plane, fp32 accumulator in TMEM.
//   kFmt = kOZ8    fp32-accurate products (damped-inverse recursion,
//                  preconditioning): each fp32 operand row is pre-sliced
//                  (slice kernel) into a power-of-two row scale 2^e and four
//                  int8 digits q0..q3 of 7 bits each (x = 2^e sum_s q_s 2^-7(s+1)).
//                  The 10 digit products with s_a + s_b <= 3 run as
//                  tcgen05.mma.kind::i8 with EXACT int32 accumulation, one TMEM
//                  accumulator per digit weight g = s_a + s_b (4 x 128 columns =
//                  all 512), recombined in FP32 in the epilogue (three fmaf,
//                  smallest weight first, then one multiply by the power-of-two
//                  row x column scale: ~1 ulp of the fp32 result).  Error:
//                  2^-28 of the ROW MAX per operand element from slicing (plus
//                  the dropped s_a + s_b >= 4 products, same order), none from
//                  accumulation.  Being relative to the row max, it hurts rows
//                  with a large max/rms ratio -- see EPI_DIAG_SPLIT.
//
// Structure (one CTA = one 128x128 output tile, 4 warps):
//   warp 0 / lane 0 : TMA producer, kStages-deep smem ring (full/empty mbarriers)
//   warp 1 / lane 0 : tcgen05.mma issuer (single thread)
//   all 4 warps     : epilogue, tcgen05.ld 32x32b -> registers -> global
// Operand tiles: bf16 128 rows x 128 B (SWIZZLE_128B, 64 elements per k-block);
// int8 digits 128 rows x 64 B (SWIZZLE_64B, 64 elements per k-block).
#pragma once

#include <cuda.h>
#include <cstdint>

#include "ptx.cuh"

namespace pf {

#ifdef PF_GEMM_PROBE
// globaltimer stamps (ns) of CTA 0 of small beta != 0 GEMMs, one record of 8
// per launch: [0..5] stamps, [6] rows, [7] cols
__device__ long long g_gemm_probe[64 * 16];
__device__ long long g_gemm_probe_epi[8];
__device__ int g_gemm_probe_n;
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define PF_GSTAMP(i, cond)                                                      \
    do {                                                                        \
        if ((cond) && probe_on) reinterpret_cast<long long*>(tail + 128)[i] = gtimer(); \
    } while (0)
#define PF_ESTAMP(i)                                                                       \
    do {                                                                                   \
        if (blockIdx.x == 0 && threadIdx.x == 0 && P.beta != 0.0f && P.rows <= kTile && P.cols <= kTile) \
            g_gemm_probe_epi[i] = gtimer();                                                \
    } while (0)
#else
#define PF_ESTAMP(i) \
    do {             \
    } while (0)
#define PF_GSTAMP(i, cond) \
    do {                   \
    } while (0)
#endif

constexpr int kTile = 128;
constexpr int kMaxMaps = 96;
constexpr int kMaxProbs = 16;
constexpr int kBF16 = 1;
constexpr int kOZ8 = 3;
constexpr int kDigits = 4;  // int8 digits per fp32 value (28 bits)

enum EpiFlag : uint32_t {
    EPI_MIRROR = 1u,     // off-diagonal tiles also stored transposed (symmetric result)
    EPI_TRANSPOSE = 2u,  // store C^T (into c) instead of C
    EPI_ALSO_T = 16u,    // additionally store C^T into c_t
    EPI_VEC4 = 32u,      // c / ldc 16-byte aligned: vectorised row stores
    EPI_EXACT_DIAG = 64u,  // kOZ8, A == B: diagonal from the operand's exact row norms
    // kOZ8 LAUUM C = (D + O)(D + O)^T with A = B = O sliced with its diagonal
    // zeroed (SLICE_ZERO_DIAG) and D = diag(X): the terms with D are added here
    // in fp32 from aux = X (row-major lower, X[r][c] = O[c][r] for c < r):
    //   C[r][c] += X[r][r] X[r][c] (c < r),  X[c][c] X[c][r] (c > r),  X[r][r]^2 (c == r).
    // The digit form's error is relative to a row's max, which for the rows of
    // L^-T is the diagonal (20-30x the rms); without it the LAUUM error grew
    // linearly with d (residual 9.5e-6 at d = 4096, 1.9e-6 with the split).
    EPI_DIAG_SPLIT = 128u,
};

// Tile (tm, tn) reads only the k-slice where both triangular operands can be
// non-zero; the rest is never touched (no zero-fill needed outside it).
enum KMode : int {
    K_FULL = 0,
    K_FROM_ROW_TILE = 1,    // k in [tm*128, k)
    K_FROM_COL_TILE = 2,    // k in [tn*128, k)
    K_TO_ROW_TILE_END = 3,  // k in [0, (tm+1)*128)
    K_TO_COL_TILE_END = 4,  // k in [0, (tn+1)*128)
};

struct GemmDesc {
    int a_map, b_map;   // CUtensorMap index per operand (kOZ8: 3-D map over the 4 digit planes)
    int rows, cols, k;
    int tiles_m, tiles_n;
    int lower;          // enumerate only tiles with tm >= tn
    int tile_begin;
    int k_mode;
    float alpha, beta;
    uint32_t flags;
    const int* a_exp;   // kOZ8: per-row scale exponents of A / B
    const int* b_exp;
    const double* a_sqnorm;  // kOZ8 + EPI_EXACT_DIAG
    float* c;
    float* c_t;
    int ldc, ldc_t;
    const float* aux;    // EPI_DIAG_SPLIT: X (16-byte aligned rows, ld_aux % 4 == 0)
    const float* aux_t;  //   and X^T (same ld)
    int ld_aux;
    int mn_major;        // kBF16: operands stored [k x rows] (row-contiguous, e.g. token-major
                         // activations [tokens x features]); two 64-wide TMA boxes per tile
};

// MN-major bf16 operand tiles: 64-feature groups of 64 tokens x 128 B
constexpr int kMnGroupBytes = 64 * 128;

struct GemmBatch {
    CUtensorMap maps[kMaxMaps];
    GemmDesc probs[kMaxProbs];
    int n_probs;
    int total_tiles;
    int interleave;  // all problems share tile count and k-mode: tile rank major, problem minor
    int k_split;     // kBF16: >= 2 -> clusters of k_split CTAs per tile, each one k_split-th of
                     // the k-blocks; the partial tiles are summed over DSMEM in cluster-rank order
};

// kN: tile width (columns of C, rows of B).  128 everywhere except short
// K_FULL kOZ8 launches with few tiles, which split each 128-wide tile over
// 2 or 4 CTAs (kN = 64 / 32) so a latency-bound update spreads its MMAs and
// epilogue over more SMs.
template <int kFmt, int kN = 128>
struct GemmTraits {
    static constexpr int kPlanes = kFmt == kOZ8 ? kDigits : 1;
    static constexpr int kPlaneBytes = kFmt == kOZ8 ? 128 * 64 : 128 * 128;  // A plane (128 rows)
    static constexpr int kPlaneBytesB = kFmt == kOZ8 ? kN * 64 : kN * 128;   // B plane (kN rows)
    static constexpr int kStageBytes = kPlanes * (kPlaneBytes + kPlaneBytesB);
    // bf16 128x256 tiles (48 KB per stage) keep two CTAs per SM with 2 stages each
    static constexpr int kStages = kFmt == kBF16 && kN == 256 ? 2 : 3;
    // C-tile prefetch buffer (beta != 0, <= kStages-1 k-blocks): the unused
    // last stage plus kCPad, rows padded to kCStride floats (bank rotation)
    static constexpr int kCStride = kN + 4;
    static constexpr int kCPad =
        kFmt == kOZ8 && kTile * kCStride * 4 > kStageBytes ? kTile * kCStride * 4 - kStageBytes : 0;
    static constexpr int kSmemBytes = kStages * kStageBytes + kCPad + 1024 + 256 + 4 * kTile;
    static constexpr int kKBlock = 64;  // elements per k-block (both formats)
    static constexpr int kKSteps = kFmt == kOZ8 ? 2 : 4;  // 32-byte UMMA k-steps per block
    static constexpr uint32_t kTmemCols = kFmt == kOZ8 ? 4 * kN : kN;
    static constexpr int kMinBlocks = kFmt == kOZ8 ? 1 : 2;
    // kOZ8 (one CTA per SM: 512 TMEM columns) runs 8 warps so the 4-accumulator
    // epilogue is split over warp pairs sharing a TMEM lane quarter
    static constexpr int kThreads = kFmt == kOZ8 ? 256 : 128;
    // kind::i8: signed int8 A/B (format 1), s32 accumulate (c_format 2)
    static constexpr uint32_t kIdesc =
        kFmt == kOZ8 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((static_cast<uint32_t>(kN) >> 3) << 17) |
                        ((128u >> 4) << 24))
                     : ptx::make_idesc(1, 128, kN);
};

__device__ __forceinline__ void decode_lower(int t, int& tm, int& tn);
__device__ __forceinline__ void decode_lower_wide(int t, int& tm, int& tn);

// Local tile index -> (tm, tn), longest k-range first (LPT): with triangular
// k-ranges the last wave would otherwise wait on the longest tiles.
__device__ __forceinline__ void map_tile(const GemmDesc& P, int lt, int& tm, int& tn) {
    if (P.lower == 2) {  // 128 x 256 tiles (kBF16 kN = 256), K_FULL
        decode_lower_wide(lt, tm, tn);
        return;
    }
    if (P.lower) {  // decode_lower walks tm ascending: K_FROM_ROW_TILE longest first
        decode_lower(lt, tm, tn);
        return;
    }
    switch (P.k_mode) {
        case K_TO_COL_TILE_END:  // k-length grows with tn
            tn = P.tiles_n - 1 - lt / P.tiles_m;
            tm = lt % P.tiles_m;
            break;
        case K_FROM_COL_TILE:  // shrinks with tn
            tn = lt / P.tiles_m;
            tm = lt % P.tiles_m;
            break;
        case K_TO_ROW_TILE_END:  // grows with tm
            tm = P.tiles_m - 1 - lt / P.tiles_n;
            tn = lt % P.tiles_n;
            break;
        default:
            tm = lt / P.tiles_n;
            tn = lt % P.tiles_n;
    }
}

// Lower tiles of 128 rows x 256 columns: row tile tm has tm / 2 + 1 of them
// (the last one holds the 128 x 128 diagonal block, plus the block right of
// it when tm is even -- never stored); rows 2a and 2a+1 start at a (a + 1).
__device__ __forceinline__ void decode_lower_wide(int t, int& tm, int& tn) {
    int a = static_cast<int>((sqrtf(4.0f * static_cast<float>(t) + 1.0f) - 1.0f) * 0.5f);
    while ((a + 1) * (a + 2) <= t) ++a;
    while (a * (a + 1) > t) --a;
    const int r = t - a * (a + 1);
    if (r <= a) {
        tm = 2 * a;
        tn = r;
    } else {
        tm = 2 * a + 1;
        tn = r - a - 1;
    }
}

__device__ __forceinline__ void decode_lower(int t, int& tm, int& tn) {
    int m = static_cast<int>((sqrtf(8.0f * static_cast<float>(t) + 1.0f) - 1.0f) * 0.5f);
    while ((m + 1) * (m + 2) / 2 <= t) ++m;
    while (m * (m + 1) / 2 > t) --m;
    tm = m;
    tn = t - m * (m + 1) / 2;
}

// Epilogue of one 128x128 tile for the calling thread's TMEM lane (= tile row
// r), chunks [chunk_begin, chunk_end) of 16 columns: TMEM -> registers ->
// (alpha, digit recombination, beta) -> global.  Shared by the standalone
// kernel (4 warps x 8 chunks) and the persistent inversion kernel (8 warps x
// 4 chunks).  Global reads use ld.global.cg (data may come from other SMs of
// the same persistent launch).
// Per-row epilogue constants, loaded before the accumulator is ready.
struct EpiRow {
    float row_scale = 1.0f;
    float diag_exact = 0.0f;
    float dg = 0.0f;  // EPI_DIAG_SPLIT: X[r][r]
};

template <int kFmt, int kN = 128, bool kSplit = false>
__device__ __forceinline__ EpiRow epi_row(const GemmDesc& P, int tm, int tn, int r) {
    EpiRow e;
    (void)tm;
    if constexpr (kFmt == kOZ8) {
        if (r < P.rows) {
            e.row_scale = P.alpha * ptx::pow2f(__ldcg(P.a_exp + r));
            if ((P.flags & EPI_EXACT_DIAG) && r >= tn * kN && r < (tn + 1) * kN)  // row's diagonal in this tile
                e.diag_exact = static_cast<float>(__ldcg(P.a_sqnorm + r));  // = (norm 2^14) 2^-14
            if (kSplit) e.dg = __ldcg(P.aux + static_cast<size_t>(r) * P.ld_aux + r);
        }
    }
    return e;
}

// beta * C and the stores of one 16-column chunk of tile row r (global row)
template <int kN>
__device__ __forceinline__ void finish_chunk(const GemmDesc& P, int tm, int tn, int r, int chunk, float (&out)[16],
                                             const float* crow) {
    const uint32_t f = P.flags;
    const bool row_ok = r < P.rows;
    const int c0 = tn * kN + chunk * 16;
    // 128-wide column block of the chunk (== tn for 128-wide tiles): a lower
    // launch never stores blocks right of the diagonal block, and mirrors the
    // ones left of it
    const int cb = c0 / kTile;
    if (!row_ok || c0 >= P.cols || (P.lower && cb > tm)) return;
    const bool mirror = (f & EPI_MIRROR) && cb != tm;
    const bool full_chunk = c0 + 16 <= P.cols;
    if (P.beta != 0.0f) {
        float cv[16];
        if (crow && full_chunk) {  // C row prefetched into shared memory
            const float4* src = reinterpret_cast<const float4*>(crow + chunk * 16);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 t = src[q];
                cv[4 * q] = t.x;
                cv[4 * q + 1] = t.y;
                cv[4 * q + 2] = t.z;
                cv[4 * q + 3] = t.w;
            }
        } else if ((f & EPI_VEC4) && full_chunk && !(f & EPI_TRANSPOSE)) {
            const float4* src = reinterpret_cast<const float4*>(P.c + static_cast<size_t>(r) * P.ldc + c0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 t = __ldcg(src + q);
                cv[4 * q] = t.x;
                cv[4 * q + 1] = t.y;
                cv[4 * q + 2] = t.z;
                cv[4 * q + 3] = t.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int c = c0 + j;
                const size_t idx = (f & EPI_TRANSPOSE) ? static_cast<size_t>(c) * P.ldc + r
                                                       : static_cast<size_t>(r) * P.ldc + c;
                cv[j] = c < P.cols ? __ldcg(P.c + idx) : 0.0f;
            }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) out[j] = fmaf(P.beta, cv[j], out[j]);
    }
#ifdef PF_PROBE_NOSTORE
    if (P.beta != 0.0f && P.rows <= kTile && P.cols <= kTile) {
        if (out[0] == 12345.678f) P.c[0] = out[1];  // keep the values live
        return;
    }
#endif
    if ((f & EPI_VEC4) && full_chunk && !(f & EPI_TRANSPOSE)) {
        float4* dst = reinterpret_cast<float4*>(P.c + static_cast<size_t>(r) * P.ldc + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            dst[q] = make_float4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
    } else if (f & EPI_TRANSPOSE) {
        // lanes hold consecutive rows -> each transposed column store is coalesced
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (c0 + j < P.cols) P.c[static_cast<size_t>(c0 + j) * P.ldc + r] = out[j];
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (c0 + j < P.cols) P.c[static_cast<size_t>(r) * P.ldc + c0 + j] = out[j];
    }
    if (mirror) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (c0 + j < P.cols) P.c[static_cast<size_t>(c0 + j) * P.ldc + r] = out[j];
    }
    if (f & EPI_ALSO_T) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (c0 + j < P.cols) P.c_t[static_cast<size_t>(c0 + j) * P.ldc_t + r] = out[j];
    }
}

// col_scale: kOZ8 -> 2^e_b per tile column, kBF16 -> unused.
// kSplit: the EPI_DIAG_SPLIT variant (a separate instantiation: its extra
// loads and registers stay out of every other digit GEMM)
template <int kFmt, int kN = 128, bool kSplit = false>
__device__ __forceinline__ void epilogue_chunks(const GemmDesc& P, int tm, int tn, uint32_t lane_base, int r,
                                                const float* col_scale, int chunk_begin, int chunk_end,
                                                bool have_acc, const EpiRow& er, const float* crow = nullptr) {
    const bool row_ok = r < P.rows;
    const uint32_t f = P.flags;
    const float row_scale = er.row_scale;
    const bool exact_diag = (f & EPI_EXACT_DIAG) && row_ok;  // diag_chunk below: global r == c
    const float diag_exact = er.diag_exact;
    PF_ESTAMP(0);
    auto finish = [&](float (&out)[16], int chunk) { finish_chunk<kN>(P, tm, tn, r, chunk, out, crow); };
    // the diagonal of a same-operand product: exact norm of the represented row
    auto diag_fix = [&](float (&out)[16], int chunk) {
        const int c0 = tn * kN + chunk * 16;
        if (exact_diag && r >= c0 && r < c0 + 16) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j == r) out[j] = (row_scale * col_scale[chunk * 16 + j]) * diag_exact;
        }
    };
    // EPI_DIAG_SPLIT: the diagonal's terms, exactly as one fp32 fma each
    auto split_fix = [&](float (&out)[16], int chunk) {
        if constexpr (!kSplit) return;
        if (!row_ok) return;
        const int c0 = tn * kN + chunk * 16;
        const float* xr = P.aux + static_cast<size_t>(r) * P.ld_aux;
        if (c0 + 16 <= r) {  // left of the diagonal (every chunk of a lower off-diagonal tile)
            const float4* src = reinterpret_cast<const float4*>(xr + c0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 t = __ldcg(src + q);
                out[4 * q] = fmaf(er.dg, t.x, out[4 * q]);
                out[4 * q + 1] = fmaf(er.dg, t.y, out[4 * q + 1]);
                out[4 * q + 2] = fmaf(er.dg, t.z, out[4 * q + 2]);
                out[4 * q + 3] = fmaf(er.dg, t.w, out[4 * q + 3]);
            }
            return;
        }
        // diagonal tiles: the row of X left of the diagonal, the row of X^T
        // right of it (both contiguous), the diagonal X[c][c] (warp-uniform c);
        // all loads issued before the fmas (fully unrolled: a runtime index
        // into `out` would move it to local memory)
        const float* tr = P.aux_t + static_cast<size_t>(r) * P.ld_aux;
        float fa[16], fb[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = c0 + 4 * q;
            // (rows are padded to ld_aux >= round_up(cols, 4): a float4 starting
            // below cols stays inside the row; elements >= cols are dropped)
            const bool any = c < P.cols;
            const float4 lo = any && c < r ? __ldcg(reinterpret_cast<const float4*>(xr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 hi = any && c + 3 > r ? __ldcg(reinterpret_cast<const float4*>(tr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
            const float l4[4] = {lo.x, lo.y, lo.z, lo.w}, h4[4] = {hi.x, hi.y, hi.z, hi.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int cc = c + e;
                const bool in = cc < P.cols;
                const float dcc = in && cc > r ? __ldg(P.aux + static_cast<size_t>(cc) * P.ld_aux + cc) : 0.0f;
                fa[4 * q + e] = !in ? 0.0f : cc < r ? er.dg : cc > r ? dcc : er.dg;
                fb[4 * q + e] = !in ? 0.0f : cc < r ? l4[e] : cc > r ? h4[e] : er.dg;
            }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) out[j] = fmaf(fa[j], fb[j], out[j]);
    };
    if constexpr (kFmt == kOZ8) {
        if (!have_acc) {  // empty k-range
#pragma unroll 1
            for (int chunk = chunk_begin; chunk < chunk_end; ++chunk) {
                float out[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) out[j] = 0.0f;
                diag_fix(out, chunk);
                split_fix(out, chunk);
                finish(out, chunk);
            }
            return;
        }
#pragma unroll 1
        for (int chunk = chunk_begin; chunk < chunk_end; ++chunk) {
            __syncwarp();  // tcgen05.ld is .sync.aligned: re-converge first
            uint32_t raw[kDigits][16];
            if (chunk == chunk_begin + 1) PF_ESTAMP(6);
#pragma unroll
            for (int g = 0; g < kDigits; ++g) ptx::tmem_ld16_nowait(lane_base + g * kN + chunk * 16, raw[g]);
#pragma unroll
            for (int g = 0; g < kDigits; ++g) ptx::tmem_wait_ld_dep(raw[g]);
            if (chunk == chunk_begin + 1) PF_ESTAMP(7);
            if (chunk == chunk_begin) PF_ESTAMP(1);
            // accumulator g counts units of 2^-7(g+2) of 2^(e_a + e_b); the four
            // exact int32 sums are recombined smallest-first in fp32 (the result
            // is stored in fp32: ~1 ulp, no accumulation error)
            float out[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                // (the product's 2^-14 is folded into the digit weights: exact)
                float s = static_cast<float>(static_cast<int>(raw[3][j])) * 0x1p-35f;
                s = fmaf(static_cast<float>(static_cast<int>(raw[2][j])), 0x1p-28f, s);
                s = fmaf(static_cast<float>(static_cast<int>(raw[1][j])), 0x1p-21f, s);
                s = fmaf(static_cast<float>(static_cast<int>(raw[0][j])), 0x1p-14f, s);
                out[j] = (row_scale * col_scale[chunk * 16 + j]) * s;
            }
            diag_fix(out, chunk);
            split_fix(out, chunk);
            finish(out, chunk);
            if (chunk - chunk_begin < 4) PF_ESTAMP(2 + chunk - chunk_begin);
        }
    } else {
#pragma unroll 1
        for (int chunk = chunk_begin; chunk < chunk_end; ++chunk) {
            __syncwarp();
            float v[16];
            if (have_acc) {
                ptx::tmem_ld16(lane_base + chunk * 16, v);
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = 0.0f;
            }
            float out[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) out[j] = P.alpha * v[j];
            finish(out, chunk);
        }
    }
}

// kBF16 split-K epilogue (GemmBatch::k_split): every CTA of the cluster parks
// its partial tile in its idle stage buffers, then CTA `kslice` sums rows
// [kslice R, (kslice+1) R) over the cluster's CTAs in rank order (the same
// sum whichever CTA finished first) and runs the epilogue on them.
template <int kN, int kThreads>
__device__ __forceinline__ void split_k_epilogue(const GemmDesc& P, int tm, int tn, uint8_t* smem, uint32_t tmem,
                                                 int ks, int kslice, bool have_acc) {
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    constexpr int kRS = kN + 4;  // row stride (floats): float4 accesses by row-strided lanes conflict-free
    float* red = reinterpret_cast<float*>(smem);
    const int row = warp * 32 + static_cast<int>(lane);
#pragma unroll 1
    for (int chunk = 0; chunk < kN / 16; ++chunk) {
        __syncwarp();
        float v[16];
        if (have_acc) {
            ptx::tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + chunk * 16, v);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.0f;
        }
        float4* dst = reinterpret_cast<float4*>(red + row * kRS + chunk * 16);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    const int rows = kTile / ks;
    const uint32_t red_u32 = ptx::smem_u32(red);
#pragma unroll 1
    for (int w = threadIdx.x; w < rows * (kN / 16); w += kThreads) {
        const int rr = kslice * rows + w % rows, chunk = w / rows;  // lanes: consecutive rows
        const uint32_t off = static_cast<uint32_t>((rr * kRS + chunk * 16) * 4);
        float out[16];
#pragma unroll 1
        for (int q = 0; q < ks; ++q) {
            const uint32_t a = ptx::mapa(red_u32 + off, static_cast<uint32_t>(q));
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const float4 t = ptx::ld_dsmem4(a + 16 * h);
                if (q == 0) {
                    out[4 * h] = t.x;
                    out[4 * h + 1] = t.y;
                    out[4 * h + 2] = t.z;
                    out[4 * h + 3] = t.w;
                } else {
                    out[4 * h] += t.x;
                    out[4 * h + 1] += t.y;
                    out[4 * h + 2] += t.z;
                    out[4 * h + 3] += t.w;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) out[j] *= P.alpha;
        finish_chunk<kN>(P, tm, tn, tm * kTile + rr, chunk, out, nullptr);
    }
    ptx::cluster_sync();  // peers may still read this CTA's partial
}

template <int kFmt, int kN = 128, bool kSplit = false>
__global__ void __launch_bounds__(GemmTraits<kFmt, kN>::kThreads, GemmTraits<kFmt, kN>::kMinBlocks)
    umma_gemm_kernel(const __grid_constant__ GemmBatch batch) {
    using T = GemmTraits<kFmt, kN>;
    constexpr int kStages = T::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* tail = smem + kStages * T::kStageBytes + T::kCPad;
    uint64_t* full = reinterpret_cast<uint64_t*>(tail);
    uint64_t* empty = full + kStages;
    uint64_t* done = empty + kStages;
    uint64_t* cbar = done + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cbar + 1);
    float* col_scale = reinterpret_cast<float*>(tail + 256);  // kOZ8: 2^e_b per tile column

    // kBF16 split-K: the CTAs of one cluster share a tile, CTA rank = k-slice
    const int ks = kFmt == kBF16 && kN == kTile && batch.k_split > 1 ? batch.k_split : 1;
    const int gt = static_cast<int>(blockIdx.x) / ks;
    const int kslice = static_cast<int>(blockIdx.x) % ks;
    int p = 0, lt;
    if (batch.interleave) {
        p = gt % batch.n_probs;
        lt = gt / batch.n_probs;
    } else {
        while (p + 1 < batch.n_probs && batch.probs[p + 1].tile_begin <= gt) ++p;
        lt = gt - batch.probs[p].tile_begin;
    }
    const GemmDesc& P = batch.probs[p];
    int tm, tn;
    map_tile(P, lt, tm, tn);
    int k_begin = 0, k_end = P.k;
    if (P.k_mode == K_FROM_ROW_TILE) k_begin = tm * kTile;
    if (P.k_mode == K_FROM_COL_TILE) k_begin = tn * kTile;
    if (P.k_mode == K_TO_ROW_TILE_END) k_end = min(P.k, (tm + 1) * kTile);
    if (P.k_mode == K_TO_COL_TILE_END) k_end = min(P.k, (tn + 1) * kTile);
    int kb0 = k_begin / T::kKBlock;
    int kb1 = max(kb0, (k_end + T::kKBlock - 1) / T::kKBlock);
    if (ks > 1) {  // contiguous k-block slices, the last ones possibly shorter / empty
        const int per = (kb1 - kb0 + ks - 1) / ks;
        kb0 = min(kb1, kb0 + kslice * per);
        kb1 = min(kb1, kb0 + per);
    }

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    // short-K beta != 0 tiles read C into the idle last stage while the MMAs run
    const int c_cols = min(kN, P.cols - tn * kN);
    const bool cpre = kFmt == kOZ8 && P.beta != 0.0f && kb1 - kb0 <= kStages - 1 && (P.flags & EPI_VEC4) &&
                      !(P.flags & EPI_TRANSPOSE) && c_cols > 0 && (c_cols & 3) == 0;
    float* cbuf = reinterpret_cast<float*>(smem + (kStages - 1) * T::kStageBytes);

#ifdef PF_GEMM_PROBE
    const bool probe_on = blockIdx.x == 0 && P.beta != 0.0f && P.rows <= kTile && P.cols <= kTile;
#endif
    PF_GSTAMP(0, threadIdx.x == 0);
    // prologue (overlaps the previous kernel's tail under PDL)
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(done, 1);
        ptx::mbar_init(cbar, kTile);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<T::kTmemCols>(tmem_slot);
    if (warp == 0 && lane == 0) {  // one map per operand (kOZ8: 3-D, all digit planes)
        ptx::prefetch_tmap(&batch.maps[P.a_map]);
        ptx::prefetch_tmap(&batch.maps[P.b_map]);
    }
    ptx::grid_dep_wait();  // operands, scales and C come from earlier launches
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    PF_GSTAMP(1, threadIdx.x == 0);
    if (cpre && threadIdx.x >= 64 && threadIdx.x < 64 + kTile) {  // warps 2-5: one C row each
        const int t = static_cast<int>(threadIdx.x) - 64;
        const int r = tm * kTile + t;
        if (r < P.rows) {
            const uint32_t bytes = static_cast<uint32_t>(c_cols) * 4u;
            ptx::mbar_arrive_expect_tx(cbar, bytes);
            ptx::bulk_load(cbuf + t * T::kCStride, P.c + static_cast<size_t>(r) * P.ldc + tn * kN, bytes, cbar);
        } else {
            ptx::mbar_arrive(cbar);
        }
    }

    auto a_plane = [&](int s, int pl) { return smem + s * T::kStageBytes + pl * T::kPlaneBytes; };
    auto b_plane = [&](int s, int pl) {
        return smem + s * T::kStageBytes + T::kPlanes * T::kPlaneBytes + pl * T::kPlaneBytesB;
    };

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer
        int s = 0;
        uint32_t ph = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(&empty[s], ph ^ 1u);
            ptx::mbar_arrive_expect_tx(&full[s], T::kStageBytes);
            const int kc = kb * T::kKBlock;
            if constexpr (kFmt == kOZ8) {
                ptx::tma_load_3d(a_plane(s, 0), &batch.maps[P.a_map], &full[s], kc, tm * kTile, 0);
                ptx::tma_load_3d(b_plane(s, 0), &batch.maps[P.b_map], &full[s], kc, tn * kN, 0);
            } else if (P.mn_major) {
                // box {64 features, 64 tokens} per 64-feature group: [group][token][64 features]
                ptx::tma_load_2d(a_plane(s, 0), &batch.maps[P.a_map], &full[s], tm * kTile, kc);
                ptx::tma_load_2d(a_plane(s, 0) + kMnGroupBytes, &batch.maps[P.a_map], &full[s], tm * kTile + 64, kc);
#pragma unroll
                for (int h = 0; h < kN / 64; ++h)
                    ptx::tma_load_2d(b_plane(s, 0) + h * kMnGroupBytes, &batch.maps[P.b_map], &full[s], tn * kN + 64 * h, kc);
            } else {
                // box {64 elements, 128 rows}; a 256-row B tile is two boxes
                ptx::tma_load_2d(a_plane(s, 0), &batch.maps[P.a_map], &full[s], kc, tm * kTile);
#pragma unroll
                for (int h = 0; h < (kN + kTile - 1) / kTile; ++h)
                    ptx::tma_load_2d(b_plane(s, 0) + h * kTile * 128, &batch.maps[P.b_map], &full[s], kc, tn * kN + kTile * h);
            }
            if (++s == kStages) {
                s = 0;
                ph ^= 1u;
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer (single thread)
        int s = 0;
        uint32_t ph = 0;
        uint32_t started = 0;  // bit g: accumulator g has been initialised
        for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(&full[s], ph);
            ptx::tc_fence_after();
            PF_GSTAMP(2, kb == kb0);
#pragma unroll
            for (int ks = 0; ks < T::kKSteps; ++ks) {
                const uint32_t off = ks * 32;  // 32 B per UMMA k-step
                if constexpr (kFmt == kOZ8) {
                    uint64_t da[kDigits], db[kDigits];
#pragma unroll
                    for (int q = 0; q < kDigits; ++q) {
                        da[q] = ptx::sw64_kmajor_desc(ptx::smem_u32(a_plane(s, q)) + off);
                        db[q] = ptx::sw64_kmajor_desc(ptx::smem_u32(b_plane(s, q)) + off);
                    }
                    ptx::umma_i8_digits(tmem, tmem + kN, tmem + 2 * kN, tmem + 3 * kN, da, db, T::kIdesc, started);
                    started = 0xFu;
                } else if (P.mn_major) {
                    // 16 K rows per UMMA = two 8-row groups of 1024 B
                    const uint32_t moff = ks * 2048;
                    ptx::umma_f16(tmem,
                                  ptx::sw128_mnmajor_desc(ptx::smem_u32(a_plane(s, 0)) + moff, kMnGroupBytes, 1024),
                                  ptx::sw128_mnmajor_desc(ptx::smem_u32(b_plane(s, 0)) + moff, kMnGroupBytes, 1024),
                                  T::kIdesc | ptx::kIdescAMnMajor | ptx::kIdescBMnMajor, started);
                    started = 1;
                } else {
                    ptx::umma_f16(tmem, ptx::sw128_kmajor_desc(ptx::smem_u32(a_plane(s, 0)) + off),
                                  ptx::sw128_kmajor_desc(ptx::smem_u32(b_plane(s, 0)) + off),
                                  T::kIdesc, started);
                    started = 1;
                }
            }
            ptx::umma_commit(&empty[s]);  // slot free once these MMAs retire
            if (++s == kStages) {
                s = 0;
                ph ^= 1u;
            }
        }
        ptx::umma_commit(done);
        PF_GSTAMP(3, true);
    }
    __syncwarp();
    if constexpr (kFmt == kOZ8) {  // warps 2-5: column scales while the MMAs run
        const int t = static_cast<int>(threadIdx.x) - 64;
        if (t >= 0 && t < kN) {
            const int c = tn * kN + t;
            col_scale[t] = c < P.cols ? ptx::pow2f(__ldcg(P.b_exp + c)) : 0.0f;
        }
        __syncthreads();
    }

    // ---------------- epilogue: TMEM -> registers -> global
    const EpiRow er = epi_row<kFmt, kN, kSplit>(P, tm, tn, tm * kTile + (warp & 3) * 32 + static_cast<int>(lane));
    const bool have_acc = kb1 > kb0;
    if (have_acc) {
        ptx::mbar_wait(done, 0);
        ptx::tc_fence_after();
    }
    PF_GSTAMP(4, threadIdx.x == 0);
    ptx::grid_dep_launch();  // main loop done: let the next launch start its prologue
    if (cpre) ptx::mbar_wait(cbar, 0);
    __syncwarp();
    bool split_k = false;
    if constexpr (kFmt == kBF16 && kN == kTile) {
        static_assert(kTile * (kN + 4) * 4 <= kStages * T::kStageBytes, "split-K tile does not fit the stages");
        if (ks > 1) {
            split_k_epilogue<kN, T::kThreads>(P, tm, tn, smem, tmem, ks, kslice, have_acc);
            split_k = true;
        }
    }
    if (!split_k) {
        constexpr int kPairs = T::kThreads / 128;  // warps sharing a TMEM lane quarter
        const int ew = warp & 3, part = warp >> 2;
        constexpr int kChunks = kN / 16 / kPairs;
        epilogue_chunks<kFmt, kN, kSplit>(P, tm, tn, tmem + (static_cast<uint32_t>(ew * 32) << 16),
                              tm * kTile + ew * 32 + static_cast<int>(lane), col_scale, part * kChunks,
                              (part + 1) * kChunks, have_acc, er,
                              cpre ? cbuf + (ew * 32 + static_cast<int>(lane)) * T::kCStride : nullptr);
    }

    PF_GSTAMP(5, threadIdx.x == 0);
    ptx::tc_fence_before();
    __syncthreads();
#ifdef PF_GEMM_PROBE
    if (probe_on && threadIdx.x == 0) {
        const int slot = atomicAdd(&g_gemm_probe_n, 1);
        if (slot < 64) {
            const long long* st = reinterpret_cast<const long long*>(tail + 128);
            for (int i = 0; i < 6; ++i) g_gemm_probe[slot * 16 + i] = st[i];
            for (int i = 0; i < 8; ++i) g_gemm_probe[slot * 16 + 6 + i] = g_gemm_probe_epi[i];
            g_gemm_probe[slot * 16 + 14] = P.rows;
            g_gemm_probe[slot * 16 + 15] = P.cols;
        }
    }
#endif
    if (warp == 0) ptx::tmem_dealloc<T::kTmemCols>(tmem);
}

// ---------------------------------------------------------------------------
// Persistent form for long-K kOZ8 launches with more tiles than SMs: one CTA
// per SM pulls tiles from an atomic ticket counter (dynamic balance for
// unequal tiles: triangular k-ranges, mixed K).  Warp 0 lane 0 fetches the
// next tile and keeps the TMA ring running into it while warps 2-9 run the
// current tile's epilogue; warp 1 lane 0 starts the next tile's MMAs once the
// epilogue warps have drained the accumulators (tmem_empty).  Tile ids reach
// the MMA and epilogue warps through a 4-entry shared-memory queue.  The last
// CTA to finish resets its launch's counter slot (slots rotate per launch).
constexpr int kPersistThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
// slots [0, kEagerSlots) rotate over eager launches, the rest are handed out
// once each to launches captured into CUDA graphs (kfac_ops.cu ticket_slot)
constexpr int kEagerSlots = 512;
constexpr int kTicketSlots = kEagerSlots + 7680;
__device__ unsigned int g_tickets[kTicketSlots * 2];  // {next tile, CTAs done} per slot

__device__ __forceinline__ void tile_of(const GemmBatch& batch, int gt, int& p, int& tm, int& tn, int& kb0,
                                        int& kb1) {
    int lt;
    p = 0;
    if (batch.interleave) {
        p = gt % batch.n_probs;
        lt = gt / batch.n_probs;
    } else {
        while (p + 1 < batch.n_probs && batch.probs[p + 1].tile_begin <= gt) ++p;
        lt = gt - batch.probs[p].tile_begin;
    }
    const GemmDesc& P = batch.probs[p];
    map_tile(P, lt, tm, tn);
    int k_begin = 0, k_end = P.k;
    if (P.k_mode == K_FROM_ROW_TILE) k_begin = tm * kTile;
    if (P.k_mode == K_FROM_COL_TILE) k_begin = tn * kTile;
    if (P.k_mode == K_TO_ROW_TILE_END) k_end = min(P.k, (tm + 1) * kTile);
    if (P.k_mode == K_TO_COL_TILE_END) k_end = min(P.k, (tn + 1) * kTile);
    constexpr int kKB = GemmTraits<kOZ8>::kKBlock;
    kb0 = k_begin / kKB;
    kb1 = max(kb0, (k_end + kKB - 1) / kKB);
}

template <bool kSplit = false>
__global__ void __launch_bounds__(kPersistThreads, 1)
    umma_gemm_persist_kernel(const __grid_constant__ GemmBatch batch, int slot) {
    using T = GemmTraits<kOZ8>;
    constexpr int kStages = T::kStages;
    constexpr int kQ = 4;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* tail = smem + kStages * T::kStageBytes + T::kCPad;
    uint64_t* full = reinterpret_cast<uint64_t*>(tail);
    uint64_t* empty = full + kStages;
    uint64_t* done = empty + kStages;
    uint64_t* tmem_empty = done + 1;
    uint64_t* tq_full = tmem_empty + 1;
    uint64_t* tq_empty = tq_full + kQ;
    int* tq = reinterpret_cast<int*>(tq_empty + kQ);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + kQ);
    float* col_scale = reinterpret_cast<float*>(tail + 256);
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(done, 1);
        ptx::mbar_init(tmem_empty, 8);  // one arrive per epilogue warp
        for (int q = 0; q < kQ; ++q) {
            ptx::mbar_init(&tq_full[q], 1);
            ptx::mbar_init(&tq_empty[q], 9);  // MMA thread + 8 epilogue warps
        }
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<T::kTmemCols>(tmem_slot);
    ptx::grid_dep_wait();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto a_plane = [&](int s, int pl) { return smem + s * T::kStageBytes + pl * T::kPlaneBytes; };
    auto b_plane = [&](int s, int pl) {
        return smem + s * T::kStageBytes + T::kPlanes * T::kPlaneBytes + pl * T::kPlaneBytesB;
    };
    const int total = batch.total_tiles;
    unsigned int* ctr = g_tickets + 2 * slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- tile fetch + TMA producer
            int s = 0;
            uint32_t ph = 0;
            for (int it = 0;; ++it) {
                const int q = it % kQ;
                ptx::mbar_wait(&tq_empty[q], ((it / kQ) & 1) ^ 1u);
                const unsigned int t = atomicAdd(ctr, 1u);
                const int gt = t < static_cast<unsigned int>(total) ? static_cast<int>(t) : -1;
                tq[q] = gt;
                ptx::mbar_arrive(&tq_full[q]);
                if (gt < 0) break;
                int p, tm, tn, kb0, kb1;
                tile_of(batch, gt, p, tm, tn, kb0, kb1);
                const GemmDesc& P = batch.probs[p];
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&empty[s], ph ^ 1u);
                    ptx::mbar_arrive_expect_tx(&full[s], T::kStageBytes);
                    const int kc = kb * T::kKBlock;
                    ptx::tma_load_3d(a_plane(s, 0), &batch.maps[P.a_map], &full[s], kc, tm * kTile, 0);
                    ptx::tma_load_3d(b_plane(s, 0), &batch.maps[P.b_map], &full[s], kc, tn * kTile, 0);
                    if (++s == kStages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
            // every CTA has fetched its terminal ticket when the count reaches
            // gridDim.x: the last one resets the slot for a later launch (the
            // fence orders this CTA's ticket fetches before its done count)
            __threadfence();
            if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
                __threadfence();
                atomicExch(ctr, 0u);
                atomicExch(ctr + 1, 0u);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            int s = 0;
            uint32_t ph = 0;
            for (int it = 0;; ++it) {
                const int q = it % kQ;
                ptx::mbar_wait(&tq_full[q], (it / kQ) & 1);
                const int gt = tq[q];
                ptx::mbar_arrive(&tq_empty[q]);
                if (gt < 0) break;
                int p, tm, tn, kb0, kb1;
                tile_of(batch, gt, p, tm, tn, kb0, kb1);
                if (it > 0) {  // accumulators drained by the previous tile's epilogue
                    ptx::mbar_wait(tmem_empty, (it - 1) & 1);
                    ptx::tc_fence_after();
                }
                uint32_t started = 0;
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&full[s], ph);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int ks = 0; ks < T::kKSteps; ++ks) {
                        const uint32_t off = ks * 32;
                        uint64_t da[kDigits], db[kDigits];
#pragma unroll
                        for (int q = 0; q < kDigits; ++q) {
                            da[q] = ptx::sw64_kmajor_desc(ptx::smem_u32(a_plane(s, q)) + off);
                            db[q] = ptx::sw64_kmajor_desc(ptx::smem_u32(b_plane(s, q)) + off);
                        }
                        ptx::umma_i8_digits(tmem, tmem + kTile, tmem + 2 * kTile, tmem + 3 * kTile, da, db, T::kIdesc,
                                            started);
                        started = 0xFu;
                    }
                    ptx::umma_commit(&empty[s]);
                    if (++s == kStages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                ptx::umma_commit(done);  // also fires at once for an empty k-range
            }
        }
    } else {  // ---------------- epilogue warps 2-9
        const int ew = warp & 3;           // TMEM lane quarter this warp may access
        const int part = (warp - 2) >> 2;  // column half
        const int et = static_cast<int>(threadIdx.x) - 64;
        for (int it = 0;; ++it) {
            const int q = it % kQ;
            ptx::mbar_wait(&tq_full[q], (it / kQ) & 1);
            const int gt = tq[q];
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tq_empty[q]);
            if (gt < 0) break;
            int p, tm, tn, kb0, kb1;
            tile_of(batch, gt, p, tm, tn, kb0, kb1);
            const GemmDesc& P = batch.probs[p];
            asm volatile("bar.sync 1, 256;" ::: "memory");  // previous tile's col_scale readers done
            if (et < kTile) {
                const int c = tn * kTile + et;
                col_scale[et] = c < P.cols ? ptx::pow2f(__ldcg(P.b_exp + c)) : 0.0f;
            }
            const int r = tm * kTile + ew * 32 + static_cast<int>(lane);
            if (P.beta != 0.0f && r < P.rows && !(P.flags & EPI_TRANSPOSE)) {
                // C (e.g. the weights of W -= eta P) is read only after this
                // tile's MMAs: pull this thread's row segment into L2 now
                const int c0 = tn * kTile + part * (kTile / 2);
                if (c0 < P.cols) {
                    const float* row = P.c + static_cast<size_t>(r) * P.ldc + c0;
                    const int n = min(kTile / 2, P.cols - c0);
#pragma unroll
                    for (int j = 0; j < kTile / 2; j += 32)
                        if (j < n) ptx::prefetch_l2(row + j);
                }
            }
            const EpiRow er = epi_row<kOZ8, kTile, kSplit>(P, tm, tn, r);
            asm volatile("bar.sync 1, 256;" ::: "memory");
            ptx::mbar_wait(done, it & 1);
            ptx::tc_fence_after();
            __syncwarp();
            constexpr int kChunks = kTile / 16 / 2;
            epilogue_chunks<kOZ8, kTile, kSplit>(P, tm, tn, tmem + (static_cast<uint32_t>(ew * 32) << 16), r, col_scale,
                                  part * kChunks, (part + 1) * kChunks, kb1 > kb0, er);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tmem_empty);
        }
    }
    ptx::grid_dep_launch();
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<T::kTmemCols>(tmem);
}

}  // namespace pf
