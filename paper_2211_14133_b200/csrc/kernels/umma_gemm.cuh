// Grouped "TN" tensor-core GEMM for sm_100a: C = alpha * A * B^T (+ beta * C)
// with A [rows x k] and B [cols x k] both K-major (K contiguous).  One kernel
// serves every K-FAC hot op:
//
//   * curvature SYRK   A = B = X (bf16 [d x n_tokens]),  lower tiles only,
//                      mirrored store -> full symmetric fp32 factor;
//   * damped inverse   trailing updates / triangular products in 3xTF32
//                      (fp32-accurate: hi*hi + hi*lo + lo*hi);
//   * precondition     U^T = A^-1 G^T, P = B^-1 U  (3xTF32) with the fused
//                      weight-update epilogue W -= eta * P.
//
// Structure (per CTA = one 128x128 output tile, 4 warps):
//   warp 0 / lane 0 : TMA producer, STAGES-deep smem ring (full/empty mbarriers)
//   warp 1 / lane 0 : tcgen05.mma issuer, accumulator in TMEM (128 lanes x 128 cols)
//   all 4 warps     : epilogue, tcgen05.ld 32x32b -> registers -> global
// Operand tiles are 128 rows x 128 B, TMA SWIZZLE_128B, so each k-block is
// 64 bf16 or 32 fp32 elements and is consumed by 4 UMMA k-steps of 32 B.
#pragma once

#include <cuda.h>
#include <cstdint>

#include "ptx.cuh"

namespace pf {

constexpr int kTile = 128;            // output tile edge (M = N = 128)
constexpr int kTileBytes = 128 * 128; // one operand plane per stage: 128 rows x 128 B
constexpr int kMaxMaps = 64;
constexpr int kMaxProbs = 16;

enum EpiFlag : uint32_t {
    EPI_MIRROR = 1u,        // off-diagonal tiles also stored transposed (symmetric result)
    EPI_TRANSPOSE = 2u,     // store C^T (into c) instead of C
    EPI_SPLIT = 4u,         // store hi=tf32(v) to c, lo=tf32(v-hi) to c_lo
    EPI_READ_SPLIT = 8u,    // old value = c + c_lo (when beta != 0)
    EPI_ALSO_T = 16u,       // additionally store C^T into c_t (+ c_t_lo if SPLIT)
    EPI_VEC4 = 32u,         // c / ldc 16-byte aligned: vectorised row stores
};

// k_mode: which slice of the reduction a tile needs (triangular operands).
// Tile (tm, tn) reads only the k-slice where both triangular operands can be
// non-zero; the rest of the slice is never touched (no zero-fill needed).
enum KMode : int {
    K_FULL = 0,
    K_FROM_ROW_TILE = 1,    // k in [tm*128, k)
    K_FROM_COL_TILE = 2,    // k in [tn*128, k)
    K_TO_ROW_TILE_END = 3,  // k in [0, (tm+1)*128)
    K_TO_COL_TILE_END = 4,  // k in [0, (tn+1)*128)
};

struct GemmDesc {
    int a_map, b_map;    // index of plane 0's CUtensorMap (plane 1 = +1)
    int rows, cols, k;   // output rows (A rows), output cols (B rows), reduction length
    int tiles_m, tiles_n;
    int lower;           // enumerate only tiles with tm >= tn
    int tile_begin;      // first global tile index of this problem
    int k_mode;
    float alpha, beta;
    uint32_t flags;
    float* c;
    float* c_lo;
    float* c_t;
    float* c_t_lo;
    int ldc, ldc_t;
};

struct GemmBatch {
    CUtensorMap maps[kMaxMaps];
    GemmDesc probs[kMaxProbs];
    int n_probs;
    int total_tiles;
};

template <int kFmt, int kPlanes, int kStages>
struct GemmTraits {
    static constexpr int kStageBytes = 2 * kPlanes * kTileBytes;
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int kKBlock = kFmt == 1 ? 64 : 32;  // elements per 128-B row
    static constexpr uint32_t kIdesc = ptx::make_idesc(kFmt, 128, 128);
};

__device__ __forceinline__ void decode_lower(int t, int& tm, int& tn) {
    int m = static_cast<int>((sqrtf(8.0f * static_cast<float>(t) + 1.0f) - 1.0f) * 0.5f);
    while ((m + 1) * (m + 2) / 2 <= t) ++m;
    while (m * (m + 1) / 2 > t) --m;
    tm = m;
    tn = t - m * (m + 1) / 2;
}

__device__ __forceinline__ void put(float* hi, float* lo, size_t idx, float v, bool split) {
    if (split) {
        const float h = ptx::tf32_round(v);
        hi[idx] = h;
        lo[idx] = ptx::tf32_round(v - h);
    } else {
        hi[idx] = v;
    }
}

template <int kFmt, int kPlanes, int kStages>
__global__ void __launch_bounds__(128, (kPlanes == 1 ? 2 : 1))
    umma_gemm_kernel(const __grid_constant__ GemmBatch batch) {
    using T = GemmTraits<kFmt, kPlanes, kStages>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * T::kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* done = empty + kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    // ---- which problem / tile
    const int gt = blockIdx.x;
    int p = 0;
    while (p + 1 < batch.n_probs && batch.probs[p + 1].tile_begin <= gt) ++p;
    const GemmDesc& P = batch.probs[p];
    const int lt = gt - P.tile_begin;
    int tm, tn;
    if (P.lower) {
        decode_lower(lt, tm, tn);
    } else {
        tm = lt / P.tiles_n;
        tn = lt % P.tiles_n;
    }
    int k_begin = 0, k_end = P.k;
    if (P.k_mode == K_FROM_ROW_TILE) k_begin = tm * kTile;
    if (P.k_mode == K_FROM_COL_TILE) k_begin = tn * kTile;
    if (P.k_mode == K_TO_ROW_TILE_END) k_end = min(P.k, (tm + 1) * kTile);
    if (P.k_mode == K_TO_COL_TILE_END) k_end = min(P.k, (tn + 1) * kTile);
    const int kb0 = k_begin / T::kKBlock;
    const int kb1 = (k_end + T::kKBlock - 1) / T::kKBlock;

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(done, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<128>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto a_plane = [&](int s, int pl) { return smem + s * T::kStageBytes + pl * kTileBytes; };
    auto b_plane = [&](int s, int pl) {
        return smem + s * T::kStageBytes + (kPlanes + pl) * kTileBytes;
    };

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer
        for (int pl = 0; pl < kPlanes; ++pl) {
            ptx::prefetch_tmap(&batch.maps[P.a_map + pl]);
            ptx::prefetch_tmap(&batch.maps[P.b_map + pl]);
        }
        int s = 0;
        uint32_t ph = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(&empty[s], ph ^ 1u);
            ptx::mbar_arrive_expect_tx(&full[s], T::kStageBytes);
            const int kc = kb * T::kKBlock;
            for (int pl = 0; pl < kPlanes; ++pl) {
                ptx::tma_load_2d(a_plane(s, pl), &batch.maps[P.a_map + pl], &full[s], kc,
                                 tm * kTile);
                ptx::tma_load_2d(b_plane(s, pl), &batch.maps[P.b_map + pl], &full[s], kc,
                                 tn * kTile);
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
        uint32_t acc = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(&full[s], ph);
            ptx::tc_fence_after();
            const uint32_t a0 = ptx::smem_u32(a_plane(s, 0));
            const uint32_t b0 = ptx::smem_u32(b_plane(s, 0));
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint32_t off = ks * 32;  // 32 B per UMMA k-step
                if constexpr (kPlanes == 1) {
                    ptx::umma_f16(tmem, ptx::sw128_kmajor_desc(a0 + off),
                                  ptx::sw128_kmajor_desc(b0 + off), T::kIdesc, acc);
                    acc = 1;
                } else {
                    const uint32_t a1 = a0 + kTileBytes;
                    const uint32_t b1 = b0 + kTileBytes;
                    // small cross terms first, then the dominant hi*hi product
                    ptx::umma_tf32(tmem, ptx::sw128_kmajor_desc(a0 + off),
                                   ptx::sw128_kmajor_desc(b1 + off), T::kIdesc, acc);
                    acc = 1;
                    ptx::umma_tf32(tmem, ptx::sw128_kmajor_desc(a1 + off),
                                   ptx::sw128_kmajor_desc(b0 + off), T::kIdesc, acc);
                    ptx::umma_tf32(tmem, ptx::sw128_kmajor_desc(a0 + off),
                                   ptx::sw128_kmajor_desc(b0 + off), T::kIdesc, acc);
                }
            }
            ptx::umma_commit(&empty[s]);  // slot free once these MMAs retire
            if (++s == kStages) {
                s = 0;
                ph ^= 1u;
            }
        }
        ptx::umma_commit(done);
    }
    __syncwarp();

    // ---------------- epilogue: TMEM -> registers -> global
    const bool have_acc = kb1 > kb0;
    if (have_acc) {
        ptx::mbar_wait(done, 0);
        ptx::tc_fence_after();
    }
    __syncwarp();
    const int r = tm * kTile + warp * 32 + static_cast<int>(lane);
    const bool row_ok = r < P.rows;
    const uint32_t f = P.flags;
    const bool mirror = (f & EPI_MIRROR) && tm != tn;
#pragma unroll 1
    for (int chunk = 0; chunk < kTile / 16; ++chunk) {
        __syncwarp();  // tcgen05.ld is .sync.aligned: re-converge first
        float v[16];
        if (have_acc) {
            ptx::tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + chunk * 16, v);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.0f;
        }
        const int c0 = tn * kTile + chunk * 16;
        if (!row_ok || c0 >= P.cols) continue;
        float out[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) out[j] = P.alpha * v[j];
        if (P.beta != 0.0f) {
            // old value from the (row-major or transposed) destination
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int c = c0 + j;
                if (c >= P.cols) break;
                const size_t idx = (f & EPI_TRANSPOSE) ? static_cast<size_t>(c) * P.ldc + r
                                                       : static_cast<size_t>(r) * P.ldc + c;
                float old = P.c[idx];
                if (f & EPI_READ_SPLIT) old += P.c_lo[idx];
                out[j] += P.beta * old;
            }
        }
        const bool full_chunk = c0 + 16 <= P.cols;
        const bool split = (f & EPI_SPLIT) != 0;
        if ((f & EPI_VEC4) && full_chunk && !(f & (EPI_TRANSPOSE | EPI_SPLIT))) {
            float4* dst = reinterpret_cast<float4*>(P.c + static_cast<size_t>(r) * P.ldc + c0);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                dst[q] = make_float4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
        } else if (f & EPI_TRANSPOSE) {
            // lanes hold consecutive rows -> each transposed column store is coalesced
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j < P.cols)
                    put(P.c, P.c_lo, static_cast<size_t>(c0 + j) * P.ldc + r, out[j], split);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j < P.cols)
                    put(P.c, P.c_lo, static_cast<size_t>(r) * P.ldc + c0 + j, out[j], split);
        }
        if (mirror) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j < P.cols)
                    put(P.c, P.c_lo, static_cast<size_t>(c0 + j) * P.ldc + r, out[j], split);
        }
        if (f & EPI_ALSO_T) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j < P.cols)
                    put(P.c_t, P.c_t_lo, static_cast<size_t>(c0 + j) * P.ldc_t + r, out[j], split);
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<128>(tmem);
}

}  // namespace pf
