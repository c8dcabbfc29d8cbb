// Persistent task-graph kernel for the damped inverse.
//
// The recursive blocked Cholesky + triangular inverse (kfac_ops.cu,
// inverse_rec) is a long chain of small dependent steps: for d = 4096 about
// 280 sequential launches (leaves, digit slicing, digit GEMMs), each paying a
// launch gap plus its own prologue (TMEM allocation, barrier setup, descriptor
// fetch).  Here the whole inversion of a batch of factors is ONE launch: one
// CTA per SM (256 threads, ~205 KB shared memory, all 512 TMEM columns
// allocated once) pulls tasks from a host-built list in topological order:
//
//   GT_DAMP   8 rows of  A = M + lambda I                (resets info)
//   GT_SLICE  8 rows of one digit-slicing job             (slice.cuh)
//   GT_LEAF   one 128x128 diagonal block                  (leaf.cuh)
//   GT_GEMM   one 128x128 output tile of a digit GEMM     (umma_gemm.cuh)
//
// Every task belongs to a phase (= one launch of the stream-ordered path);
// a task waits until its predecessor phase has completed (counter reaches the
// phase size, acquire at gpu scope) and bumps its own phase counter when done
// (release).  Phases of independent factor groups (the d=4096 and d=1024
// factors of a layer) are interleaved so their chains overlap.  Tasks are
// claimed in list order and only ever wait on lower-indexed tasks, so the
// lowest unfinished task can always run: no co-residency assumption.
//
// Memory-model notes: producers write with generic st.global; consumers read
// with ld.global.cg (L1 bypass) or TMA.  The claiming thread issues
// fence.proxy.async after its acquire so TMA (async proxy) observes the
// generic writes; leaf tasks fence their generic shared-memory writes before
// the TMA ring reuses that memory.  The GEMM ring's full/empty/done barrier
// phases persist across tiles (no re-initialisation).
#pragma once

#include <cstdint>

#include "leaf.cuh"
#include "ptx.cuh"
#include "slice.cuh"
#include "umma_gemm.cuh"

namespace pf {

struct Damp2D {
    const float* src;
    float* dst;
    int* info;  // reset to 0 (success) before the factorisation
    int d, ld_src, ld_dst;
    float damping;
};

enum GraphTaskType : int { GT_DAMP = 0, GT_SLICE = 1, GT_LEAF = 2, GT_GEMM = 3 };

struct GraphTask {
    int type;
    int phase;  // counter bumped on completion
    int wait;   // phase that must be complete first (-1: none)
    int a;      // DAMP / SLICE: job, LEAF: leaf, GEMM: descriptor
    int b;      // DAMP / SLICE: first row, GEMM: local tile index
};

struct GraphProgram {
    const GraphTask* tasks;
    int n_tasks;
    const int* phase_size;
    int* phase_done;  // zeroed before every launch
    int* cursor;      // zeroed before every launch
    const GemmDesc* gemms;
    const CUtensorMap* maps;  // 64-byte aligned, global memory
    const SliceJob* slices;
    const LeafArgs* leaves;
    const Damp2D* damps;
    unsigned long long* trace;  // nullable: per task {claimed, ready, done} globaltimer ns + SM id
};

constexpr int kGraphThreads = 256;
constexpr int kGraphRows = 8;  // rows per DAMP / SLICE task (one per warp)
using GOZ = GemmTraits<kOZ8>;
constexpr int kGraphRing = GOZ::kStages * GOZ::kStageBytes;
constexpr int kGraphWork = ((kGraphRing > kLeafSmemBytes ? kGraphRing : kLeafSmemBytes) + 1023) / 1024 * 1024;
constexpr int kGraphSmemBytes = 1024 + kGraphWork + 256 + 4 * kTile;

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// rows [r0, r0 + kGraphRows) of dst = src + damping I (lower triangle incl. diagonal)
__device__ __noinline__ void damp_rows(const Damp2D& s, int r0) {
    if (r0 == 0 && threadIdx.x == 0) *s.info = 0;
    const int r1 = min(s.d, r0 + kGraphRows);
    for (int r = r0 + (threadIdx.x >> 5); r < r1; r += kGraphThreads / 32)
        for (int c = threadIdx.x & 31; c <= r; c += 32) {
            float v = __ldcg(s.src + static_cast<int64_t>(r) * s.ld_src + c);
            if (r == c) v += s.damping;
            s.dst[static_cast<int64_t>(r) * s.ld_dst + c] = v;
        }
}

// One 128x128 tile of a digit GEMM, all 256 threads: thread 0 = TMA producer,
// thread 32 = MMA issuer (persistent ring state), then warps w and w+4 share
// TMEM lanes 32(w%4).. and split the 8 column chunks.
struct RingState {
    int prod_s = 0;
    uint32_t prod_ph = 0;
    int mma_s = 0;
    uint32_t mma_ph = 0;
    uint32_t done_ph = 0;
};

__device__ __noinline__ void graph_gemm_tile(const GraphProgram& g, int di, int lt, uint8_t* ring,
                                                uint64_t* full, uint64_t* empty, uint64_t* done,
                                                float* col_scale, uint32_t tmem, RingState& st,
                                                unsigned long long* tr) {
    using T = GOZ;
    const GemmDesc P = g.gemms[di];  // by value: stores below must not force reloads
    int tm, tn;
    map_tile(P, lt, tm, tn);
    int k_begin = 0, k_end = P.k;
    if (P.k_mode == K_FROM_ROW_TILE) k_begin = tm * kTile;
    if (P.k_mode == K_FROM_COL_TILE) k_begin = tn * kTile;
    if (P.k_mode == K_TO_ROW_TILE_END) k_end = min(P.k, (tm + 1) * kTile);
    if (P.k_mode == K_TO_COL_TILE_END) k_end = min(P.k, (tn + 1) * kTile);
    const int kb0 = k_begin / T::kKBlock;
    const int kb1 = max(kb0, (k_end + T::kKBlock - 1) / T::kKBlock);
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t lane = tid & 31;
    auto a_plane = [&](int s, int pl) { return ring + s * T::kStageBytes + pl * T::kPlaneBytes; };
    auto b_plane = [&](int s, int pl) { return ring + s * T::kStageBytes + (T::kPlanes + pl) * T::kPlaneBytes; };

    if (tid == 0) {
        const CUtensorMap* am = g.maps + P.a_map;
        const CUtensorMap* bm = g.maps + P.b_map;
        for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(&empty[st.prod_s], st.prod_ph ^ 1u);
            ptx::mbar_arrive_expect_tx(&full[st.prod_s], T::kStageBytes);
            const int kc = kb * T::kKBlock;
            ptx::tma_load_3d(a_plane(st.prod_s, 0), am, &full[st.prod_s], kc, tm * kTile, 0);
            ptx::tma_load_3d(b_plane(st.prod_s, 0), bm, &full[st.prod_s], kc, tn * kTile, 0);
            if (++st.prod_s == T::kStages) {
                st.prod_s = 0;
                st.prod_ph ^= 1u;
            }
        }
    } else if (tid == 32) {
        uint32_t started = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(&full[st.mma_s], st.mma_ph);
            ptx::tc_fence_after();
#pragma unroll
            for (int ks = 0; ks < T::kKSteps; ++ks) {
                const uint32_t off = ks * 32;
#pragma unroll
                for (int gg = 0; gg < kDigits; ++gg) {
#pragma unroll
                    for (int sa = 0; sa <= gg; ++sa) {
                        const int sb = gg - sa;
                        const uint64_t da = ptx::sw64_kmajor_desc(ptx::smem_u32(a_plane(st.mma_s, sa)) + off);
                        const uint64_t db = ptx::sw64_kmajor_desc(ptx::smem_u32(b_plane(st.mma_s, sb)) + off);
                        ptx::umma_i8(tmem + gg * 128, da, db, T::kIdesc, (started >> gg) & 1u);
                        started |= 1u << gg;
                    }
                }
            }
            ptx::umma_commit(&empty[st.mma_s]);
            if (++st.mma_s == T::kStages) {
                st.mma_s = 0;
                st.mma_ph ^= 1u;
            }
        }
        ptx::umma_commit(done);  // arrives at once if no MMA was issued
    }
    __syncwarp();
    if (tid >= 64 && tid < 64 + kTile) {  // warps 2-5: column scales while the MMAs run
        const int c = tn * kTile + tid - 64;
        col_scale[tid - 64] = c < P.cols ? ptx::pow2f(__ldcg(P.b_exp + c)) : 0.0f;
    }
    __syncthreads();
    if (tid == 0 && tr) tr[5] = global_ns();
    ptx::mbar_wait(done, st.done_ph);
    st.done_ph ^= 1u;
    ptx::tc_fence_after();
    if (tid == 0 && tr) tr[6] = global_ns();
    {  // direct stores (they overlap the TMEM reads); warps w, w+4 split the chunks
        const int ew = warp & 3, half = warp >> 2;
        epilogue_chunks<kOZ8>(P, tm, tn, tmem + (static_cast<uint32_t>(ew * 32) << 16),
                              tm * kTile + ew * 32 + static_cast<int>(lane), col_scale, 4 * half, 4 * half + 4,
                              kb1 > kb0, epi_row<kOZ8>(P, tm, tn, tm * kTile + ew * 32 + static_cast<int>(lane)));
    }
    ptx::tc_fence_before();
    if (tid == 0 && tr) tr[7] = global_ns();
}

// Task bodies are separate (non-inlined) functions so each gets its own
// register allocation inside the persistent kernel.
__device__ __noinline__ void graph_leaf(const LeafArgs A, float* smem) { leaf_body(A, smem, false); }

__device__ __noinline__ void graph_slice(const SliceJob J, int r0) {
    const int r1 = min(J.rows, r0 + kGraphRows);
    for (int r = r0 + (threadIdx.x >> 5); r < r1; r += kGraphThreads / 32) slice_row(J, r, threadIdx.x & 31);
}

__global__ void __launch_bounds__(kGraphThreads, 1) inv_graph_kernel(const __grid_constant__ GraphProgram g) {
    extern __shared__ uint8_t graph_smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(graph_smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kGraphWork);
    uint64_t* empty = full + GOZ::kStages;
    uint64_t* done = empty + GOZ::kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    int* task_slot = reinterpret_cast<int*>(tmem_slot + 1);
    float* col_scale = reinterpret_cast<float*>(smem + kGraphWork + 256);
    const int tid = threadIdx.x, warp = tid >> 5;

    if (tid == 0) {
        for (int s = 0; s < GOZ::kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(done, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<GOZ::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    ptx::grid_dep_wait();  // PDL: the factors come from the previous launch
    RingState st;

    for (;;) {
        if (tid == 0) *task_slot = atomicAdd(g.cursor, 1);
        __syncthreads();
        const int t = *task_slot;
        if (t >= g.n_tasks) break;
        const GraphTask T = g.tasks[t];
        if (tid == 0 && g.trace) g.trace[8 * t] = global_ns();
        if (tid == 0 && T.type == GT_GEMM) {  // descriptors do not depend on the data: fetch early
            ptx::prefetch_tmap(g.maps + g.gemms[T.a].a_map);
            ptx::prefetch_tmap(g.maps + g.gemms[T.a].b_map);
        }
        if (tid == 0 && T.wait >= 0) {
            const int need = g.phase_size[T.wait];
                    while (ld_acquire_gpu(g.phase_done + T.wait) < need) __nanosleep(32);
            fence_proxy_async_global();
        }
        __syncthreads();
        long long clk0 = 0;
        if (tid == 0 && g.trace) {
            g.trace[8 * t + 1] = global_ns();
            clk0 = clock64();
        }
        switch (T.type) {
            case GT_GEMM:
                graph_gemm_tile(g, T.a, T.b, smem, full, empty, done, col_scale, tmem, st,
                                g.trace ? g.trace + 8 * t : nullptr);
                break;
            case GT_SLICE: {
                const SliceJob J = g.slices[T.a];
                graph_slice(J, T.b);
                break;
            }
            case GT_LEAF: {
                const LeafArgs A = g.leaves[T.a];
                graph_leaf(A, reinterpret_cast<float*>(smem));
                fence_proxy_async_smem();  // generic smem writes before the TMA ring reuses it
                break;
            }
            default: {
                const Damp2D D = g.damps[T.a];
                damp_rows(D, T.b);
                break;
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicAdd(g.phase_done + T.phase, 1);
            if (g.trace) {
                g.trace[8 * t + 2] = global_ns();
                g.trace[8 * t + 3] = smid();
                if (T.type != GT_GEMM) g.trace[8 * t + 4] = clock64() - clk0;  // cycles (effective clock)
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<GOZ::kTmemCols>(tmem);
}

}  // namespace pf
