// Thin inline-PTX layer for sm_100a: mbarriers, TMA, tcgen05 (UMMA + TMEM).
// Everything the K-FAC kernels need from the Blackwell async machinery, with
// no CUTLASS dependency (bit layouts follow the PTX ISA / the descriptor
// documentation in cute/arch/mma_sm100_desc.hpp).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pf {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() {
    uint32_t l;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
// Programmatic dependent launch (PDL).  Kernels launched with the
// programmatic-stream-serialization attribute run their prologue while the
// previous kernel drains; `grid_dep_wait` blocks until that kernel has
// completed and its writes are visible.  Both are no-ops without the attribute.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Block until the phase with parity `parity` of `bar` has completed.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// 2-D tiled bulk tensor load global -> shared, completion on `bar` (tx bytes).
// c0 = innermost (contiguous) coordinate, c1 = row coordinate, in elements.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int c0,
                                            int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// Plain (non-tensor) bulk copy global -> shared of `bytes` (multiple of 16,
// both addresses 16-B aligned), completion on `bar` (tx bytes).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Plain bulk copy shared -> global (bulk-group completion), and its group ops.
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (bulk copies)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 3-D tiled bulk tensor load (c0 innermost): the int8 digit planes of one
// operand tile arrive in one instruction, plane-major in shared memory.
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// ---------------------------------------------------------------- tcgen05
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot_in_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(slot_in_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 inputs, fp32 accumulate).
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Same with kind::i8 (signed int8 digits, exact s32 accumulate).
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                        uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// The 10 digit products of one 32-byte k-step (kind::i8, s_a + s_b <= 3)
// into the four weight accumulators t[g] (g = s_a + s_b), in ONE asm block:
// as separate statements each MMA was wrapped by ptxas in its own
// register -> uniform-register waterfall loop (~70 cycles per MMA, more than
// a 128 x 32 x 32 MMA takes on the tensor core).  start_mask bit g: the
// accumulator g already holds a partial sum (else its first product
// overwrites it).
__device__ __forceinline__ void umma_i8_digits(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3,
                                               const uint64_t (&a)[4], const uint64_t (&b)[4], uint32_t idesc,
                                               uint32_t start_mask) {
    asm volatile(
        "{\n\t.reg .pred q0, q1, q2, q3, qt;\n\t"
        ".reg .b32 m;\n\t"
        "setp.eq.u32 qt, 0, 0;\n\t"
        "and.b32 m, %13, 1;\n\tsetp.ne.b32 q0, m, 0;\n\t"
        "and.b32 m, %13, 2;\n\tsetp.ne.b32 q1, m, 0;\n\t"
        "and.b32 m, %13, 4;\n\tsetp.ne.b32 q2, m, 0;\n\t"
        "and.b32 m, %13, 8;\n\tsetp.ne.b32 q3, m, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %4, %8, %12, q0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%1], %4, %9, %12, q1;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%1], %5, %8, %12, qt;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%2], %4, %10, %12, q2;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%2], %5, %9, %12, qt;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%2], %6, %8, %12, qt;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%3], %4, %11, %12, q3;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%3], %5, %10, %12, qt;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%3], %6, %9, %12, qt;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%3], %7, %8, %12, qt;\n\t"
        "}" ::"r"(t0),
        "r"(t1), "r"(t2), "r"(t3), "l"(a[0]), "l"(a[1]), "l"(a[2]), "l"(a[3]), "l"(b[0]), "l"(b[1]), "l"(b[2]),
        "l"(b[3]), "r"(idesc), "r"(start_mask)
        : "memory");
}

// Arrive on `bar` once every previously issued tcgen05.mma of this thread
// has completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// 32 lanes x 32-bit, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Same without the wait: issue several loads, then one tmem_wait_ld().
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// The wait with a register dependency on `r`, so that no use of the loaded
// registers can be scheduled above it (needed when loads are in flight across
// other work).
__device__ __forceinline__ void tmem_wait_ld_dep(uint32_t (&r)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                   "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
                   "+r"(r[14]), "+r"(r[15])
                 :
                 : "memory");
}

// 2^e as an exact double for |e| <= 1022 (no libm call).
__device__ __forceinline__ double pow2(int e) {
    return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
}

// 2^e as a float, saturating outside the normal range (row/column scales of
// finite fp32 data: e in [-148, 128]).
__device__ __forceinline__ float pow2f(int e) {
    return e > 127 ? __int_as_float(0x7f000000) * 2.0f
                   : (e < -126 ? 0.0f : __int_as_float((e + 127) << 23));
}

// ---------------------------------------------------------------- descriptors
// Shared-memory matrix descriptor for a K-major operand tile laid out by TMA
// with SWIZZLE_128B: rows of 128 B, 8-row (1024 B) swizzle atoms stacked
// along M/N.  start_address/LBO/SBO in 16-byte units, version=1 (sm_100),
// layout_type=2 (SWIZZLE_128B).  LBO is unused for swizzled K-major (=1).
__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(1u) << 16;            // LBO (ignored)
    d |= static_cast<uint64_t>(1024u >> 4) << 32;    // SBO: next 8-row group
    d |= static_cast<uint64_t>(1u) << 46;            // version
    d |= static_cast<uint64_t>(2u) << 61;            // SWIZZLE_128B
    return d;
}

// Same for SWIZZLE_64B tiles (rows of 64 B; 8-row atoms of 512 B).
__device__ __forceinline__ uint64_t sw64_kmajor_desc(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(1u) << 16;            // LBO (ignored)
    d |= static_cast<uint64_t>(512u >> 4) << 32;     // SBO: next 8-row group
    d |= static_cast<uint64_t>(1u) << 46;            // version
    d |= static_cast<uint64_t>(4u) << 61;            // SWIZZLE_64B
    return d;
}

// MN-major (feature-contiguous) operand tile with SWIZZLE_128B, as TMA
// writes a box of {64 MN elements, K rows}: 128-B rows along K, 8-row
// (1024 B) swizzle atoms; LBO = byte stride between the 64-element MN blocks,
// SBO = byte stride between 8-row K groups (canonical MN-major SW128 layout
// ((T,8,m),(8,k)) : ((1,T,LBO),(8T,SBO)), T = 8 bf16 per 16 B).
__device__ __forceinline__ uint64_t sw128_mnmajor_desc(uint32_t smem_addr, uint32_t lbo_bytes,
                                                       uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1u) << 46;            // version
    d |= static_cast<uint64_t>(2u) << 61;            // SWIZZLE_128B
    return d;
}
// instruction-descriptor bits: A / B read MN-major ("transposed")
constexpr uint32_t kIdescAMnMajor = 1u << 15;
constexpr uint32_t kIdescBMnMajor = 1u << 16;

// Instruction descriptor: fp32 accumulate, K-major A and B, MxN tile.
// fmt: 1 = BF16 (kind::f16), 2 = TF32 (kind::tf32).
__host__ __device__ constexpr uint32_t make_idesc(uint32_t fmt, uint32_t m, uint32_t n) {
    return (1u << 4)            // c_format = F32
           | (fmt << 7)         // a_format
           | (fmt << 10)        // b_format
           | ((n >> 3) << 17)   // n_dim
           | ((m >> 4) << 24);  // m_dim
}

// ---------------------------------------------------------------- flags
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// ---------------------------------------------------------------- clusters
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// every thread of every CTA of the cluster; release / acquire orders the
// shared-memory writes before the barrier with the remote reads after it
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cta address -> the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

__device__ __forceinline__ float4 ld_dsmem4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

}  // namespace ptx
}  // namespace pf
