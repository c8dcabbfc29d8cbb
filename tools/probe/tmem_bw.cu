// TMEM -> register read bandwidth per SM for tcgen05.ld shapes (dev probe).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int N>
__device__ __forceinline__ void ld32x32b(uint32_t taddr, uint32_t (&r)[N]);

#define LD_X16(taddr, r)                                                                                   \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),   \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),          \
                   "=r"(r[15])                                                                                     \
                 : "r"(taddr))
#define LD_X32(taddr, r)                                                                                   \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),   \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),          \
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),        \
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),        \
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                          \
                 : "r"(taddr))
#define LD_16x256_X4(taddr, r)                                                                                   \
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),   \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),          \
                   "=r"(r[15])                                                                                     \
                 : "r"(taddr))
#define WAIT() asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory")

template <int kMode>
__global__ void __launch_bounds__(256, 1) k(long long* out, uint32_t* sink, int reps) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const int half = warp >> 2;  // two warps per lane quarter: 256 columns each
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        if (kMode == 0) {  // 32x32b.x16, 4 in flight then wait
            for (int c = 0; c < 256; c += 64) {
                uint32_t r[4][16];
                LD_X16(tmem + half * 256 + c, r[0]);
                LD_X16(tmem + half * 256 + c + 16, r[1]);
                LD_X16(tmem + half * 256 + c + 32, r[2]);
                LD_X16(tmem + half * 256 + c + 48, r[3]);
                WAIT();
#pragma unroll
                for (int g = 0; g < 4; ++g)
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc += r[g][j];
            }
        } else if (kMode == 1) {  // 32x32b.x32, 2 in flight
            for (int c = 0; c < 256; c += 64) {
                uint32_t r[2][32];
                LD_X32(tmem + half * 256 + c, r[0]);
                LD_X32(tmem + half * 256 + c + 32, r[1]);
                WAIT();
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                    for (int j = 0; j < 32; ++j) acc += r[g][j];
            }
        } else {  // 16x256b.x4: 16 lanes x (4 x 256 bit) per instr -> 16 regs
            for (int c = 0; c < 256; c += 32) {
                uint32_t r[2][16];
                LD_16x256_X4(tmem + half * 256 + c, r[0]);
                LD_16x256_X4(tmem + (16u << 16) + half * 256 + c, r[1]);
                WAIT();
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc += r[g][j];
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    long long* d_out;
    uint32_t* sink;
    cudaMalloc(&d_out, 8);
    cudaMalloc(&sink, 4096);
    const int reps = 200;
    const double bytes = 128.0 * 512 * 4 * reps;  // all 512 columns x 128 lanes per rep
    for (int mode = 0; mode < 3; ++mode) {
        for (int w = 0; w < 2; ++w) {
            if (mode == 0) k<0><<<1, 256>>>(d_out, sink, reps);
            if (mode == 1) k<1><<<1, 256>>>(d_out, sink, reps);
            if (mode == 2) k<2><<<1, 256>>>(d_out, sink, reps);
        }
        long long cyc = 0;
        cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
        printf("mode %d (%s): %lld cycles, %.1f B/cycle, err=%s\n", mode,
               mode == 0 ? "32x32b.x16 x4" : mode == 1 ? "32x32b.x32 x2" : "16x256b.x4 x2", cyc, bytes / cyc,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
