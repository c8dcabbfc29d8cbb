// Standalone probe: times leaf_chol_inv_kernel phases with clock64 stamps.
// nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -DPF_LEAF_PROBE -I paper_2211_14133_b200/csrc/kernels tools/probe/leaf_probe.cu -o /tmp/leaf_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <string>
#include "leaf.cuh"
using namespace pf;

// Contention modes (argv[1]): "mem" = 147 CTAs stream a 1 GiB buffer
// (read + write, ~BR's HBM traffic pattern) on a second stream while the
// leaf runs; "spin" = 147 CTAs of FFMA chains (SM load, no memory traffic);
// "l2" = 147 CTAs re-reading a 32 MiB buffer (L2-resident traffic).
__global__ void busy_mem(float4* buf, size_t n4, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
            float4 v = buf[i];
            v.x += 1.0f;
            buf[i] = v;
        }
}
__global__ void busy_spin(float* out, int iters) {
    float a = threadIdx.x, b = 1.0001f;
    for (int i = 0; i < iters; ++i) a = fmaf(a, b, 0.5f);
    if (a == 12345.0f) out[0] = a;
}

int main(int argc, char** argv) {
    const char* mode = argc > 1 ? argv[1] : "none";
    const int n = 128, ld = 128;
    std::vector<float> a(n * n);
    srand(1);
    std::vector<float> x(n * 256);
    for (auto& v : x) v = (rand() / (float)RAND_MAX - 0.5f) * 3.4f;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0;
            for (int k = 0; k < 256; ++k) s += x[i * 256 + k] * x[j * 256 + k];
            a[i * n + j] = s / 256 + (i == j ? 0.1 : 0.0);
        }
    float *da, *dx, *dxt; int* info; long long* stamps;
    cudaMalloc(&da, n * n * 4); cudaMalloc(&dx, n * n * 4); cudaMalloc(&dxt, n * n * 4);
    cudaMalloc(&info, 4); cudaMalloc(&stamps, 64 * 8); cudaMemset(stamps, 0, 64 * 8);
    cudaMemcpy(da, a.data(), n * n * 4, cudaMemcpyHostToDevice);
    cudaMemset(info, 0, 4);
    cudaFuncSetAttribute(leaf_chol_inv_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kLeafSmemBytes);
    LeafBatch b{};
    b.e[0] = LeafArgs{da, dx, dxt, info, ld, n, 0};
    cudaMemcpyToSymbol(g_probe, &stamps, sizeof(stamps));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaStream_t s0, s1;
    cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    float4* big = nullptr;
    const size_t big_n4 = std::string(mode) == "l2" ? (32u << 20) / 16 : (1u << 30) / 16;
    cudaMalloc(&big, big_n4 * 16);
    cudaMemset(big, 0, big_n4 * 16);
    auto busy = [&] {
        if (std::string(mode) == "mem") busy_mem<<<147, 512, 0, s1>>>(big, big_n4, 1);
        if (std::string(mode) == "l2") busy_mem<<<147, 512, 0, s1>>>(big, big_n4, 40);
        if (std::string(mode) == "spin") busy_spin<<<147, 256, 0, s1>>>(reinterpret_cast<float*>(big), 400000);
    };
    for (int it = 0; it < 5; ++it) leaf_chol_inv_kernel<false><<<1, kLeafThreads, kLeafSmemBytes, s0>>>(b);
    cudaDeviceSynchronize();
    cudaEventRecord(e0, s0);
    for (int it = 0; it < 20; ++it) leaf_chol_inv_kernel<false><<<1, kLeafThreads, kLeafSmemBytes, s0>>>(b);
    cudaEventRecord(e1, s0);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("err=%s  avg %.2f us per launch (stream, back to back)\n", cudaGetErrorString(cudaGetLastError()), ms * 1000 / 20);
    // last: one leaf launched while the busy kernel runs (its stamps are printed)
    float busy_ms = 0;
    for (int it = 0; it < 5; ++it) {
        busy();
        cudaEventRecord(e0, s0);
        leaf_chol_inv_kernel<false><<<1, kLeafThreads, kLeafSmemBytes, s0>>>(b);
        cudaEventRecord(e1, s0);
        cudaDeviceSynchronize();
        float t; cudaEventElapsedTime(&t, e0, e1); busy_ms += t;
    }
    printf("mode %s: %.2f us per leaf launched under load (event pair)\n", mode, busy_ms * 1000 / 5);
    long long h[64]; cudaMemcpy(h, stamps, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[] = {"start", "zero", "load", "p0A", "p0B", "p0C", "p1A", "p1B", "p1C",
                           "p2A", "p2B", "p2C", "p3A", "inv33", "x3", "", "", "", "", "store"};
    long long prev = h[0];
    for (int i = 1; i < 20; ++i) if (h[i]) { printf("%-8s %7lld cycles\n", names[i], h[i] - prev); prev = h[i]; }
    printf("total    %7lld cycles\n", h[19] - h[0]);
    // phase A split: warp 0's chol32 vs warp 1's share of the trailing/T work
    const int a_start[4] = {2, 5, 8, 11};  // stamp index that precedes phase A of panel p
    for (int p = 0; p < 4; ++p)
        printf("p%dA: chol32 %6lld  other warps %6lld  phase %6lld cycles\n", p, h[20 + p] - h[a_start[p]],
               p ? h[24 + p] - h[a_start[p]] : 0LL, h[3 + 3 * p] - h[a_start[p]]);
    // residual check on host
    std::vector<float> X(n * n); cudaMemcpy(X.data(), dx, n * n * 4, cudaMemcpyDeviceToHost);
    // L^-1 check: X A X^T = I
    double mx = 0;
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) {
        double s = 0;
        for (int k = 0; k < n; ++k) { double t = 0; for (int l = 0; l < n; ++l) t += (double)a[k * n + l] * X[j * n + l]; s += X[i * n + k] * t; }
        mx = fmax(mx, fabs(s - (i == j)));
    }
    printf("max|X A X^T - I| = %.3e\n", mx);
}
