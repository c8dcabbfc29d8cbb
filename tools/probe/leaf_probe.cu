// Standalone probe: times leaf_chol_inv_kernel phases with clock64 stamps.
// nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -DPF_LEAF_PROBE -I paper_2211_14133_b200/csrc/kernels tools/probe/leaf_probe.cu -o /tmp/leaf_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "leaf.cuh"
using namespace pf;

int main() {
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
    for (int it = 0; it < 5; ++it) leaf_chol_inv_kernel<false><<<1, kLeafThreads, kLeafSmemBytes>>>(b);
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) leaf_chol_inv_kernel<false><<<1, kLeafThreads, kLeafSmemBytes>>>(b);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("err=%s  avg %.2f us per launch (stream, back to back)\n", cudaGetErrorString(cudaGetLastError()), ms * 1000 / 20);
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
