// random-row gather ceiling for C = 8 (64-byte rows), dual (two matrices), like E8
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
template <int C, int U>
__global__ void __launch_bounds__(256) gather(const double* __restrict__ T, const double* __restrict__ T2,
    const unsigned* __restrict__ idx, long long n_idx, double* out) {
    const int lane = threadIdx.x & 31;
    constexpr int Q = 32 / C;                       // rows per warp load
    const long long warps = (gridDim.x * (long long)blockDim.x) >> 5;
    long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    double acc = 0.0, acc2 = 0.0;
    for (long long base = w * 32; base < n_idx; base += warps * 32) {
        unsigned my = idx[base + lane];
        #pragma unroll
        for (int k0 = 0; k0 < 32; k0 += Q * U) {
            double v[U], p[U];
            #pragma unroll
            for (int u = 0; u < U; ++u) {
                unsigned o = __shfl_sync(0xffffffff, my, k0 + u * Q + lane / C) * C + (lane % C);
                v[u] = __ldg(T + o);
                p[u] = __ldg(T2 + o);
            }
            #pragma unroll
            for (int u = 0; u < U; ++u) { acc += v[u]; acc2 += p[u]; }
        }
    }
    if (acc + acc2 == 12345.0) out[0] = acc;
}
int main() {
    const long long N = 4000000; const long long n_idx = 159434706 / 32 * 32;
    double *T, *T2, *out; unsigned *idx;
    cudaMalloc(&T, N * 8 * 8); cudaMalloc(&T2, N * 8 * 8); cudaMalloc(&idx, n_idx * 4); cudaMalloc(&out, 8);
    cudaMemset(T, 0, N * 64); cudaMemset(T2, 0, N * 64);
    std::vector<unsigned> h(n_idx); std::mt19937_64 r(1); for (auto& x : h) x = r() % N;
    cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int occ : {4, 8}) {
        for (int rep = 0; rep < 2; ++rep) gather<8, 8><<<sms * occ, 256>>>(T, T2, idx, n_idx, out);
        cudaEventRecord(a); gather<8, 8><<<sms * occ, 256>>>(T, T2, idx, n_idx, out); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("C=8 dual gather occ=%d: %.2f ms, %.0f GB/s (row bytes) \n", occ, ms, n_idx * (2 * 64.0 + 4) / ms / 1e6);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
