// C = 8 dual gather ceiling: two separate 64-byte rows per neighbour (the current layout,
// U[bar], U[prev]) vs one interleaved 128-byte row [bar | prev] per neighbour, over the same
// uniform random index stream (E8 size: 4e6 rows, 1.59e8 indices).  Decides whether the E8
// sweep (0.55 of the copy peak) would gain from an interleaved pair layout.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
template <bool PAIR>
__global__ void __launch_bounds__(256) gather(const double* __restrict__ T, const double* __restrict__ T2,
                                              const unsigned* __restrict__ idx, long long n_idx, double* out) {
    const int lane = threadIdx.x & 31;
    const long long warps = (gridDim.x * (long long)blockDim.x) >> 5;
    long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    double acc = 0.0, acc2 = 0.0;
    for (long long base = w * 32; base < n_idx; base += warps * 32) {
        const unsigned my = idx[base + lane];
        if (PAIR) {   // 16 lanes per neighbour (8 bar + 8 prev, one 128-byte row): 2 neighbours per load
#pragma unroll
            for (int k0 = 0; k0 < 32; k0 += 16) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const unsigned o = __shfl_sync(0xffffffff, my, k0 + 2 * u + lane / 16) * 16 + (lane % 16);
                    v[u] = __ldg(T + o);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) acc += v[u];
            }
        } else {      // 8 lanes per neighbour per matrix: 4 neighbours per load, two loads
#pragma unroll
            for (int k0 = 0; k0 < 32; k0 += 32) {
                double v[8], p[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const unsigned o = __shfl_sync(0xffffffff, my, k0 + 4 * u + lane / 8) * 8 + (lane % 8);
                    v[u] = __ldg(T + o);
                    p[u] = __ldg(T2 + o);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) { acc += v[u]; acc2 += p[u]; }
            }
        }
    }
    if (acc + acc2 == 12345.0) out[0] = acc;
}
int main() {
    const long long N = 4000000; const long long n_idx = 159434706 / 32 * 32;
    double *T, *T2, *P, *out; unsigned *idx;
    cudaMalloc(&T, N * 64); cudaMalloc(&T2, N * 64); cudaMalloc(&P, N * 128); cudaMalloc(&idx, n_idx * 4); cudaMalloc(&out, 8);
    cudaMemset(T, 0, N * 64); cudaMemset(T2, 0, N * 64); cudaMemset(P, 0, N * 128);
    std::vector<unsigned> h(n_idx); std::mt19937_64 r(1); for (auto& x : h) x = r() % N;
    cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int occ : {4, 8}) {
        for (int pair = 0; pair < 2; ++pair) {
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                if (pair) gather<true><<<sms * occ, 256>>>(P, nullptr, idx, n_idx, out);
                else gather<false><<<sms * occ, 256>>>(T, T2, idx, n_idx, out);
                cudaEventRecord(b); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep == 2)
                    printf("{\"layout\": \"%s\", \"occ\": %d, \"ms\": %.3f, \"gbs_row_bytes\": %.0f}\n",
                           pair ? "pair128" : "separate64", occ, ms, n_idx * (2 * 64.0 + 4) / ms / 1e6);
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
