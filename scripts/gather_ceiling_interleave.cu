// Does interleaving the replicas per row help the dual gather?  (a) bar and prev rows
// in separate arrays (today), (b) [bar|prev] adjacent (512 B), (c) 3 replicas per row
// [U0|U1|U2] reading segments 0 and 2.
#include <cstdio>
#include <vector>
#include <random>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(256) gather(const double* __restrict__ A, const double* __restrict__ B,
    const unsigned* __restrict__ idx, long long n_idx, double* out) {
    const int lane = threadIdx.x & 31;
    const long long warps = (gridDim.x * (long long)blockDim.x) >> 5;
    long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    double acc = 0.0, acc2 = 0.0;
    for (long long base = w * 32; base < n_idx; base += warps * 32) {
        unsigned my = idx[base + lane];
#pragma unroll
        for (int k0 = 0; k0 < 32; k0 += 8) {
            double v[8], p[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const unsigned r = __shfl_sync(0xffffffff, my, k0 + u);
                if (MODE == 0) { v[u] = __ldg(A + (size_t)r * 32 + lane); p[u] = __ldg(B + (size_t)r * 32 + lane); }
                else if (MODE == 1) { v[u] = __ldg(A + (size_t)r * 64 + lane); p[u] = __ldg(A + (size_t)r * 64 + 32 + lane); }
                else { v[u] = __ldg(A + (size_t)r * 96 + lane); p[u] = __ldg(A + (size_t)r * 96 + 64 + lane); }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) { acc += v[u]; acc2 += p[u]; }
        }
    }
    if (acc + acc2 == 12345.0) out[0] = acc;
}
int main(int argc, char** argv) {
    const long long N = 10000000; const long long n_idx = 398404788 / 32 * 32;
    double *A, *B, *out; unsigned *idx;
    cudaMalloc(&A, N * 96 * 8); cudaMalloc(&B, N * 32 * 8); cudaMalloc(&idx, n_idx * 4); cudaMalloc(&out, 8);
    cudaMemset(A, 0, N * 96 * 8); cudaMemset(B, 0, N * 32 * 8);
    // the real config-C column stream if given, else uniform random
    std::vector<unsigned> h(n_idx);
    FILE* f = argc > 1 ? fopen(argv[1], "rb") : nullptr;
    if (f) { fread(h.data(), 4, n_idx, f); fclose(f); }
    else { std::mt19937_64 r(1); for (auto& x : h) x = r() % N; }
    cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[3] = {"separate arrays", "adjacent [bar|prev]", "3-replica rows, seg 0+2"};
    for (int mode = 0; mode < 3; ++mode) for (int occ : {4, 8}) {
        auto run = [&]() {
            if (mode == 0) gather<0><<<sms * occ, 256>>>(A, B, idx, n_idx, out);
            else if (mode == 1) gather<1><<<sms * occ, 256>>>(A, B, idx, n_idx, out);
            else gather<2><<<sms * occ, 256>>>(A, B, idx, n_idx, out);
        };
        run(); run();
        cudaEventRecord(a); run(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-26s occ=%d %.2f ms %.0f GB/s\n", names[mode], occ, ms, n_idx * (512.0 + 4) / ms / 1e6);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
