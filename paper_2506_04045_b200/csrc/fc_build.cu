// fc_build.cu -- SparseSimilarity construction on the device.
//
// Replaces the reference's host construction (sparse.hpp:28-75): from_triplets
// sorts (i, j, v) triplets by (column, row), rejects duplicates, prefix-sums the
// column pointers, validates exact symmetry and sums v*v in stored order; on the
// CPU this costs ~160 s at config C.  Here: a CUB radix sort of
// 64-bit (column << 32 | row) keys, duplicate and symmetry checks as parallel
// kernels that report the FIRST failing entry in the reference's loop order (so
// the exception and its message are the reference's), and the stored-order
// frob_sq (exactly nnz for the all-ones A + I pattern; a sequential host loop
// otherwise, because a parallel sum would round differently).  The result is
// downloaded to the caller's arrays and made the context's resident similarity
// through fc_upload_csr.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <vector>

#include "fc_internal.h"
#include "fuzzyclust_cuda.h"

namespace {

constexpr unsigned long long kNoFailure = ~0ULL;

// triplet k's first failing check, in the reference's order (sparse.hpp:30-33)
__global__ void k_check_triplets(const uint32_t* r, const uint32_t* c, const double* v, uint64_t nnz, uint64_t n,
                                 unsigned long long* first_bad) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz; k += (uint64_t)gridDim.x * blockDim.x) {
        unsigned code = 0;
        if (r[k] >= n || c[k] >= n) code = 1;
        else if (v && (!(v[k] >= 0.0) || !isfinite(v[k]))) code = 2;
        if (code) atomicMin(first_bad, (unsigned long long)((k << 2) | code));
    }
}

__global__ void k_make_keys(const uint32_t* r, const uint32_t* c, uint64_t nnz, unsigned long long* keys) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz; k += (uint64_t)gridDim.x * blockDim.x)
        keys[k] = ((unsigned long long)c[k] << 32) | r[k];
}

// build_similarity's triplet list (sparse.hpp:66-75): diagonal first, then (u,v), (v,u) per edge
__global__ void k_edges_to_triplets(const uint32_t* edges, uint64_t m, uint64_t n, uint32_t* r, uint32_t* c) {
    const uint64_t total = n + 2 * m;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
        if (k < n) {
            r[k] = (uint32_t)k;
            c[k] = (uint32_t)k;
        } else {
            const uint64_t e = (k - n) / 2;
            const bool flip = ((k - n) & 1) != 0;
            const uint32_t u = edges[2 * e], w = edges[2 * e + 1];
            r[k] = flip ? w : u;
            c[k] = flip ? u : w;
        }
    }
}

__global__ void k_check_dups(const unsigned long long* keys, uint64_t nnz, int* flag) {
    for (uint64_t k = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz; k += (uint64_t)gridDim.x * blockDim.x)
        if (keys[k] == keys[k - 1]) *flag = 1;
}

__device__ __forceinline__ uint64_t lower_bound_u64(const unsigned long long* a, uint64_t lo, uint64_t hi,
                                                    unsigned long long x) {
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_col_ptr(const unsigned long long* keys, uint64_t nnz, uint64_t n, long long* ptr) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c <= n; c += (uint64_t)gridDim.x * blockDim.x)
        ptr[c] = (long long)lower_bound_u64(keys, 0, nnz, (unsigned long long)c << 32);
}

__global__ void k_split_rows(const unsigned long long* keys, uint64_t nnz, uint32_t* rows) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz; k += (uint64_t)gridDim.x * blockDim.x)
        rows[k] = (uint32_t)(keys[k] & 0xFFFFFFFFu);
}

// validate_symmetry (sparse.hpp:115-139): entry k = (i, j) needs (j, i) with the same value.
__global__ void k_check_symmetry(const unsigned long long* keys, const long long* ptr, const double* vals,
                                 uint64_t nnz, unsigned long long* first_bad) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j = (uint32_t)(keys[k] >> 32), i = (uint32_t)(keys[k] & 0xFFFFFFFFu);
        if (i == j) continue;
        const unsigned long long want = ((unsigned long long)i << 32) | j;   // (row j, column i)
        const uint64_t m = lower_bound_u64(keys, (uint64_t)ptr[i], (uint64_t)ptr[i + 1], want);
        unsigned code = 0;
        if (m >= (uint64_t)ptr[i + 1] || keys[m] != want) code = 1;
        else if (vals && vals[m] != vals[k]) code = 2;
        if (code) atomicMin(first_bad, (unsigned long long)((k << 2) | code));
    }
}

__global__ void k_any_not_one(const double* v, uint64_t nnz, int* flag) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nnz; k += (uint64_t)gridDim.x * blockDim.x)
        if (v[k] != 1.0) *flag = 1;
}

// FC_TRACE_HOST=1: per-phase wall times on stderr (syncs the stream at each mark)
struct Marks {
    cudaStream_t s;
    bool on;
    std::chrono::steady_clock::time_point t;
    explicit Marks(cudaStream_t st) : s(st), on(std::getenv("FC_TRACE_HOST") != nullptr), t(std::chrono::steady_clock::now()) {}
    void operator()(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[fc_build] %-14s %9.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

struct Dev {
    std::vector<void*> ptrs;
    cudaStream_t s;
    explicit Dev(cudaStream_t st) : s(st) {}
    template <class T>
    cudaError_t alloc(T** p, size_t count) {
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T), s);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    ~Dev() {
        for (void* p : ptrs) cudaFreeAsync(p, s);
        cudaStreamSynchronize(s);
    }
};

unsigned grid_of(uint64_t items) { return (unsigned)std::min<uint64_t>((items + 255) / 256, 148ull * 32); }

#define CUB_TRY(call)                                                                                   \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess) return fc_internal_fail(ctx, FC_DEVICE, std::string("CUDA error in construction: ") + cudaGetErrorString(e_)); \
    } while (0)

// Shared pipeline once (d_r, d_c[, d_v]) triplets are on the device.
int build_from_device_triplets(fc_ctx* ctx, uint64_t n, uint64_t nnz, uint32_t* d_r, uint32_t* d_c, double* d_v,
                               int64_t* row_ptr_out, uint32_t* col_out, double* values_out, double* frob_out,
                               int* pattern_only_out, Dev& dev) {
    cudaStream_t s = dev.s;
    Marks mark(s);
    unsigned long long* d_bad = nullptr;
    int* d_flag = nullptr;
    CUB_TRY(dev.alloc(&d_bad, 1));
    CUB_TRY(dev.alloc(&d_flag, 2));
    CUB_TRY(cudaMemsetAsync(d_bad, 0xFF, sizeof(unsigned long long), s));
    CUB_TRY(cudaMemsetAsync(d_flag, 0, 2 * sizeof(int), s));
    unsigned long long h_bad = kNoFailure;
    k_check_triplets<<<grid_of(nnz), 256, 0, s>>>(d_r, d_c, d_v, nnz, n, d_bad);
    CUB_TRY(cudaMemcpyAsync(&h_bad, d_bad, sizeof h_bad, cudaMemcpyDeviceToHost, s));
    CUB_TRY(cudaStreamSynchronize(s));
    if (h_bad != kNoFailure)
        return fc_internal_fail(ctx, FC_INVALID, (h_bad & 3) == 1 ? "similarity: index out of range"
                                                                   : "similarity: values must be finite and nonnegative");
    // sort by (column, row)
    unsigned long long *d_keys = nullptr, *d_keys2 = nullptr;
    double* d_v2 = nullptr;
    CUB_TRY(dev.alloc(&d_keys, nnz));
    CUB_TRY(dev.alloc(&d_keys2, nnz));
    if (d_v) CUB_TRY(dev.alloc(&d_v2, nnz));
    k_make_keys<<<grid_of(nnz), 256, 0, s>>>(d_r, d_c, nnz, d_keys);
    int hi_bits = 1;
    while ((1ull << hi_bits) < n) ++hi_bits;
    const int end_bit = 32 + hi_bits;
    size_t tmp_bytes = 0;
    void* d_tmp = nullptr;
    if (d_v) {
        CUB_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_keys, d_keys2, d_v, d_v2, (int64_t)nnz, 0, end_bit, s));
        CUB_TRY(dev.alloc(reinterpret_cast<char**>(&d_tmp), tmp_bytes));
        CUB_TRY(cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, d_keys, d_keys2, d_v, d_v2, (int64_t)nnz, 0, end_bit, s));
    } else {
        CUB_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, d_keys, d_keys2, (int64_t)nnz, 0, end_bit, s));
        CUB_TRY(dev.alloc(reinterpret_cast<char**>(&d_tmp), tmp_bytes));
        CUB_TRY(cub::DeviceRadixSort::SortKeys(d_tmp, tmp_bytes, d_keys, d_keys2, (int64_t)nnz, 0, end_bit, s));
    }
    mark("check+sort");
    k_check_dups<<<grid_of(nnz), 256, 0, s>>>(d_keys2, nnz, d_flag);
    int h_flag[2] = {0, 0};
    CUB_TRY(cudaMemcpyAsync(h_flag, d_flag, sizeof h_flag, cudaMemcpyDeviceToHost, s));
    CUB_TRY(cudaStreamSynchronize(s));
    if (h_flag[0]) return fc_internal_fail(ctx, FC_INVALID, "similarity: duplicate coordinate entry");
    long long* d_ptr = nullptr;
    uint32_t* d_rows = nullptr;
    CUB_TRY(dev.alloc(&d_ptr, n + 1));
    CUB_TRY(dev.alloc(&d_rows, nnz));
    k_col_ptr<<<grid_of(n + 1), 256, 0, s>>>(d_keys2, nnz, n, d_ptr);
    k_split_rows<<<grid_of(nnz), 256, 0, s>>>(d_keys2, nnz, d_rows);
    CUB_TRY(cudaMemsetAsync(d_bad, 0xFF, sizeof(unsigned long long), s));
    k_check_symmetry<<<grid_of(nnz), 256, 0, s>>>(d_keys2, d_ptr, d_v2, nnz, d_bad);
    if (d_v2) k_any_not_one<<<grid_of(nnz), 256, 0, s>>>(d_v2, nnz, d_flag + 1);
    CUB_TRY(cudaMemcpyAsync(&h_bad, d_bad, sizeof h_bad, cudaMemcpyDeviceToHost, s));
    CUB_TRY(cudaMemcpyAsync(h_flag, d_flag, sizeof h_flag, cudaMemcpyDeviceToHost, s));
    CUB_TRY(cudaStreamSynchronize(s));
    if (h_bad != kNoFailure) {
        if ((h_bad & 3) == 1) return fc_internal_fail(ctx, FC_INVALID, "similarity: matrix is not symmetric");
        unsigned long long key = 0;
        CUB_TRY(cudaMemcpy(&key, d_keys2 + (h_bad >> 2), sizeof key, cudaMemcpyDeviceToHost));
        return fc_internal_fail(ctx, FC_INVALID, "similarity: asymmetric values at (" +
                                                     std::to_string((unsigned)(key & 0xFFFFFFFFu)) + ", " +
                                                     std::to_string((unsigned)(key >> 32)) + ")");
    }
    // results to the caller
    mark("ptr+symmetry");
    int rc;
    if ((rc = fc_internal_d2h(ctx, row_ptr_out, d_ptr, (n + 1) * sizeof(int64_t)))) return rc;
    if ((rc = fc_internal_d2h(ctx, col_out, d_rows, nnz * sizeof(uint32_t)))) return rc;
    const bool weighted = d_v2 && h_flag[1];
    std::vector<double> vals;
    if (weighted) {
        vals.resize(nnz);
        if ((rc = fc_internal_d2h(ctx, vals.data(), d_v2, nnz * sizeof(double)))) return rc;
    }
    mark("download");
    double frob = 0.0;   // sparse.hpp:59-60, stored order
    if (weighted) {
        for (uint64_t k = 0; k < nnz; ++k) frob += vals[k] * vals[k];
        if (values_out) std::copy(vals.begin(), vals.end(), values_out);
    } else {
        frob = (double)nnz;   // every term 1.0: exact (nnz < 2^53)
        if (values_out)
            for (uint64_t k = 0; k < nnz; ++k) values_out[k] = 1.0;
    }
    if (frob_out) *frob_out = frob;
    if (pattern_only_out) *pattern_only_out = weighted ? 0 : 1;
    rc = fc_internal_adopt_device_csr(ctx, n, nnz, row_ptr_out, d_rows, weighted ? d_v2 : nullptr, frob);
    mark("frob+adopt");
    return rc;
}

}  // namespace

extern "C" int fc_build_from_triplets(fc_ctx* ctx, uint64_t n, uint64_t nnz, const uint32_t* rows,
                                      const uint32_t* cols, const double* values, int64_t* row_ptr_out,
                                      uint32_t* col_idx_out, double* values_out, double* frob_sq_out,
                                      int* pattern_only_out) {
    if (!ctx) return fc_internal_fail(nullptr, FC_INVALID, "null context");
    if (n == 0) return fc_internal_fail(ctx, FC_INVALID, "membership: empty matrix");
    if (n >= 0x80000000ULL) return fc_internal_fail(ctx, FC_INVALID, "similarity: 2^31 or more nodes");
    if (nnz >= 0x80000000ULL) return fc_internal_fail(ctx, FC_INVALID, "similarity: 2^31 or more entries");
    CUB_TRY(cudaSetDevice(fc_internal_device(ctx)));
    Dev dev(fc_internal_stream(ctx));
    uint32_t *d_r = nullptr, *d_c = nullptr;
    double* d_v = nullptr;
    CUB_TRY(dev.alloc(&d_r, nnz));
    CUB_TRY(dev.alloc(&d_c, nnz));
    int rc;
    if ((rc = fc_internal_h2d(ctx, d_r, rows, nnz * sizeof(uint32_t)))) return rc;
    if ((rc = fc_internal_h2d(ctx, d_c, cols, nnz * sizeof(uint32_t)))) return rc;
    if (values) {
        CUB_TRY(dev.alloc(&d_v, nnz));
        if ((rc = fc_internal_h2d(ctx, d_v, values, nnz * sizeof(double)))) return rc;
    }
    return build_from_device_triplets(ctx, n, nnz, d_r, d_c, d_v, row_ptr_out, col_idx_out, values_out, frob_sq_out,
                                      pattern_only_out, dev);
}

extern "C" int fc_build_similarity(fc_ctx* ctx, uint64_t num_nodes, uint64_t num_edges, const uint32_t* edges,
                                   int64_t* row_ptr_out, uint32_t* col_idx_out, double* frob_sq_out) {
    if (!ctx) return fc_internal_fail(nullptr, FC_INVALID, "null context");
    if (num_nodes == 0) return fc_internal_fail(ctx, FC_INVALID, "membership: empty matrix");
    if (num_nodes >= 0x80000000ULL) return fc_internal_fail(ctx, FC_INVALID, "similarity: 2^31 or more nodes");
    const uint64_t nnz = num_nodes + 2 * num_edges;
    if (nnz >= 0x80000000ULL) return fc_internal_fail(ctx, FC_INVALID, "similarity: 2^31 or more entries");
    CUB_TRY(cudaSetDevice(fc_internal_device(ctx)));
    Dev dev(fc_internal_stream(ctx));
    uint32_t *d_e = nullptr, *d_r = nullptr, *d_c = nullptr;
    CUB_TRY(dev.alloc(&d_e, 2 * num_edges));
    CUB_TRY(dev.alloc(&d_r, nnz));
    CUB_TRY(dev.alloc(&d_c, nnz));
    if (num_edges) {
        const int rc = fc_internal_h2d(ctx, d_e, edges, 2 * num_edges * sizeof(uint32_t));
        if (rc) return rc;
    }
    k_edges_to_triplets<<<grid_of(nnz), 256, 0, dev.s>>>(d_e, num_edges, num_nodes, d_r, d_c);
    return build_from_device_triplets(ctx, num_nodes, nnz, d_r, d_c, nullptr, row_ptr_out, col_idx_out, nullptr,
                                      frob_sq_out, nullptr, dev);
}
