// fc_internal.h -- context accessors shared by the library's translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "fuzzyclust_cuda.h"

cudaStream_t fc_internal_stream(fc_ctx* ctx);
int fc_internal_device(fc_ctx* ctx);
int fc_internal_fail(fc_ctx* ctx, int code, const std::string& msg);
// make a CSR built on the device the resident similarity (row_ptr on the host, col /
// values on the device; d_val NULL = all ones)
int fc_internal_adopt_device_csr(fc_ctx* ctx, uint64_t n, uint64_t nnz, const int64_t* h_row_ptr,
                                 const uint32_t* d_col, const double* d_val, double frob_sq);
// large copies through the context's pinned staging ring (h2d: returns once src is
// consumed, stream-ordered; d2h: synchronous)
int fc_internal_h2d(fc_ctx* ctx, void* dst, const void* src, size_t bytes);
int fc_internal_d2h(fc_ctx* ctx, void* dst, const void* src, size_t bytes);
// the resident CSR of a single-rank context (all rows): n, row_ptr, col (hot bit
// possible in bit 31), values (NULL = pattern)
int fc_internal_csr(fc_ctx* ctx, uint64_t* n, const long long** row_ptr, const unsigned** col, const double** val);
