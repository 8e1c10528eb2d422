// TEST INFRASTRUCTURE ONLY -- a host-only build of the repo's synthetic-graph
// generator (paper_2506_04045_b200/csrc/generator.cpp, compiled from the same
// source) for bench.py's `--impl reference` arm, so that arm builds its input
// graph without loading the CUDA library (libfuzzyclust_cuda.so): the only
// native code it runs is this generator and oracle/_ref/libfcref.so.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fuzzyclust_cuda.h"

extern "C" int fc_generate_graph_impl(const fc_graph_spec* spec, uint64_t* nnz_out, int64_t** row_ptr_out,
                                      uint32_t** col_idx_out, std::string* err);

extern "C" int fcgen_generate(const fc_graph_spec* spec, uint64_t* nnz_out, int64_t** row_ptr_out,
                              uint32_t** col_idx_out, char* err, size_t err_len) {
    std::string e;
    const int rc = fc_generate_graph_impl(spec, nnz_out, row_ptr_out, col_idx_out, &e);
    if (rc && err && err_len) std::snprintf(err, err_len, "%s", e.c_str());
    return rc;
}

extern "C" void fcgen_free(void* p) { std::free(p); }
