// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/include/fuzzyclust/*.hpp, header-only C++20), compiled by
// oracle/Makefile with the reference's own Release flags (-std=gnu++20 -O3
// -DNDEBUG, no -march => no FMA; proj/CMakeLists.txt:7-9) into
// oracle/_ref/libfcref.so.  No reference source is copied: this file only
// #includes the headers where they lie.
//
// Used (a) by tests/ to pin the plain-C restatement (oracle/fc_oracle.c) and the
// CUDA path bitwise against the real reference, and (b) by bench.py as the CPU
// baseline / `--impl reference` arm (the reference's own run_fista/run_gpa on the
// box's host cores).
//
// SparseSimilarity keeps its CSR private (sparse.hpp:141-145) and its only
// constructors sort triplets (sparse.hpp:28-62: ~160 s at N=1e7).  For large,
// already-validated CSR (our generator's output, which the small-size tests
// push through from_triplets) the shim fills the private fields directly: all
// standard headers are included first, then `private` is redefined for the
// reference headers only.  The solver code that runs is unchanged.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <istream>
#include <limits>
#include <optional>
#include <ostream>
#include <queue>
#include <set>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <utility>
#include <vector>

#define private public
#include "fuzzyclust/fuzzyclust.hpp"
#undef private

using namespace fuzzyclust;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const IoError& e) {
        g_err = e.what();
        return 1;
    } catch (const InvalidInput& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

MembershipMatrix wrap(const double* x, std::size_t c, std::size_t n) {
    MembershipMatrix m(c, n);
    std::memcpy(m.data().data(), x, c * n * sizeof(double));
    return m;
}
}  // namespace

extern "C" {

struct fcref_record {
    uint64_t iteration;
    double loss;
    int32_t loss_increased;
    int32_t pad;
    double elapsed_ms;
};

struct fcref_summary {
    int32_t reason;
    int32_t pad;
    uint64_t iterations;
    double final_loss;
    double step_size;
    uint64_t n_records;
    double solve_ms;
};

const char* fcref_last_error() { return g_err.c_str(); }
const char* fcref_version() { return kVersion; }
unsigned fcref_resolve_workers(unsigned requested) { return resolve_workers(requested); }

// fast != 0: fill the private CSR fields directly (no sort / symmetry check).
// fast == 0: SparseSimilarity::from_triplets (full reference validation).
int fcref_similarity_create(uint64_t n, uint64_t nnz, const int64_t* row_ptr, const uint32_t* col_idx,
                            const double* values, int fast, void** out) {
    return guarded([&] {
        auto* s = new SparseSimilarity();
        if (fast) {
            s->n_ = n;
            s->col_ptr_.assign(row_ptr, row_ptr + n + 1);
            s->rows_.assign(col_idx, col_idx + nnz);
            if (values) {
                s->values_.assign(values, values + nnz);
            } else {
                s->values_.assign(nnz, 1.0);
            }
            s->frob_sq_ = 0.0;
            for (double v : s->values_) s->frob_sq_ += v * v;
        } else {
            std::vector<std::tuple<std::uint32_t, std::uint32_t, double>> t;
            t.reserve(nnz);
            for (uint64_t j = 0; j < n; ++j)
                for (int64_t e = row_ptr[j]; e < row_ptr[j + 1]; ++e)
                    t.emplace_back(col_idx[e], static_cast<std::uint32_t>(j), values ? values[e] : 1.0);
            *s = SparseSimilarity::from_triplets(n, std::move(t));
        }
        *out = s;
    });
}

// SparseSimilarity::from_triplets (sparse.hpp:28-62) on raw triplets in caller order
// (unsorted, possibly invalid): pins the device construction, messages included.
int fcref_from_triplets(uint64_t n, uint64_t count, const uint32_t* rows, const uint32_t* cols,
                        const double* values, void** out) {
    return guarded([&] {
        std::vector<std::tuple<std::uint32_t, std::uint32_t, double>> t;
        t.reserve(count);
        for (uint64_t k = 0; k < count; ++k) t.emplace_back(rows[k], cols[k], values[k]);
        auto* s = new SparseSimilarity(SparseSimilarity::from_triplets(n, std::move(t)));
        *out = s;
    });
}

void fcref_similarity_free(void* s) { delete static_cast<SparseSimilarity*>(s); }
double fcref_similarity_frob_sq(void* s) { return static_cast<SparseSimilarity*>(s)->frob_sq(); }
uint64_t fcref_similarity_nnz(void* s) { return static_cast<SparseSimilarity*>(s)->nnz(); }

// Copy the stored CSR back out (pins that from_triplets reproduces our layout).
int fcref_similarity_export(void* h, int64_t* row_ptr, uint32_t* col_idx, double* values) {
    return guarded([&] {
        const auto& s = *static_cast<SparseSimilarity*>(h);
        uint64_t pos = 0;
        row_ptr[0] = 0;
        for (std::size_t j = 0; j < s.size(); ++j) {
            const auto r = s.col_rows(j);
            const auto v = s.col_values(j);
            for (std::size_t k = 0; k < r.size(); ++k) {
                col_idx[pos] = r[k];
                values[pos] = v[k];
                ++pos;
            }
            row_ptr[j + 1] = static_cast<int64_t>(pos);
        }
    });
}

// Edge list (u, v) -> Graph -> build_similarity (sparse.hpp:66-75).
int fcref_build_similarity(uint64_t num_nodes, uint64_t m, const uint32_t* edges, void** out) {
    return guarded([&] {
        Graph g;
        g.num_nodes = num_nodes;
        g.edges.reserve(m);
        for (uint64_t e = 0; e < m; ++e) g.edges.emplace_back(edges[2 * e], edges[2 * e + 1]);
        normalize_edges(g.edges);
        *out = new SparseSimilarity(SparseSimilarity::build_similarity(g));
    });
}

int fcref_project_simplex(double* x, uint64_t c) {
    return guarded([&] { project_simplex_inplace(std::span<double>(x, c)); });
}

uint64_t fcref_splitmix(uint64_t seed, uint64_t k) {
    SplitMix64 r(seed);
    uint64_t v = 0;
    for (uint64_t i = 0; i <= k; ++i) v = r.next();
    return v;
}

// kind: 0 random, 1 dirichlet, 2 rowone, 3 uniform
int fcref_init_membership(uint64_t n, uint64_t c, int kind, uint64_t seed, uint64_t row, double* out) {
    return guarded([&] {
        InitStrategy st;
        st.kind = kind == 0 ? InitKind::kRandom
                 : kind == 1 ? InitKind::kDirichlet
                 : kind == 2 ? InitKind::kRowOne
                             : InitKind::kUniform;
        st.seed = seed;
        st.row = row;
        const auto x = init_membership(n, c, st);
        std::memcpy(out, x.data().data(), n * c * sizeof(double));
    });
}

int fcref_share_matrix(const double* x, uint64_t c, uint64_t n, unsigned workers, double* g) {
    return guarded([&] {
        const auto m = wrap(x, c, n);
        const ShareMatrix s = share_matrix(m, workers);
        for (std::size_t r = 0; r < c; ++r)
            for (std::size_t q = 0; q < c; ++q) g[r * c + q] = s(r, q);
    });
}

int fcref_fused_column_pass(void* h, const double* x, uint64_t c, unsigned workers, double* xs,
                            double* merge) {
    return guarded([&] {
        const auto& s = *static_cast<SparseSimilarity*>(h);
        const auto m = wrap(x, c, s.size());
        const ColumnPass p = fused_column_pass(m, s, workers);
        std::memcpy(xs, p.xs.data(), p.xs.size() * sizeof(double));
        *merge = p.merge;
    });
}

int fcref_cross_share(const double* a, const double* b, uint64_t c, uint64_t n, unsigned workers, double* g) {
    return guarded([&] {
        const auto ma = wrap(a, c, n), mb = wrap(b, c, n);
        const ShareMatrix s = cross_share(ma, mb, workers);
        for (std::size_t r = 0; r < c; ++r)
            for (std::size_t q = 0; q < c; ++q) g[r * c + q] = s(r, q);
    });
}

int fcref_hessian_vector_product(void* h, const double* x, const double* v, uint64_t c, unsigned workers,
                                 double* out, double* qform) {
    return guarded([&] {
        const auto& s = *static_cast<SparseSimilarity*>(h);
        const auto mx = wrap(x, c, s.size()), mv = wrap(v, c, s.size());
        const DenseMatrix hv = hessian_vector_product(mx, mv, s, workers);
        std::memcpy(out, hv.data().data(), hv.data().size() * sizeof(double));
        if (qform) *qform = quadratic_form(mx, mv, s, workers);
    });
}

// tools/fuzzyclust.cpp:62-89 load_pipeline, composed from the reference's graph.hpp
// (parse_edge_list -> largest_connected_component_nodes -> induced_subgraph ->
// two_core_nodes -> induced_subgraph).  Outputs malloc'ed; fcref_free_buf.
int fcref_load_pipeline(const char* text, uint64_t len, int stages, uint64_t* parsed_nodes, uint64_t* lcc_nodes,
                        uint64_t* num_nodes, uint64_t* num_edges, uint32_t** edges, int64_t** ids) {
    return guarded([&] {
        std::istringstream in(std::string(text, len));
        auto parsed = parse_edge_list(in);
        Graph g = parsed.graph;
        std::vector<std::int64_t> orig = parsed.original_ids;
        *parsed_nodes = g.num_nodes;
        *lcc_nodes = 0;
        if (stages >= 1) {
            const auto lcc = largest_connected_component_nodes(g);
            g = induced_subgraph(g, lcc);
            std::vector<std::int64_t> kept;
            for (std::uint32_t v : lcc) kept.push_back(orig[v]);
            orig = kept;
            *lcc_nodes = g.num_nodes;
            if (stages >= 2) {
                const auto core = two_core_nodes(g);
                g = induced_subgraph(g, core);
                std::vector<std::int64_t> surv;
                for (std::uint32_t v : core) surv.push_back(orig[v]);
                orig = surv;
            }
        }
        *num_nodes = g.num_nodes;
        *num_edges = g.edges.size();
        *edges = static_cast<uint32_t*>(std::malloc(std::max<std::size_t>(2 * g.edges.size(), 1) * 4));
        *ids = static_cast<int64_t*>(std::malloc(std::max<std::size_t>(orig.size(), 1) * 8));
        for (std::size_t k = 0; k < g.edges.size(); ++k) {
            (*edges)[2 * k] = g.edges[k].first;
            (*edges)[2 * k + 1] = g.edges[k].second;
        }
        std::copy(orig.begin(), orig.end(), *ids);
    });
}

int fcref_graph_nodes(uint64_t n, uint64_t m, const uint32_t* edges, int which, uint32_t** nodes, uint64_t* count) {
    return guarded([&] {
        Graph g;
        g.num_nodes = n;
        for (uint64_t k = 0; k < m; ++k) g.edges.emplace_back(edges[2 * k], edges[2 * k + 1]);
        const auto v = which == 0 ? largest_connected_component_nodes(g) : two_core_nodes(g);
        *nodes = static_cast<uint32_t*>(std::malloc(std::max<std::size_t>(v.size(), 1) * 4));
        std::copy(v.begin(), v.end(), *nodes);
        *count = v.size();
    });
}

void fcref_free_buf(void* p) { std::free(p); }

struct fcref_verdict {
    int status;
    int has_witness;
    int has_base;
    int interior_shortcut;
    uint64_t tested;
    double value;
};
// secondorder.hpp:343-368 refine on the reference; dense witnesses copied out (n x c node-major)
int fcref_refine(void* h, const double* x, uint64_t c, double tau_probe, double eps_critical, double eps_active,
                 double eps_grad_orth, double eps_quad, double eps_cone, uint64_t random_directions, uint64_t seed,
                 uint64_t budget, int* critical, double* residual, int* status, uint64_t* generated,
                 fcref_verdict* a, fcref_verdict* b, double* a_witness, double* b_witness, double* b_base) {
    return guarded([&] {
        const auto& s = *static_cast<SparseSimilarity*>(h);
        const auto m = wrap(x, c, s.size());
        SecondOrderConfig cfg;
        cfg.tau_probe = tau_probe;
        cfg.eps_critical = eps_critical;
        cfg.eps_active = eps_active;
        cfg.eps_grad_orth = eps_grad_orth;
        cfg.eps_quad = eps_quad;
        cfg.eps_cone = eps_cone;
        cfg.random_directions = random_directions;
        cfg.seed = seed;
        cfg.budget = budget;
        const RefinementReport r = refine(m, s, cfg);
        *critical = r.critical ? 1 : 0;
        *residual = r.residual;
        *status = static_cast<int>(r.status);
        *generated = r.directions_generated;
        auto fill = [&](const RefinementVerdict& v, fcref_verdict* o, double* w, double* base) {
            o->status = static_cast<int>(v.status);
            o->tested = v.directions_tested;
            o->value = v.witness_value;
            o->interior_shortcut = v.used_interior_shortcut ? 1 : 0;
            o->has_witness = v.witness.has_value() ? 1 : 0;
            o->has_base = v.witness_base.has_value() ? 1 : 0;
            if (v.witness && w) std::memcpy(w, v.witness->data().data(), v.witness->data().size() * sizeof(double));
            if (v.witness_base && base)
                std::memcpy(base, v.witness_base->data().data(), v.witness_base->data().size() * sizeof(double));
        };
        fill(r.condition_a, a, a_witness, nullptr);
        fill(r.condition_b, b, b_witness, b_base);
    });
}



int fcref_loss_decomposed(void* h, const double* x, uint64_t c, unsigned workers, double* loss) {
    return guarded([&] {
        const auto& s = *static_cast<SparseSimilarity*>(h);
        const auto m = wrap(x, c, s.size());
        *loss = loss_decomposed(m, s, share_matrix(m, workers), workers);
    });
}

int fcref_gpa_step_fused(const double* x, uint64_t c, uint64_t n, const double* g, const double* xs,
                         double tau, unsigned workers, double* out) {
    return guarded([&] {
        const auto m = wrap(x, c, n);
        ShareMatrix share(c);
        for (std::size_t r = 0; r < c; ++r)
            for (std::size_t q = 0; q < c; ++q) share(r, q) = g[r * c + q];
        const std::vector<double> xsv(xs, xs + c * n);
        const auto next = gpa_step_fused(m, share, xsv, tau, workers);
        std::memcpy(out, next.data().data(), c * n * sizeof(double));
    });
}

double fcref_default_step_size(void* h) {
    const auto& s = *static_cast<SparseSimilarity*>(h);
    return default_step_size(s, s.size());
}

double fcref_fista_t_next(double t) { return fista_t_next(t); }

// method: 0 GPA, 1 FISTA.  Records carry the reference's own elapsed_ms.
int fcref_solve(void* h, double step_size, uint64_t max_iter, double tol, int method,
                uint64_t trace_every, int fista_restart, unsigned workers, uint64_t c,
                const double* x0, double* x_out, fcref_record* trace, uint64_t cap,
                fcref_summary* out) {
    return guarded([&] {
        const auto& s = *static_cast<SparseSimilarity*>(h);
        SolverConfig cfg;
        cfg.step_size = step_size;
        cfg.max_iter = max_iter;
        cfg.tol = tol;
        cfg.method = method == 1 ? Method::kFista : Method::kGpa;
        cfg.trace_every = trace_every;
        cfg.fista_restart = fista_restart != 0;
        cfg.workers = workers;
        const auto m = wrap(x0, c, s.size());
        const auto t0 = std::chrono::steady_clock::now();
        const SolverResult r = solve(m, s, cfg);
        const auto t1 = std::chrono::steady_clock::now();
        if (x_out) std::memcpy(x_out, r.membership.data().data(), c * s.size() * sizeof(double));
        for (std::size_t k = 0; k < r.trace.records.size() && k < cap; ++k) {
            trace[k].iteration = r.trace.records[k].iteration;
            trace[k].loss = r.trace.records[k].loss;
            trace[k].loss_increased = r.trace.records[k].loss_increased;
            trace[k].elapsed_ms = r.trace.records[k].elapsed_ms;
        }
        out->reason = static_cast<int32_t>(r.trace.reason);
        out->iterations = r.trace.iterations;
        out->final_loss = r.trace.final_loss;
        out->step_size = r.trace.step_size;
        out->n_records = r.trace.records.size();
        out->solve_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    });
}

}  // extern "C"
