// fuzzyclust/solver.hpp -- drop-in for the solver drivers (solver.hpp:18-295).
// run_gpa / run_fista / solve execute the whole iteration loop on the device
// (fc_solve): loss, stop rule, FISTA momentum and restart are decided by the
// device, bit-identically to the reference.  New: Method::kFistaBacktracking
// (Beck-Teboulle line search; the reference has none).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <ostream>
#include <string>
#include <vector>

#include "fuzzyclust/common.hpp"
#include "fuzzyclust/device.hpp"
#include "fuzzyclust/membership.hpp"
#include "fuzzyclust/objective.hpp"
#include "fuzzyclust/parallel.hpp"
#include "fuzzyclust/sparse.hpp"

namespace fuzzyclust {

enum class Method { kGpa, kFista, kFistaBacktracking };

enum class TerminationReason { kTolReached, kMaxIter, kLossIncreaseFista };

inline const char* to_string(TerminationReason r) {
    switch (r) {
        case TerminationReason::kTolReached: return "tol_reached";
        case TerminationReason::kMaxIter: return "max_iter";
        case TerminationReason::kLossIncreaseFista: return "loss_increase_fista";
    }
    return "unknown";
}

struct SolverConfig {
    double step_size = 0.0;          ///< <= 0 selects default_step_size
    std::size_t max_iter = 100000;
    double tol = 0.0;
    Method method = Method::kGpa;
    std::size_t trace_every = 1;
    bool fista_restart = false;
    unsigned workers = 1;            ///< accepted for signature parity; the device ignores it
    double bt_eta = 2.0;             ///< new: backtracking growth of L = 1/step
    unsigned bt_max = 30;            ///< new: max backtracks per iteration

    void validate() const {
        if (max_iter < 1) throw InvalidInput("solver: max_iter must be >= 1");
        if (tol < 0.0) throw InvalidInput("solver: tol must be >= 0");
        if (trace_every < 1) throw InvalidInput("solver: trace_every must be >= 1");
        if (!(step_size > 0.0) && step_size != 0.0)
            throw InvalidInput("solver: step_size must be positive (or 0 for auto)");
    }
};

struct TraceRecord {
    std::size_t iteration = 0;
    double loss = 0.0;
    double elapsed_ms = 0.0;
    bool loss_increased = false;
    unsigned backtracks = 0;         ///< new
    double step = 0.0;               ///< new: step used at this record
};

struct SolverTrace {
    std::vector<TraceRecord> records;
    TerminationReason reason = TerminationReason::kMaxIter;
    std::size_t iterations = 0;
    double final_loss = 0.0;
    double step_size = 0.0;
};

struct SolverResult {
    MembershipMatrix membership;
    SolverTrace trace;
};

inline double fista_t_next(double t) { return (1.0 + std::sqrt(1.0 + 4.0 * t * t)) / 2.0; }

inline double default_step_size(const SparseSimilarity& s, std::size_t n) {
    return 1.0 / (4.0 * s.frob_norm() + 12.0 * static_cast<double>(n));
}

inline double resolve_step_size(const SolverConfig& config, const SparseSimilarity& s, std::size_t n) {
    return config.step_size > 0.0 ? config.step_size : default_step_size(s, n);
}

/// solver.hpp:89-107 (one projected-gradient update from precomputed X s_i).
inline MembershipMatrix gpa_step_fused(const MembershipMatrix& x, const ShareMatrix& share,
                                       const std::vector<double>& xs, double tau, unsigned /*workers*/ = 1) {
    auto& d = detail::context_for_size(x.nodes());
    MembershipMatrix next(x.clusters(), x.nodes());
    device::check(fc_gpa_step_fused(d.ctx, static_cast<uint32_t>(x.clusters()), x.data().data(), share.raw(),
                                    xs.data(), tau, next.data().data()),
                  d.ctx);
    return next;
}

/// solver.hpp:110-114
inline MembershipMatrix gpa_step(const MembershipMatrix& x, const SparseSimilarity& s, const ShareMatrix& share,
                                 double tau, unsigned /*workers*/ = 1) {
    if (s.size() != x.nodes()) throw InvalidInput("objective: similarity/membership size mismatch");
    s.ensure_resident();
    MembershipMatrix next(x.clusters(), x.nodes());
    auto& d = device::context();
    device::check(fc_gpa_step(d.ctx, static_cast<uint32_t>(x.clusters()), x.data().data(), share.raw(), tau,
                              next.data().data()),
                  d.ctx);
    return next;
}

namespace detail {
inline SolverResult run_on_device(const MembershipMatrix& x0, const SparseSimilarity& s, const SolverConfig& config,
                                  Method method, const char* who) {
    config.validate();
    if (s.size() != x0.nodes()) {
        x0.validate(1e-9);
        throw InvalidInput(std::string(who) + ": similarity/membership size mismatch");
    }
    s.ensure_resident();
    fc_solver_config c{};
    c.step_size = config.step_size;
    c.max_iter = config.max_iter;
    c.tol = config.tol;
    c.method = method == Method::kGpa ? FC_GPA : method == Method::kFista ? FC_FISTA : FC_FISTA_BT;
    c.fista_restart = config.fista_restart ? 1 : 0;
    c.trace_every = config.trace_every;
    c.bt_eta = config.bt_eta;
    c.bt_max = config.bt_max;
    const std::size_t cap = std::min<std::size_t>(config.max_iter + 2, std::size_t(1) << 20);
    std::vector<fc_trace_record> rec(cap);
    fc_solve_summary sum{};
    SolverResult r;
    r.membership = MembershipMatrix(x0.clusters(), x0.nodes());
    auto& d = device::context();
    device::check(fc_solve(d.ctx, &c, static_cast<uint32_t>(x0.clusters()), x0.data().data(),
                           r.membership.data().data(), rec.data(), cap, &sum),
                  d.ctx);
    const std::size_t k = std::min<std::size_t>(sum.n_records, cap);
    r.trace.records.reserve(k);
    for (std::size_t i = 0; i < k; ++i)
        r.trace.records.push_back({rec[i].iteration, rec[i].loss, rec[i].elapsed_ms, rec[i].loss_increased != 0,
                                   static_cast<unsigned>(rec[i].backtracks), rec[i].step});
    r.trace.reason = static_cast<TerminationReason>(sum.reason);
    r.trace.iterations = sum.iterations;
    r.trace.final_loss = sum.final_loss;
    r.trace.step_size = sum.step_size;
    return r;
}
}  // namespace detail

/// Algorithm 3 (solver.hpp:137-180)
inline SolverResult run_gpa(const MembershipMatrix& x0, const SparseSimilarity& s, const SolverConfig& config) {
    return detail::run_on_device(x0, s, config, Method::kGpa, "run_gpa");
}

/// Algorithm 4 (solver.hpp:188-272); kFistaBacktracking adds the line search.
inline SolverResult run_fista(const MembershipMatrix& x0, const SparseSimilarity& s, const SolverConfig& config) {
    const Method m = config.method == Method::kFistaBacktracking ? Method::kFistaBacktracking : Method::kFista;
    return detail::run_on_device(x0, s, config, m, "run_fista");
}

inline SolverResult solve(const MembershipMatrix& x0, const SparseSimilarity& s, const SolverConfig& config) {
    return config.method == Method::kGpa ? run_gpa(x0, s, config) : run_fista(x0, s, config);
}

/// solver.hpp:282-295
inline void write_trace_csv(const SolverTrace& trace, std::ostream& out, bool include_timing = false) {
    out << (include_timing ? "iteration,loss,elapsed_ms\n" : "iteration,loss\n");
    char buf[32];
    for (const auto& r : trace.records) {
        std::snprintf(buf, sizeof buf, "%.17g", r.loss);
        out << r.iteration << ',' << buf;
        if (include_timing) {
            std::snprintf(buf, sizeof buf, "%.3f", r.elapsed_ms);
            out << ',' << buf;
        }
        out << '\n';
    }
}

}  // namespace fuzzyclust
