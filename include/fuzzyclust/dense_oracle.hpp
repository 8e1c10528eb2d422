// fuzzyclust/dense_oracle.hpp -- host-side dense test oracles, the names and contracts of
// objective.hpp:225-329 (kDenseOracleMaxN, dense_similarity, gradient_dense_reference,
// loss_dense_reference, hvp_dense_reference).  Written fresh for the drop-in so the
// reference's own suites (objective_test.cpp, solver_test.cpp, support.hpp) compile
// against include/ unchanged.  They materialise the N x N similarity, so they are
// guarded to N <= kDenseOracleMaxN and never touch the device: they are the
// independent brute-force cross-check of the device operators, not a fallback.
//
// Formulas (X is C x N, columns = nodes; M = S - X^T X):
//   f(X)     = sum_ij M_ij^2
//   grad f   = -4 X M
//   H[V]     = -4 V M + 4 X (V^T X + X^T V)
#pragma once

#include <cstddef>
#include <span>
#include <vector>

#include "fuzzyclust/common.hpp"
#include "fuzzyclust/dense.hpp"
#include "fuzzyclust/sparse.hpp"

namespace fuzzyclust {

inline constexpr std::size_t kDenseOracleMaxN = 5000;

namespace dense_oracle_detail {

inline void guard(std::size_t n) {
    if (n > kDenseOracleMaxN) throw InvalidInput("dense oracle: N exceeds guard");
}

// <a_i, b_j> over the C components of columns i and j
inline double column_dot(const DenseMatrix& a, std::size_t i, const DenseMatrix& b, std::size_t j) {
    const auto u = a.col(i);
    const auto w = b.col(j);
    double s = 0.0;
    for (std::size_t k = 0; k < u.size(); ++k) s += u[k] * w[k];
    return s;
}

// M = S - X^T X, row-major N x N
inline std::vector<double> residual(const DenseMatrix& x, std::span<const double> s) {
    const std::size_t n = x.cols();
    guard(n);
    if (s.size() != n * n) throw InvalidInput("dense oracle: similarity shape mismatch");
    std::vector<double> m(s.begin(), s.end());
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) m[i * n + j] -= column_dot(x, i, x, j);
    return m;
}

// out[:, j] += scale * sum_i a[:, i] * m[i][j]   (a is C x N, m row-major N x N)
inline void accumulate_times(DenseMatrix& out, const DenseMatrix& a, const std::vector<double>& m, double scale) {
    const std::size_t n = a.cols(), c = a.rows();
    std::vector<double> col(c);
    for (std::size_t j = 0; j < n; ++j) {
        std::fill(col.begin(), col.end(), 0.0);
        for (std::size_t i = 0; i < n; ++i) {
            const double mij = m[i * n + j];
            if (mij == 0.0) continue;
            const auto ai = a.col(i);
            for (std::size_t k = 0; k < c; ++k) col[k] += ai[k] * mij;
        }
        auto oj = out.col(j);
        for (std::size_t k = 0; k < c; ++k) oj[k] += scale * col[k];
    }
}

}  // namespace dense_oracle_detail

/// Row-major dense copy of S (N <= kDenseOracleMaxN).
inline std::vector<double> dense_similarity(const SparseSimilarity& s) {
    const std::size_t n = s.size();
    dense_oracle_detail::guard(n);
    std::vector<double> d(n * n, 0.0);
    for (std::size_t j = 0; j < n; ++j) {
        const auto r = s.col_rows(j);
        const auto v = s.col_values(j);
        for (std::size_t k = 0; k < r.size(); ++k) d[static_cast<std::size_t>(r[k]) * n + j] = v[k];
    }
    return d;
}

/// -4 X (S - X^T X), any X (test oracle).
inline DenseMatrix gradient_dense_reference(const DenseMatrix& x, std::span<const double> s_dense) {
    const auto m = dense_oracle_detail::residual(x, s_dense);
    DenseMatrix out(x.rows(), x.cols());
    dense_oracle_detail::accumulate_times(out, x, m, -4.0);
    return out;
}

/// ||S - X^T X||_F^2, evaluated densely.
inline double loss_dense_reference(const DenseMatrix& x, std::span<const double> s_dense) {
    const auto m = dense_oracle_detail::residual(x, s_dense);
    double f = 0.0;
    for (double e : m) f += e * e;
    return f;
}

/// -4 V (S - X^T X) + 4 X (V^T X + X^T V), evaluated densely.
inline DenseMatrix hvp_dense_reference(const DenseMatrix& xbar, const DenseMatrix& v,
                                       std::span<const double> s_dense) {
    const std::size_t n = xbar.cols();
    const auto m = dense_oracle_detail::residual(xbar, s_dense);
    DenseMatrix out(xbar.rows(), n);
    dense_oracle_detail::accumulate_times(out, v, m, -4.0);
    std::vector<double> w(n * n);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j)
            w[i * n + j] = dense_oracle_detail::column_dot(v, i, xbar, j) +
                           dense_oracle_detail::column_dot(xbar, i, v, j);
    dense_oracle_detail::accumulate_times(out, xbar, w, 4.0);
    return out;
}

}  // namespace fuzzyclust
