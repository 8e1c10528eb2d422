// fuzzyclust/objective.hpp -- drop-in for the objective core
// (objective.hpp:14-180): ShareMatrix, share_matrix / cross_share, the CSR
// column products, gradient and loss terms, fused_column_pass, loss_decomposed.
// Everything N-scaled runs on the device (libfuzzyclust_cuda.so); the C x C
// value-type methods of ShareMatrix are plain host code.  The Hessian-vector
// product (objective.hpp:182-223) runs on the device too; the
// dense N x N oracles (objective.hpp:225-329) are not part of this build.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <span>
#include <vector>

#include "fuzzyclust/common.hpp"
#include "fuzzyclust/dense.hpp"
#include "fuzzyclust/dense_oracle.hpp"
#include "fuzzyclust/device.hpp"
#include "fuzzyclust/parallel.hpp"
#include "fuzzyclust/sparse.hpp"

namespace fuzzyclust {

class ShareMatrix {
public:
    ShareMatrix() = default;
    explicit ShareMatrix(std::size_t c) : c_(c), v_(c * c, 0.0) {}
    std::size_t dim() const { return c_; }
    double operator()(std::size_t r, std::size_t c) const { return v_[r * c_ + c]; }
    double& operator()(std::size_t r, std::size_t c) { return v_[r * c_ + c]; }
    double frob_sq() const {
        double s = 0.0;
        for (double v : v_) s += v * v;
        return s;
    }
    double trace() const {
        double s = 0.0;
        for (std::size_t k = 0; k < c_; ++k) s += (*this)(k, k);
        return s;
    }
    void apply(std::span<const double> y, std::span<double> out) const {
        for (std::size_t k = 0; k < c_; ++k) {
            double acc = 0.0;
            for (std::size_t l = 0; l < c_; ++l) acc += v_[k * c_ + l] * y[l];
            out[k] = acc;
        }
    }
    void transpose_apply(std::span<const double> y, std::span<double> out) const {
        for (std::size_t k = 0; k < c_; ++k) {
            double acc = 0.0;
            for (std::size_t l = 0; l < c_; ++l) acc += v_[l * c_ + k] * y[l];
            out[k] = acc;
        }
    }
    double* raw() { return v_.data(); }
    const double* raw() const { return v_.data(); }

private:
    std::size_t c_ = 0;
    std::vector<double> v_;
};

namespace detail {
/// The context an N-only operator (Gram) runs on: the main one when its resident
/// similarity has N nodes, else the auxiliary one with an N-node identity pattern
/// (the main context's resident similarity stays where it is).
inline device::Context& context_for_size(std::size_t n) {
    auto& d = device::context();
    if (d.resident != 0 && d.resident_n == n) return d;
    auto& a = device::aux_context();
    if (a.resident_n != n || a.resident == 0) {
        std::vector<std::int64_t> rp(n + 1);
        std::vector<std::uint32_t> ci(n);
        for (std::size_t i = 0; i <= n; ++i) rp[i] = static_cast<std::int64_t>(i);
        for (std::size_t i = 0; i < n; ++i) ci[i] = static_cast<std::uint32_t>(i);
        device::check(fc_upload_csr(a.ctx, n, n, rp.data(), ci.data(), nullptr, static_cast<double>(n)), a.ctx);
        a.resident = device::next_id();
        a.resident_n = n;
    }
    return a;
}

/// 64-bit fingerprint of X's contents (every bit of every entry, order-sensitive).
inline std::uint64_t content_fingerprint(std::span<const double> v) {
    std::uint64_t h = 0x9E3779B97F4A7C15ULL ^ v.size();
    for (double e : v) {
        std::uint64_t u;
        std::memcpy(&u, &e, sizeof u);
        h = (h ^ u) * 0x100000001B3ULL;
        h ^= h >> 29;
    }
    return h;
}

/// The last device sweep, reused while (similarity, X) are unchanged: a reference-style
/// loop over columns (similarity_column_product / gradient_column / loss_terms_column
/// for i = 0..N-1) then costs one sweep plus an O(N C) host fingerprint per call,
/// not one O(nnz) sweep and an N x C upload per column.
struct SweepCache {
    std::uint64_t sim = 0, fp = 0;
    std::size_t rows = 0, cols = 0;
    std::vector<double> xs;
    double merge = 0.0;
};
inline SweepCache& sweep_cache() {
    static SweepCache c;
    return c;
}
}  // namespace detail

/// X X^T (objective.hpp:92-95) on the device, 1024-column blocks combined in order.
inline ShareMatrix share_matrix(const DenseMatrix& x, unsigned /*workers*/ = 1) {
    auto& d = detail::context_for_size(x.cols());
    ShareMatrix out(x.rows());
    device::check(fc_share_matrix(d.ctx, static_cast<uint32_t>(x.rows()), x.data().data(), out.raw()), d.ctx);
    return out;
}

/// A B^T (objective.hpp:61-90) on the device: the off-diagonal block of the Gram of
/// the stacked N x 2C matrix [A | B] -- same per-entry products, same block order.
inline ShareMatrix cross_share(const DenseMatrix& a, const DenseMatrix& b, unsigned /*workers*/ = 1) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) throw InvalidInput("cross_share: shape mismatch");
    auto& d = detail::context_for_size(a.cols());
    ShareMatrix out(a.rows());
    device::check(fc_cross_share(d.ctx, static_cast<uint32_t>(a.rows()), a.data().data(), b.data().data(), out.raw()),
                  d.ctx);
    return out;
}

struct ColumnPass {
    std::vector<double> xs;   ///< C x N column-major, column i = X s_i
    double merge = 0.0;
};

/// objective.hpp:151-173: one CSR sweep on the device.
inline ColumnPass fused_column_pass(const DenseMatrix& x, const SparseSimilarity& s, unsigned /*workers*/ = 1) {
    if (s.size() != x.cols()) throw InvalidInput("objective: similarity/membership size mismatch");
    s.ensure_resident();
    ColumnPass p;
    p.xs.resize(x.rows() * x.cols());
    auto& d = device::context();
    device::check(fc_fused_column_pass(d.ctx, static_cast<uint32_t>(x.rows()), x.data().data(), p.xs.data(), &p.merge),
                  d.ctx);
    return p;
}

/// objective.hpp:98-109.  One column of the device sweep; the sweep of (s, x) is cached
/// (detail::SweepCache), so looping over all columns runs it once.
inline void similarity_column_product(const DenseMatrix& x, const SparseSimilarity& s, std::size_t i,
                                      std::span<double> out) {
    if (s.size() != x.cols()) throw InvalidInput("objective: similarity/membership size mismatch");
    auto& c = detail::sweep_cache();
    const std::uint64_t fp = detail::content_fingerprint(x.data());
    if (c.sim != s.device_id() || c.fp != fp || c.rows != x.rows() || c.cols != x.cols()) {
        ColumnPass p = fused_column_pass(x, s);
        c.xs = std::move(p.xs);
        c.merge = p.merge;
        c.sim = s.device_id();
        c.fp = fp;
        c.rows = x.rows();
        c.cols = x.cols();
    }
    for (std::size_t k = 0; k < x.rows(); ++k) out[k] = c.xs[i * x.rows() + k];
}

/// Batched form (new): X s_i for every i in `cols`, one device sweep; C x |cols| column-major.
inline std::vector<double> similarity_column_products(const DenseMatrix& x, const SparseSimilarity& s,
                                                      std::span<const std::size_t> cols) {
    const ColumnPass p = fused_column_pass(x, s);
    std::vector<double> out(x.rows() * cols.size());
    for (std::size_t j = 0; j < cols.size(); ++j) {
        if (cols[j] >= x.cols()) throw InvalidInput("objective: column index out of range");
        for (std::size_t k = 0; k < x.rows(); ++k) out[j * x.rows() + k] = p.xs[cols[j] * x.rows() + k];
    }
    return out;
}

/// objective.hpp:113-118
inline void gradient_column_fused(const ShareMatrix& share, std::span<const double> xs_i, std::span<const double> x_i,
                                  std::span<double> out) {
    auto& d = device::context();
    device::check(fc_gradient_rows(d.ctx, static_cast<uint32_t>(share.dim()), 1, share.raw(), xs_i.data(), x_i.data(),
                                   out.data()),
                  d.ctx);
}

/// Batched form (new): gradient_column_fused for m columns at once (xs, x, out: C x m
/// column-major), one launch.
inline void gradient_columns_fused(const ShareMatrix& share, std::span<const double> xs, std::span<const double> x,
                                   std::span<double> out) {
    const std::size_t c = share.dim();
    if (c == 0 || xs.size() != x.size() || out.size() != x.size() || x.size() % c)
        throw InvalidInput("gradient_columns_fused: shape mismatch");
    auto& d = device::context();
    device::check(fc_gradient_rows(d.ctx, static_cast<uint32_t>(c), x.size() / c, share.raw(), xs.data(), x.data(),
                                   out.data()),
                  d.ctx);
}

/// objective.hpp:121-128
inline std::vector<double> gradient_column(const DenseMatrix& x, const ShareMatrix& share, const SparseSimilarity& s,
                                           std::size_t i) {
    std::vector<double> xs(x.rows()), out(x.rows());
    similarity_column_product(x, s, i, xs);
    gradient_column_fused(share, xs, x.col(i), out);
    return out;
}

/// objective.hpp:131-135
inline double loss_terms_column(std::span<const double> xs_i, std::span<const double> x_i) {
    double out = 0.0;
    auto& d = device::context();
    device::check(fc_loss_terms_rows(d.ctx, static_cast<uint32_t>(x_i.size()), 1, xs_i.data(), x_i.data(), &out),
                  d.ctx);
    return out;
}

/// Batched form (new): loss_terms_column for m columns (C x m column-major), one launch.
inline std::vector<double> loss_terms_columns(std::size_t c, std::span<const double> xs, std::span<const double> x) {
    if (c == 0 || xs.size() != x.size() || x.size() % c) throw InvalidInput("loss_terms_columns: shape mismatch");
    std::vector<double> out(x.size() / c);
    auto& d = device::context();
    device::check(fc_loss_terms_rows(d.ctx, static_cast<uint32_t>(c), out.size(), xs.data(), x.data(), out.data()),
                  d.ctx);
    return out;
}

/// objective.hpp:137-141
inline double loss_terms_column(const DenseMatrix& x, const SparseSimilarity& s, std::size_t i) {
    std::vector<double> xs(x.rows());
    similarity_column_product(x, s, i, xs);
    return loss_terms_column(xs, x.col(i));
}

/// objective.hpp:176-180: ||S||^2 + ||share||^2 - 2 merge
inline double loss_decomposed(const DenseMatrix& x, const SparseSimilarity& s, const ShareMatrix& share,
                              unsigned workers = 1) {
    const ColumnPass p = fused_column_pass(x, s, workers);
    return s.frob_sq() + share.frob_sq() - 2.0 * p.merge;
}

/// Hessian-vector product at xbar applied to v (objective.hpp:182-217), on the device:
/// column i = -4 (V s_i - A x_i - A^T x_i - B v_i), A = cross_share(V, X), B = X X^T.
inline DenseMatrix hessian_vector_product(const DenseMatrix& xbar, const DenseMatrix& v, const SparseSimilarity& s,
                                          unsigned /*workers*/ = 1) {
    if (xbar.rows() != v.rows() || xbar.cols() != v.cols()) throw InvalidInput("hessian_vector_product: shape mismatch");
    if (s.size() != xbar.cols()) throw InvalidInput("hessian_vector_product: similarity size mismatch");
    s.ensure_resident();
    DenseMatrix out(xbar.rows(), xbar.cols());
    auto& d = device::context();
    device::check(fc_hessian_vector_product(d.ctx, static_cast<uint32_t>(xbar.rows()), xbar.data().data(),
                                            v.data().data(), out.data().data()),
                  d.ctx);
    return out;
}

/// <H(xbar) v, v>_F (objective.hpp:219-223): the HVP on the device, then the
/// reference's single sequential frob_inner over the storage order on the host.
inline double quadratic_form(const DenseMatrix& xbar, const DenseMatrix& v, const SparseSimilarity& s,
                             unsigned workers = 1) {
    return frob_inner(hessian_vector_product(xbar, v, s, workers), v);
}

}  // namespace fuzzyclust
