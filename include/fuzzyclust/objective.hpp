// fuzzyclust/objective.hpp -- drop-in for the objective core
// (objective.hpp:14-180): ShareMatrix, share_matrix / cross_share, the CSR
// column products, gradient and loss terms, fused_column_pass, loss_decomposed.
// Everything N-scaled runs on the device (libfuzzyclust_cuda.so); the C x C
// value-type methods of ShareMatrix are plain host code.  The Hessian-vector
// product (objective.hpp:182-223) runs on the device too; the
// dense N x N oracles (objective.hpp:225-329) are not part of this build.
#pragma once

#include <cmath>
#include <span>
#include <vector>

#include "fuzzyclust/common.hpp"
#include "fuzzyclust/dense.hpp"
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
/// Make an N-node similarity resident when only N matters (share_matrix).
inline void ensure_size(std::size_t n) {
    static SparseSimilarity ident;
    if (ident.size() != n) {
        std::vector<std::int64_t> rp(n + 1);
        std::vector<std::uint32_t> ci(n);
        for (std::size_t i = 0; i <= n; ++i) rp[i] = static_cast<std::int64_t>(i);
        for (std::size_t i = 0; i < n; ++i) ci[i] = static_cast<std::uint32_t>(i);
        ident = SparseSimilarity::from_csr(n, std::move(rp), std::move(ci), {}, false);
    }
    ident.ensure_resident();
}
inline bool resident_size_is(std::size_t n) {
    const auto& d = device::context();
    return d.resident != 0 && d.resident_n == n;
}
}  // namespace detail

/// X X^T (objective.hpp:92-95) on the device, 1024-column blocks combined in order.
inline ShareMatrix share_matrix(const DenseMatrix& x, unsigned /*workers*/ = 1) {
    if (!detail::resident_size_is(x.cols())) detail::ensure_size(x.cols());
    ShareMatrix out(x.rows());
    auto& d = device::context();
    device::check(fc_share_matrix(d.ctx, static_cast<uint32_t>(x.rows()), x.data().data(), out.raw()), d.ctx);
    return out;
}

/// A B^T (objective.hpp:61-90) on the device: the off-diagonal block of the Gram of
/// the stacked N x 2C matrix [A | B] -- same per-entry products, same block order.
inline ShareMatrix cross_share(const DenseMatrix& a, const DenseMatrix& b, unsigned /*workers*/ = 1) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) throw InvalidInput("cross_share: shape mismatch");
    if (!detail::resident_size_is(a.cols())) detail::ensure_size(a.cols());
    ShareMatrix out(a.rows());
    auto& d = device::context();
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

/// objective.hpp:98-109 (one column: runs the device sweep, O(nnz) per call).
inline void similarity_column_product(const DenseMatrix& x, const SparseSimilarity& s, std::size_t i,
                                      std::span<double> out) {
    const ColumnPass p = fused_column_pass(x, s);
    for (std::size_t k = 0; k < x.rows(); ++k) out[k] = p.xs[i * x.rows() + k];
}

/// objective.hpp:113-118
inline void gradient_column_fused(const ShareMatrix& share, std::span<const double> xs_i, std::span<const double> x_i,
                                  std::span<double> out) {
    auto& d = device::context();
    device::check(fc_gradient_rows(d.ctx, static_cast<uint32_t>(share.dim()), 1, share.raw(), xs_i.data(), x_i.data(),
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
