// laplex/gradients.hpp -- drop-in VJPs (proj/include/laplex/gradients.hpp:
// 17-219) on the B200 backward kernels.
//
// matvec_vjp / phased_matvec_vjp run ONE fused device pass (x_bar, a_bar,
// b_bar and, phased, phi_bar/psi_bar) instead of the reference's re-sorted
// transpose plus split-sum passes.  x_bar is bit-identical to
// op.matvec_transpose(g).  Tie subgradient 0 as in the
// reference.  The stats counters advance exactly as the reference's
// decomposition would (1 matvec for matvec_vjp, 4 for phased_matvec_vjp,
// n for gram_vjp_weights).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <vector>

#include "laplex/common.hpp"
#include "laplex/errors.hpp"
#include "laplex/operator.hpp"
#include "laplex/scan.hpp"
#include "laplex_c.h"

namespace laplex {

template <typename Real>
struct MatvecCotangents {
    std::vector<Real> x_bar;
    std::vector<Real> a_bar;
    std::vector<Real> b_bar;
    std::vector<Real> phi_bar;  // empty for the unphased VJP
    std::vector<Real> psi_bar;
};

namespace detail {

template <typename Real>
MatvecCotangents<Real> run_vjp(const LaplexOperator<Real>& op, const std::vector<Real>& x,
                               const std::vector<Real>& g, bool phased, const char* what) {
    if (x.size() != op.k()) throw DimensionMismatch(std::string(what) + ": x length");
    if (g.size() != op.n()) throw DimensionMismatch(std::string(what) + ": g length");
    require_finite(x, what);
    require_finite(g, what);
    MatvecCotangents<Real> out;
    out.x_bar.resize(op.k());
    out.a_bar.resize(op.n());
    out.b_bar.resize(op.k());
    if (phased) {
        out.phi_bar.resize(op.n());
        out.psi_bar.resize(op.k());
    }
    throw_for_code(laplex_backward(op.plan(), phased ? LAPLEX_PHASED : 0u, x.data(), 1, x.size(), g.data(),
                                   g.size(), out.x_bar.data(), out.a_bar.data(), out.b_bar.data(),
                                   phased ? out.phi_bar.data() : nullptr, phased ? out.psi_bar.data() : nullptr));
    return out;
}

}  // namespace detail

/// Exact gradients of L = g^T matvec(op, x) (gradients.hpp:110-135).
template <typename Real>
MatvecCotangents<Real> matvec_vjp(const LaplexOperator<Real>& op, const std::vector<Real>& x,
                                  const std::vector<Real>& g) {
    if (op.has_phases()) throw PhasePresent("matvec_vjp: use phased_matvec_vjp");
    auto out = detail::run_vjp(op, x, g, false, "matvec_vjp");
    stats::matvec_calls().fetch_add(1, std::memory_order_relaxed);
    return out;
}

/// Gradients through the phased product, incl. phase cotangents (gradients.hpp:139-184).
template <typename Real>
MatvecCotangents<Real> phased_matvec_vjp(const LaplexOperator<Real>& op, const std::vector<Real>& x,
                                         const std::vector<Real>& g) {
    if (!op.has_phases()) throw PhaseAbsent("phased_matvec_vjp: operator has no phases");
    auto out = detail::run_vjp(op, x, g, true, "phased_matvec_vjp");
    stats::matvec_calls().fetch_add(4, std::memory_order_relaxed);
    return out;
}

/// d<G_bar, weighted_gram(op, D)>/dD for symmetric G_bar (gradients.hpp:190-219).
template <typename Real>
std::vector<Real> gram_vjp_weights(const LaplexOperator<Real>& op, const std::vector<Real>& D,
                                   const Matrix<Real>& G_bar) {
    if (op.has_phases()) throw PhasePresent("gram_vjp_weights: phased operator not supported");
    if (D.size() != op.k()) throw DimensionMismatch("gram_vjp_weights: D length");
    if (G_bar.rows != op.n() || G_bar.cols != op.n()) throw DimensionMismatch("gram_vjp_weights: G_bar shape");
    require_finite(G_bar.data, "gram_vjp_weights G_bar");
    std::vector<Real> out(op.k());
    throw_for_code(laplex_gram_vjp_weights(op.plan(), D.data(), D.size(), G_bar.data.data(), G_bar.rows,
                                           G_bar.cols, out.data()));
    stats::matvec_calls().fetch_add(op.n(), std::memory_order_relaxed);
    return out;
}

}  // namespace laplex
