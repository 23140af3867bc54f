// laplex/operator.hpp -- drop-in LaplexOperator<Real> on the B200 kernels.
//
// Same public surface, argument meaning, validation order and exception types
// as the reference class (proj/include/laplex/operator.hpp:64-248).  The
// object is a value type holding a shared, immutable device plan
// (laplex_plan, refcounted): copies are cheap, transposed() is a role-swapped
// view of the same plan (no re-sort, unlike operator.hpp:157-159), and the
// sorted-anchor / co-rank accessors are fetched from the device on first use.
// Dispatch is accepted and ignored: the device has one algorithm, and both
// reference branches agree with it to 1e-12 in fp64.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>

#include "laplex/common.hpp"
#include "laplex/errors.hpp"
#include "laplex/scan.hpp"
#include "laplex_c.h"

namespace laplex {

/// Explicit symmetric n x n Gram matrix M = A diag(D) A^T (bit-exactly symmetric).
template <typename Real>
struct GramResult {
    Matrix<Real> matrix;
};

enum class Dispatch {
    Auto,
    ForceA,
    ForceB,
};

template <typename Real>
class LaplexOperator {
    struct State {
        laplex_plan plan = nullptr;
        std::vector<Real> rows, cols, row_phases, col_phases;
        Real t = Real(1);
        std::mutex mu;
        bool have_sorted[2] = {false, false};
        SortedAnchors<Real> sorted[2];
        bool have_buckets[2] = {false, false};
        std::vector<std::size_t> buckets[2];  // [0] j_of_row, [1] r_of_col
        ~State() {
            if (plan) laplex_plan_release(plan);
        }
    };

  public:
    LaplexOperator(std::vector<Real> row_anchors, std::vector<Real> col_anchors, Real temperature = Real(1))
        : LaplexOperator(std::move(row_anchors), std::move(col_anchors), temperature, {}, {}) {}

    LaplexOperator(std::vector<Real> row_anchors, std::vector<Real> col_anchors, Real temperature,
                   std::vector<Real> row_phases, std::vector<Real> col_phases)
        : s_(std::make_shared<State>()) {
        State& s = *s_;
        s.rows = std::move(row_anchors);
        s.cols = std::move(col_anchors);
        s.t = temperature;
        s.row_phases = std::move(row_phases);
        s.col_phases = std::move(col_phases);
        // validation order of operator.hpp:88-101
        if (s.rows.empty() || s.cols.empty()) throw EmptyInput("LaplexOperator: empty anchor set");
        require_finite(s.rows, "LaplexOperator row anchors");
        require_finite(s.cols, "LaplexOperator col anchors");
        if (!(s.t > Real(0)) || !std::isfinite(s.t))
            throw NonFinite("LaplexOperator: temperature must be positive and finite");
        if (s.row_phases.empty() != s.col_phases.empty())
            throw DimensionMismatch("LaplexOperator: phases must be given for both sides");
        const bool phased = !s.row_phases.empty();
        if (phased) {
            if (s.row_phases.size() != s.rows.size() || s.col_phases.size() != s.cols.size())
                throw DimensionMismatch("LaplexOperator: phase lengths");
            require_finite(s.row_phases, "LaplexOperator row phases");
            require_finite(s.col_phases, "LaplexOperator col phases");
        }
        throw_for_code(laplex_plan_create(detail::dtype_tag<Real>(), s.rows.data(), s.rows.size(), s.cols.data(),
                                          s.cols.size(), static_cast<double>(s.t),
                                          phased ? s.row_phases.data() : nullptr,
                                          phased ? s.col_phases.data() : nullptr, &s.plan));
    }

    std::size_t n() const { return s_->rows.size(); }
    std::size_t k() const { return s_->cols.size(); }
    Real temperature() const { return s_->t; }
    bool has_phases() const { return !s_->row_phases.empty(); }

    const std::vector<Real>& row_anchors() const { return s_->rows; }
    const std::vector<Real>& col_anchors() const { return s_->cols; }
    const std::vector<Real>& row_phases() const { return s_->row_phases; }
    const std::vector<Real>& col_phases() const { return s_->col_phases; }

    /// Sorted, temperature-scaled anchors (copied from the device once).
    const SortedAnchors<Real>& sorted_rows() const { return sorted(LAPLEX_ROWS); }
    const SortedAnchors<Real>& sorted_cols() const { return sorted(LAPLEX_COLS); }
    /// r_of_col[j] = #{i : a_i <= b_j}, sorted order (operator.hpp:111-115).
    const std::vector<std::size_t>& col_buckets() const { return buckets(LAPLEX_COLS); }
    /// j_of_row[i] = #{j : b_j <= a_i}, sorted order (operator.hpp:116-120).
    const std::vector<std::size_t>& row_buckets() const { return buckets(LAPLEX_ROWS); }

    /// Role-swapped operator LAPLEX(b, a): a view of the same device plan.
    LaplexOperator transposed() const {
        LaplexOperator out;
        out.s_ = std::make_shared<State>();
        State& d = *out.s_;
        d.rows = s_->cols;
        d.cols = s_->rows;
        d.t = s_->t;
        d.row_phases = s_->col_phases;
        d.col_phases = s_->row_phases;
        throw_for_code(laplex_plan_transposed(s_->plan, &d.plan));
        return out;
    }

    std::vector<Real> matvec(const std::vector<Real>& x, Dispatch dispatch = Dispatch::Auto) const {
        if (has_phases()) throw PhasePresent("matvec: operator has phases, use phased_matvec");
        return apply(0u, x, "matvec", dispatch);
    }

    std::vector<Real> matvec_transpose(const std::vector<Real>& g, Dispatch dispatch = Dispatch::Auto) const {
        if (has_phases()) throw PhasePresent("matvec_transpose: operator has phases, use phased path");
        return apply(LAPLEX_TRANSPOSE, g, "matvec_transpose", dispatch);
    }

    Matrix<Real> batch_matvec(const Matrix<Real>& X, Dispatch = Dispatch::Auto) const {
        if (has_phases()) throw PhasePresent("batch_matvec: operator has phases");
        if (X.cols != k()) throw DimensionMismatch("batch_matvec: X columns");
        require_finite(X.data, "batch_matvec X");
        Matrix<Real> Y(X.rows, n());
        if (X.rows) throw_for_code(laplex_apply(s_->plan, 0u, X.data.data(), X.rows, X.cols, Y.data.data()));
        stats::matvec_calls().fetch_add(X.rows, std::memory_order_relaxed);
        return Y;
    }

    /// Extension (not a reference member): the Gram-vector product
    /// Y_r = A^T (A X_r) of SPEC.md:187, i.e. matvec_transpose(matvec(x)) per
    /// row in one device call; counts as the composition's two matvecs per row.
    Matrix<Real> batch_gram_matvec(const Matrix<Real>& X) const {
        if (has_phases()) throw PhasePresent("batch_gram_matvec: operator has phases");
        if (X.cols != k()) throw DimensionMismatch("batch_gram_matvec: X columns");
        require_finite(X.data, "batch_gram_matvec X");
        Matrix<Real> Y(X.rows, k());
        if (X.rows) throw_for_code(laplex_gram_apply(s_->plan, X.data.data(), X.rows, X.cols, Y.data.data()));
        stats::matvec_calls().fetch_add(2 * X.rows, std::memory_order_relaxed);
        return Y;
    }

    GramResult<Real> weighted_gram(const std::vector<Real>& D) const {
        if (has_phases()) throw PhasePresent("weighted_gram: operator has phases");
        return gram(0u, D, "weighted_gram", 1);
    }

    /// Angle-sum reduction; counts as exactly two plain matvecs (operator.hpp:196-213).
    std::vector<Real> phased_matvec(const std::vector<Real>& x, Dispatch = Dispatch::Auto) const {
        if (!has_phases()) throw PhaseAbsent("phased_matvec: operator has no phases");
        if (x.size() != k()) throw DimensionMismatch("phased_matvec: x length");
        require_finite(x, "phased_matvec x");
        std::vector<Real> y(n());
        throw_for_code(laplex_apply(s_->plan, LAPLEX_PHASED, x.data(), 1, x.size(), y.data()));
        stats::matvec_calls().fetch_add(2, std::memory_order_relaxed);
        return y;
    }

    /// Three-real-Gram reduction; counts as exactly three plain Grams (operator.hpp:215-248).
    GramResult<Real> phased_gram(const std::vector<Real>& D) const {
        if (!has_phases()) throw PhaseAbsent("phased_gram: operator has no phases");
        return gram(LAPLEX_PHASED, D, "phased_gram", 3);
    }

    /// The underlying C-ABI plan (for device-pointer entry points).
    laplex_plan plan() const { return s_->plan; }

  private:
    LaplexOperator() = default;

    std::vector<Real> apply(unsigned flags, const std::vector<Real>& v, const char* what, Dispatch) const {
        const std::size_t in_len = (flags & LAPLEX_TRANSPOSE) ? n() : k();
        if (v.size() != in_len) throw DimensionMismatch(std::string(what) + ": x length");
        require_finite(v, what);
        std::vector<Real> y((flags & LAPLEX_TRANSPOSE) ? k() : n());
        throw_for_code(laplex_apply(s_->plan, flags, v.data(), 1, v.size(), y.data()));
        stats::matvec_calls().fetch_add(1, std::memory_order_relaxed);
        return y;
    }

    GramResult<Real> gram(unsigned flags, const std::vector<Real>& D, const char* what, int calls) const {
        if (D.size() != k()) throw DimensionMismatch(std::string(what) + ": D length");
        require_finite(D, what);
        GramResult<Real> out;
        out.matrix = Matrix<Real>(n(), n());
        throw_for_code(laplex_gram(s_->plan, flags, D.data(), D.size(), out.matrix.data.data()));
        stats::weighted_gram_calls().fetch_add(calls, std::memory_order_relaxed);
        return out;
    }

    const SortedAnchors<Real>& sorted(int side) const {
        State& s = *s_;
        std::lock_guard<std::mutex> g(s.mu);
        if (!s.have_sorted[side]) {
            const std::size_t m = side == LAPLEX_ROWS ? n() : k();
            SortedAnchors<Real>& out = s.sorted[side];
            out.values.resize(m);
            out.decays.resize(m - 1);
            std::vector<std::uint64_t> perm(m);
            throw_for_code(laplex_plan_sorted(s.plan, side, out.values.data(), perm.data(),
                                              m > 1 ? out.decays.data() : nullptr));
            out.perm = detail::widen(perm);
            s.have_sorted[side] = true;
        }
        return s.sorted[side];
    }

    const std::vector<std::size_t>& buckets(int side) const {
        State& s = *s_;
        std::lock_guard<std::mutex> g(s.mu);
        if (!s.have_buckets[side]) {
            std::vector<std::uint64_t> r(side == LAPLEX_ROWS ? n() : k());
            throw_for_code(laplex_plan_ranks(s.plan, side, 0, r.data()));
            s.buckets[side] = detail::widen(r);
            s.have_buckets[side] = true;
        }
        return s.buckets[side];
    }

    std::shared_ptr<State> s_;
};

}  // namespace laplex
