// laplex/scan.hpp -- drop-in for the reference scan core
// (proj/include/laplex/scan.hpp:17-86) on the B200 kernels.
//
//   sort_anchors       -> laplex_sort  (device onesweep radix sort; stable,
//                         -0 == +0 keep input order, sign of zero kept)
//   prefix/suffix_decay_scan -> laplex_scan (tiled anchored scan; every carry
//                         applied as exp(anchor difference))
//   symmetric_matvec   -> prefix + (suffix - x), as scan.hpp:83-85
#pragma once

#include <cstddef>
#include <type_traits>
#include <vector>

#include "laplex/common.hpp"
#include "laplex/errors.hpp"
#include "laplex_c.h"

namespace laplex {

template <typename Real>
struct SortedAnchors {
    std::vector<Real> values;       // ascending, duplicates allowed
    std::vector<std::size_t> perm;  // sorted index -> original index
    std::vector<Real> decays;       // exp(values[i] - values[i+1]), size()-1 entries

    std::size_t size() const { return values.size(); }
};

namespace detail {

template <typename Real>
constexpr int dtype_tag() {
    static_assert(std::is_same_v<Real, float> || std::is_same_v<Real, double>,
                  "the B200 LAPLEX path is instantiated for float and double");
    return std::is_same_v<Real, double> ? LAPLEX_F64 : LAPLEX_F32;
}

inline std::vector<std::size_t> widen(const std::vector<std::uint64_t>& v) {
    return std::vector<std::size_t>(v.begin(), v.end());
}

}  // namespace detail

template <typename Real>
SortedAnchors<Real> sort_anchors(const std::vector<Real>& raw) {
    if (raw.empty()) throw EmptyInput("sort_anchors: empty input");
    require_finite(raw, "sort_anchors");
    const std::size_t m = raw.size();
    SortedAnchors<Real> out;
    out.values.resize(m);
    out.decays.resize(m - 1);
    std::vector<std::uint64_t> perm(m);
    throw_for_code(laplex_sort(detail::dtype_tag<Real>(), raw.data(), m, out.values.data(), perm.data(),
                               m > 1 ? out.decays.data() : nullptr));
    out.perm = detail::widen(perm);
    return out;
}

namespace detail {

template <typename Real>
std::vector<Real> run_scan(const SortedAnchors<Real>& anchors, const std::vector<Real>& payload, bool prefix,
                           const char* what) {
    const std::size_t m = anchors.size();
    if (payload.size() != m) throw DimensionMismatch(std::string(what) + ": payload length");
    std::vector<Real> out(m);
    if (m == 0) return out;
    throw_for_code(laplex_scan(dtype_tag<Real>(), anchors.values.data(), m, payload.data(),
                               prefix ? out.data() : nullptr, prefix ? nullptr : out.data()));
    return out;
}

}  // namespace detail

/// t_i = sum_{j <= i} exp(a_j - a_i) payload_j  (payload in sorted order).
template <typename Real>
std::vector<Real> prefix_decay_scan(const SortedAnchors<Real>& anchors, const std::vector<Real>& payload) {
    return detail::run_scan(anchors, payload, true, "prefix_decay_scan");
}

/// s_i = sum_{j >= i} exp(a_i - a_j) payload_j.
template <typename Real>
std::vector<Real> suffix_decay_scan(const SortedAnchors<Real>& anchors, const std::vector<Real>& payload) {
    return detail::run_scan(anchors, payload, false, "suffix_decay_scan");
}

/// y_i = sum_j exp(-|a_i - a_j|) x_j: both scans, diagonal subtracted once.
template <typename Real>
std::vector<Real> symmetric_matvec(const SortedAnchors<Real>& anchors, const std::vector<Real>& x) {
    if (x.size() != anchors.size()) throw DimensionMismatch("symmetric_matvec: x length");
    std::vector<Real> y = prefix_decay_scan(anchors, x);
    const std::vector<Real> s = suffix_decay_scan(anchors, x);
    for (std::size_t i = 0; i < y.size(); ++i) y[i] += s[i] - x[i];
    return y;
}

}  // namespace laplex
