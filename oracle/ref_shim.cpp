// oracle/ref_shim.cpp -- C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against
// /root/reference/proj/include (read-only, never copied) into
// oracle/_ref/libref_laplex.so.  It is the ground truth the C restatement in
// laplex_oracle.c is pinned against, and the "reference" arm of bench.py's
// CPU baseline.  Each entry mirrors one reference call:
//   LaplexOperator ctor        operator.hpp:81-137
//   transposed()               operator.hpp:157-159
//   matvec / matvec_transpose  operator.hpp:162-172
//   batch_matvec               operator.hpp:176-188
//   phased_matvec              operator.hpp:197-213
//   weighted_gram/phased_gram  operator.hpp:191-248
//   matvec_vjp                 gradients.hpp:110-135
//   phased_matvec_vjp          gradients.hpp:139-184
//   gram_vjp_weights           gradients.hpp:190-219
//   sort_anchors / scans       scan.hpp:27-73
// Exceptions map to the same integer codes the product C-ABI uses.
#include <cstdint>
#include <cstring>
#include <vector>

#include "laplex/laplex.hpp"

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const laplex::EmptyInput&) {
        return 1;
    } catch (const laplex::NonFinite&) {
        return 2;
    } catch (const laplex::DimensionMismatch&) {
        return 3;
    } catch (const laplex::PhasePresent&) {
        return 4;
    } catch (const laplex::PhaseAbsent&) {
        return 5;
    } catch (const laplex::AsymmetricCotangent&) {
        return 6;
    } catch (...) {
        return 99;
    }
}

template <class R>
std::vector<R> vec(const R* p, size_t m) {
    return p ? std::vector<R>(p, p + m) : std::vector<R>{};
}

template <class R>
void put(const std::vector<R>& v, R* out) {
    if (out) std::memcpy(out, v.data(), v.size() * sizeof(R));
}

laplex::Dispatch disp(int d) {
    return d == 1 ? laplex::Dispatch::ForceA : d == 2 ? laplex::Dispatch::ForceB : laplex::Dispatch::Auto;
}

}  // namespace

#define LXR_DEFINE(R, SFX)                                                                            \
    extern "C" int lxr_op_create##SFX(const R* a, size_t n, const R* b, size_t k, R t, const R* phi,  \
                                      const R* psi, void** out) {                                      \
        *out = nullptr;                                                                                \
        return guarded([&] {                                                                           \
            *out = new laplex::LaplexOperator<R>(vec(a, n), vec(b, k), t, vec(phi, phi ? n : 0),       \
                                                 vec(psi, psi ? k : 0));                               \
        });                                                                                            \
    }                                                                                                  \
    extern "C" void lxr_op_destroy##SFX(void* op) { delete static_cast<laplex::LaplexOperator<R>*>(op); } \
    extern "C" int lxr_op_transposed##SFX(void* op_, void** out) {                                    \
        *out = nullptr;                                                                                \
        return guarded([&] {                                                                           \
            *out = new laplex::LaplexOperator<R>(static_cast<laplex::LaplexOperator<R>*>(op_)->transposed()); \
        });                                                                                            \
    }                                                                                                  \
    extern "C" void lxr_op_sorted##SFX(void* op_, int side, R* values, uint64_t* perm, R* decays) {   \
        auto* op = static_cast<laplex::LaplexOperator<R>*>(op_);                                       \
        const auto& s = side == 0 ? op->sorted_rows() : op->sorted_cols();                             \
        put(s.values, values);                                                                         \
        if (perm)                                                                                      \
            for (size_t i = 0; i < s.perm.size(); ++i) perm[i] = s.perm[i];                            \
        put(s.decays, decays);                                                                         \
    }                                                                                                  \
    extern "C" void lxr_op_ranks##SFX(void* op_, int side, uint64_t* ranks) {                          \
        auto* op = static_cast<laplex::LaplexOperator<R>*>(op_);                                       \
        const auto& r = side == 0 ? op->row_buckets() : op->col_buckets();                             \
        for (size_t i = 0; i < r.size(); ++i) ranks[i] = r[i];                                         \
    }                                                                                                  \
    extern "C" int lxr_matvec##SFX(void* op_, const R* x, size_t xl, int d, R* y) {                    \
        auto* op = static_cast<laplex::LaplexOperator<R>*>(op_);                                       \
        return guarded([&] { put(op->matvec(vec(x, xl), disp(d)), y); });                              \
    }                                                                                                  \
    extern "C" int lxr_matvec_transpose##SFX(void* op_, const R* g, size_t gl, int d, R* y) {          \
        auto* op = static_cast<laplex::LaplexOperator<R>*>(op_);                                       \
        return guarded([&] { put(op->matvec_transpose(vec(g, gl), disp(d)), y); });                    \
    }                                                                                                  \
    extern "C" int lxr_batch_matvec##SFX(void* op_, const R* X, size_t B, size_t cols, int d, R* Y) {  \
        auto* op = static_cast<laplex::LaplexOperator<R>*>(op_);                                       \
        return guarded([&] {                                                                           \
            laplex::Matrix<R> M(B, cols);                                                              \
            std::memcpy(M.data.data(), X, B * cols * sizeof(R));                                       \
            put(op->batch_matvec(M, disp(d)).data, Y);                                                 \
        });                                                                                            \
    }                                                                                                  \
    extern "C" int lxr_phased_matvec##SFX(void* op_, const R* x, size_t xl, int d, R* y) {             \
        auto* op = static_cast<laplex::LaplexOperator<R>*>(op_);                                       \
        return guarded([&] { put(op->phased_matvec(vec(x, xl), disp(d)), y); });                       \
    }                                                                                                  \
    extern "C" int lxr_weighted_gram##SFX(void* op_, const R* D, size_t dl, R* M) {                    \
        auto* op = static_cast<laplex::LaplexOperator<R>*>(op_);                                       \
        return guarded([&] { put(op->weighted_gram(vec(D, dl)).matrix.data, M); });                   \
    }                                                                                                  \
    extern "C" int lxr_phased_gram##SFX(void* op_, const R* D, size_t dl, R* M) {                      \
        auto* op = static_cast<laplex::LaplexOperator<R>*>(op_);                                       \
        return guarded([&] { put(op->phased_gram(vec(D, dl)).matrix.data, M); });                      \
    }                                                                                                  \
    extern "C" int lxr_matvec_vjp##SFX(void* op_, const R* x, size_t xl, const R* g, size_t gl,        \
                                       R* xb, R* ab, R* bb) {                                          \
        auto* op = static_cast<laplex::LaplexOperator<R>*>(op_);                                       \
        return guarded([&] {                                                                           \
            auto c = laplex::matvec_vjp(*op, vec(x, xl), vec(g, gl));                                  \
            put(c.x_bar, xb);                                                                          \
            put(c.a_bar, ab);                                                                          \
            put(c.b_bar, bb);                                                                          \
        });                                                                                            \
    }                                                                                                  \
    extern "C" int lxr_phased_matvec_vjp##SFX(void* op_, const R* x, size_t xl, const R* g, size_t gl, \
                                              R* xb, R* ab, R* bb, R* pb, R* qb) {                     \
        auto* op = static_cast<laplex::LaplexOperator<R>*>(op_);                                       \
        return guarded([&] {                                                                           \
            auto c = laplex::phased_matvec_vjp(*op, vec(x, xl), vec(g, gl));                           \
            put(c.x_bar, xb);                                                                          \
            put(c.a_bar, ab);                                                                          \
            put(c.b_bar, bb);                                                                          \
            put(c.phi_bar, pb);                                                                        \
            put(c.psi_bar, qb);                                                                        \
        });                                                                                            \
    }                                                                                                  \
    extern "C" int lxr_gram_vjp_weights##SFX(void* op_, const R* D, size_t dl, const R* Gb, size_t gr, \
                                             size_t gc, R* Db) {                                       \
        auto* op = static_cast<laplex::LaplexOperator<R>*>(op_);                                       \
        return guarded([&] {                                                                           \
            laplex::Matrix<R> G(gr, gc);                                                               \
            std::memcpy(G.data.data(), Gb, gr * gc * sizeof(R));                                       \
            put(laplex::gram_vjp_weights(*op, vec(D, dl), G), Db);                                     \
        });                                                                                            \
    }                                                                                                  \
    extern "C" int lxr_sort_anchors##SFX(const R* raw, size_t m, R* values, uint64_t* perm, R* decays) { \
        return guarded([&] {                                                                           \
            auto s = laplex::sort_anchors(vec(raw, m));                                                \
            put(s.values, values);                                                                     \
            if (perm)                                                                                  \
                for (size_t i = 0; i < s.perm.size(); ++i) perm[i] = s.perm[i];                        \
            put(s.decays, decays);                                                                     \
        });                                                                                            \
    }                                                                                                  \
    extern "C" int lxr_decay_scan##SFX(const R* sorted_values, size_t m, const R* payload, R* prefix,  \
                                       R* suffix) {                                                    \
        return guarded([&] {                                                                           \
            laplex::SortedAnchors<R> s;                                                                \
            s.values = vec(sorted_values, m);                                                          \
            s.perm.resize(m);                                                                          \
            s.decays.resize(m > 0 ? m - 1 : 0);                                                        \
            for (size_t i = 0; i + 1 < m; ++i) s.decays[i] = std::exp(s.values[i] - s.values[i + 1]);  \
            if (prefix) put(laplex::prefix_decay_scan(s, vec(payload, m)), prefix);                    \
            if (suffix) put(laplex::suffix_decay_scan(s, vec(payload, m)), suffix);                    \
        });                                                                                            \
    }

LXR_DEFINE(double, _f64)
LXR_DEFINE(float, _f32)

// std::mt19937_64 + uniform_real_distribution<double>: the reference's input
// recipe (tests/helpers.hpp:12-24); used to pin oracle.Mt19937_64Uniform.
#include <random>
extern "C" void lxr_mt_uniform(uint64_t seed, size_t n, double lo, double hi, double* out) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> d(lo, hi);
    for (size_t i = 0; i < n; ++i) out[i] = d(g);
}
