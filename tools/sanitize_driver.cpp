// tools/sanitize_driver.cpp -- a small, torch-free driver of the C-ABI for
// compute-sanitizer (tests/test_sanitizer_gpu.py): one plan build (device
// radix sort, partition, store order), forward, transpose, backward, phased
// forward/backward, Gram-vector and the free sort / scan, at a size given on
// the command line.  Exit code 0 when every call returns LAPLEX_OK.
//
//   sanitize_driver <n> [rows]
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../include/laplex_c.h"

#define CK(x)                                                                         \
    do {                                                                              \
        int rc_ = (x);                                                                \
        if (rc_ != LAPLEX_OK) {                                                       \
            std::fprintf(stderr, "%s -> %d: %s\n", #x, rc_, laplex_last_error());     \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 5000;
    const size_t rows = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 2;
    const size_t k = n + n / 3 + 1;
    std::mt19937_64 rng(42);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    std::vector<float> a(n), b(k), phi(n), psi(k), X(rows * k), G(rows * n);
    for (auto& v : a) v = (float)(20 * U(rng));
    for (auto& v : b) v = (float)(20 * U(rng));
    for (size_t i = 0; i < n / 4; ++i) b[i] = a[i];  // exact ties
    for (auto& v : phi) v = (float)(3 + 3 * U(rng));
    for (auto& v : psi) v = (float)(3 + 3 * U(rng));
    for (auto& v : X) v = (float)U(rng);
    for (auto& v : G) v = (float)U(rng);
    std::vector<float> Y(rows * n), Yt(rows * k), xb(rows * k), ab(n), bb(k), pb(n), qb(k), Z(rows * k);

    laplex_plan p = nullptr, q = nullptr;
    CK(laplex_plan_create(LAPLEX_F32, a.data(), n, b.data(), k, 0.7, nullptr, nullptr, &p));
    CK(laplex_apply(p, 0u, X.data(), rows, k, Y.data()));
    CK(laplex_apply(p, LAPLEX_TRANSPOSE, G.data(), rows, n, Yt.data()));
    CK(laplex_backward(p, 0u, X.data(), rows, k, G.data(), n, xb.data(), ab.data(), bb.data(), nullptr, nullptr));
    CK(laplex_gram_apply(p, X.data(), rows, k, Z.data()));
    CK(laplex_plan_release(p));

    CK(laplex_plan_create(LAPLEX_F32, a.data(), n, b.data(), k, 0.7, phi.data(), psi.data(), &q));
    CK(laplex_apply(q, LAPLEX_PHASED, X.data(), rows, k, Y.data()));
    CK(laplex_backward(q, LAPLEX_PHASED, X.data(), rows, k, G.data(), n, xb.data(), ab.data(), bb.data(), pb.data(),
                       qb.data()));
    CK(laplex_plan_release(q));

    std::vector<float> vals(n), pre(n), suf(n), dec(n);
    std::vector<uint64_t> perm(n);
    CK(laplex_sort(LAPLEX_F32, a.data(), n, vals.data(), perm.data(), dec.data()));
    CK(laplex_scan(LAPLEX_F32, vals.data(), n, G.data(), pre.data(), suf.data()));
    std::printf("ok n=%zu k=%zu rows=%zu y0=%g xb0=%g\n", n, k, rows, (double)Y[0], (double)xb[0]);
    return 0;
}
