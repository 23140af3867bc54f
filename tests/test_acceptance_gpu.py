"""Analogues of the reference's acceptance checks that exercise the hot path
(proj/tests/acceptance.cpp checks 1, 3, 6, 12; checks 2, 4, 5 are in
test_parity_gpu.py).  Same seeds-style loops, same thresholds."""
import time

import numpy as np
import pytest

import oracle as O
import paper_2605_24584_b200 as L

pytestmark = pytest.mark.gpu


def test_check1_matvec_exactness_both_branches():
    # acceptance.cpp:66-90: 200 instances per branch, n,k <= 256, ties, <= 1e-12, < 10 s
    rng = np.random.default_rng(101)
    t0 = time.time()
    worst = 0.0
    for d in (L.Dispatch.ForceA, L.Dispatch.ForceB):
        for trial in range(200):
            n, k = rng.integers(1, 257, 2)
            a, b = rng.uniform(-6, 6, n), rng.uniform(-6, 6, k)
            if trial % 3 == 0:
                m = min(n, k) // 2 + 1
                b[rng.integers(0, k, m)] = a[rng.integers(0, n, m)]
            x = rng.uniform(-1, 1, k)
            t = 1.0 if trial % 2 else 0.42
            got = L.LaplexOperator(a, b, t).matvec(x, d)
            worst = max(worst, O.rel_err_l2(got, O.dense_matvec(a, b, t, x)))
    assert worst <= 1e-12
    assert time.time() - t0 < 10.0


def test_check3_phased_reductions():
    # acceptance.cpp:127-157 (call counts are pinned in the C++ drop-in suite)
    rng = np.random.default_rng(103)
    n, k = 96, 140
    a, b = rng.uniform(-4, 4, n), rng.uniform(-4, 4, k)
    phi, psi = rng.uniform(0, 6.28, n), rng.uniform(0, 6.28, k)
    x, D = rng.uniform(-1, 1, k), rng.uniform(-1, 1, k)
    op = L.LaplexOperator(a, b, 0.9, phi, psi)
    assert O.rel_err_l2(op.phased_matvec(x), O.dense_matvec(a, b, 0.9, x, phi, psi)) <= 1e-10
    assert O.rel_err_l2(op.phased_gram(D).matrix, O.dense_gram(a, b, 0.9, D, phi, psi)) <= 1e-10


def _best(f, reps=15):
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        best = min(best, time.perf_counter() - t0)
    return best


def test_check6_matvec_scaling():
    # acceptance.cpp:325-356: T(2^21)/T(2^17) <= 24 (matvec on a built plan, fp64)
    rng = np.random.default_rng(600)
    ops = {}
    for lg in (17, 21):
        n = 1 << lg
        a, b, x = rng.uniform(-100, 100, n), rng.uniform(-100, 100, n), rng.uniform(-1, 1, n)
        ops[lg] = (L.LaplexOperator(a, b, 1.0), x)
    for lg in ops:
        ops[lg][0].matvec(ops[lg][1])
    ts = {lg: _best(lambda lg=lg: ops[lg][0].matvec(ops[lg][1])) for lg in ops}
    assert ts[21] / ts[17] <= 24.0, ts


def test_check12_gram_plateau_and_growth():
    # acceptance.cpp:586-613: plateau T(2^13)/T(2^10) <= 2, growth T(2^16)/T(2^13) <= 8
    rng = np.random.default_rng(612)
    n = 32
    a = rng.uniform(-5, 5, n)
    ts = {}
    for lg in (10, 13, 16):
        k = 1 << lg
        b, D = rng.uniform(-5, 5, k), rng.uniform(0.1, 1.0, k)
        op = L.LaplexOperator(a, b, 1.0)
        op.weighted_gram(D)
        ts[lg] = _best(lambda: op.weighted_gram(D), 7)
    assert ts[13] / ts[10] <= 2.0, ts
    assert ts[16] / ts[13] <= 8.0, ts
