"""CPU: pin the oracle (C restatement of the reference hot path) before it is
trusted as the checker.

(a) known-answer vectors from the reference's own tests and SPEC;
(b) bit-exact agreement with golden fixtures produced by the UNMODIFIED
    reference (tests/golden/make_golden.py -> oracle/_ref);
(c) when oracle/_ref is built (dev container), fresh random cases against it.
"""
import math

import numpy as np
import pytest

import oracle as O
from _golden import load

F64, F32 = np.float64, np.float32


# ---------------------------------------------------------------- (a) KATs
def test_sort_golden_case_reference_test_scan():
    # tests/test_scan.cpp:10-21
    v, p, d = O.sort_anchors([3.0, -1.0, 2.0, -1.0])
    assert v.tolist() == [-1.0, -1.0, 2.0, 3.0]
    assert p[0] == 1 and p[1] == 3
    assert d[0] == 1.0
    assert d[1] == pytest.approx(math.exp(-3.0), rel=1e-15)


def test_sort_spec_examples():
    # SPEC.md:38-40
    v, p, d = O.sort_anchors([3.0])
    assert v.tolist() == [3.0] and p.tolist() == [0] and len(d) == 0
    v, p, d = O.sort_anchors([1.0, 0.0])
    assert v.tolist() == [0.0, 1.0] and p.tolist() == [1, 0] and d[0] == pytest.approx(math.exp(-1))
    v, p, _ = O.sort_anchors([0.0, 0.0, -1.0])
    assert p.tolist() == [2, 0, 1]


def test_sort_signed_zero_probe():
    # {+0,-0,1,-0,+0} -> perm 0 1 3 4 2, sign bits preserved in values
    v, p, _ = O.sort_anchors([0.0, -0.0, 1.0, -0.0, 0.0])
    assert p.tolist() == [0, 1, 3, 4, 2]
    assert np.signbit(v).tolist() == [False, True, True, False, False]


def test_sort_validation():
    # tests/test_scan.cpp:23-28
    with pytest.raises(O.OracleError) as e:
        O.sort_anchors([])
    assert e.value.kind == "EmptyInput"
    with pytest.raises(O.OracleError) as e:
        O.sort_anchors([1.0, float("nan")])
    assert e.value.kind == "NonFinite"
    with pytest.raises(O.OracleError) as e:
        O.sort_anchors([float("inf")])
    assert e.value.kind == "NonFinite"


def test_coranks_probe():
    # a={-0,1}, b={0,-0,2} -> r_of_col=[1,1,2], j_of_row=[2,2]
    op = O.OracleOp([-0.0, 1.0], [0.0, -0.0, 2.0])
    assert op.ranks(1).tolist() == [1, 1, 2]
    assert op.ranks(0).tolist() == [2, 2]


def test_scan_spec_examples():
    # SPEC.md:48-49,56-57
    pre, suf = O.decay_scan([0.0, math.log(2.0)], [1.0, 0.0])
    assert pre.tolist() == pytest.approx([1.0, 0.5])
    pre, suf = O.decay_scan([0.0, math.log(2.0)], [0.0, 1.0])
    assert suf.tolist() == pytest.approx([0.5, 1.0])
    pre, suf = O.decay_scan([0.0], [7.0])
    assert pre.tolist() == [7.0] and suf.tolist() == [7.0]


def test_matvec_kats():
    # tests/test_operator.cpp:63-76 and SPEC.md:122-123
    assert O.OracleOp([0.0], [0.0]).matvec([3.0]).tolist() == [3.0]
    y = O.OracleOp([0.0, math.log(2.0)], [0.0]).matvec([1.0])
    assert y.tolist() == pytest.approx([1.0, 0.5])
    z = O.OracleOp([1.0, 1.0, 1.0], [1.0, 1.0]).matvec([2.0, 3.0])
    assert z.tolist() == pytest.approx([5.0, 5.0, 5.0])
    assert O.OracleOp([0.0], [0.0, 0.0]).matvec([1.0, 1.0]).tolist() == [2.0]
    y = O.OracleOp([0.0, math.log(2.0)], [math.log(2.0)]).matvec([1.0])
    assert y.tolist() == pytest.approx([0.5, 1.0])


def test_vjp_kats():
    # tests/test_gradients.cpp:85-106
    xb, ab, bb = O.OracleOp([2.0], [2.0]).vjp([1.5], [3.0])
    assert ab[0] == 0.0 and bb[0] == 0.0 and xb[0] == pytest.approx(3.0)
    xb, ab, bb = O.OracleOp([0.0, 5.0], [5.0]).vjp([1.0], [1.0, 1.0])
    assert ab[0] == pytest.approx(math.exp(-5.0)) and ab[1] == 0.0
    assert bb[0] == pytest.approx(-math.exp(-5.0))
    xb, ab, bb = O.OracleOp([0.0], [5.0]).vjp([1.0], [1.0])
    assert ab[0] == pytest.approx(math.exp(-5.0), rel=1e-14)
    assert bb[0] == pytest.approx(-math.exp(-5.0), rel=1e-14)


def test_gram_kat():
    # SPEC.md:151
    assert O.OracleOp([0.0], [0.0]).weighted_gram([3.0]).tolist() == [[3.0]]


def test_validation_codes():
    # tests/test_operator.cpp:205-222 (error taxonomy, validation order)
    def kind(f):
        with pytest.raises(O.OracleError) as e:
            f()
        return e.value.kind
    assert kind(lambda: O.OracleOp([], [1.0])) == "EmptyInput"
    assert kind(lambda: O.OracleOp([float("nan")], [1.0])) == "NonFinite"
    assert kind(lambda: O.OracleOp([0.0], [1.0], 0.0)) == "NonFinite"
    assert kind(lambda: O.OracleOp([0.0], [1.0], -2.0)) == "NonFinite"
    op = O.OracleOp([0.0, 1.0], [0.5])
    assert kind(lambda: op.matvec([1.0, 2.0])) == "DimensionMismatch"
    assert kind(lambda: op.weighted_gram([1.0, 2.0])) == "DimensionMismatch"
    assert kind(lambda: op.phased_matvec([1.0])) == "PhaseAbsent"
    ph = O.OracleOp([0.0], [0.5], 1.0, [0.2], [0.3])
    assert kind(lambda: ph.matvec([1.0])) == "PhasePresent"


def test_dense_oracle_agrees_with_operator():
    rng = np.random.default_rng(3)
    for _ in range(10):
        n, k = rng.integers(1, 50, 2)
        a, b = rng.uniform(-5, 5, n), rng.uniform(-5, 5, k)
        x = rng.uniform(-1, 1, k)
        for d in (1, 2):
            assert O.rel_err_l2(O.OracleOp(a, b, 0.6).matvec(x, d), O.dense_matvec(a, b, 0.6, x)) <= 1e-13


# ------------------------------------------------------- (b) golden fixtures
@pytest.mark.parametrize("case", sorted(load("sort.npz")))
def test_oracle_sort_matches_reference_golden(case):
    c = load("sort.npz")[case]
    dt = c["raw"].dtype
    v, p, d = O.sort_anchors(c["raw"], dtype=dt)
    assert np.array_equal(p, c["perm"])
    assert np.array_equal(v.view(np.uint8), c["values"].view(np.uint8))  # incl. sign of zero
    assert np.array_equal(d, c["decays"])


@pytest.mark.parametrize("case", sorted(load("operator.npz")))
def test_oracle_operator_matches_reference_golden(case):
    c = load("operator.npz")[case]
    dt = c["a"].dtype
    phased = "phi" in c
    op = O.OracleOp(c["a"], c["b"], float(c["t"]), c.get("phi"), c.get("psi"), dtype=dt)
    rv, rp, rd = op.sorted(0)
    cv, cp, cd = op.sorted(1)
    assert np.array_equal(rp, c["rows_perm"]) and np.array_equal(cp, c["cols_perm"])
    assert np.array_equal(rv, c["rows_values"]) and np.array_equal(cv, c["cols_values"])
    assert np.array_equal(op.ranks(0), c["j_of_row"]) and np.array_equal(op.ranks(1), c["r_of_col"])
    # same arithmetic, same order, same libm -> bit-identical
    if phased:
        assert np.array_equal(op.phased_matvec(c["x"]), c["phased_matvec"])
        got = op.phased_vjp(c["x"], c["g"])
        for g, key in zip(got, ("x_bar", "a_bar", "b_bar", "phi_bar", "psi_bar")):
            assert np.array_equal(g, c["pvjp_" + key])
        assert np.array_equal(op.phased_gram(c["D"]), c["phased_gram"])
    else:
        assert np.array_equal(op.matvec(c["x"], 1), c["matvec_A"])
        assert np.array_equal(op.matvec(c["x"], 2), c["matvec_B"])
        assert np.array_equal(op.matvec_transpose(c["g"]), c["matvec_transpose"])
        assert np.array_equal(op.batch_matvec(c["X"]), c["batch_matvec"])
        for g, key in zip(op.vjp(c["x"], c["g"]), ("x_bar", "a_bar", "b_bar")):
            assert np.array_equal(g, c["vjp_" + key])
        assert np.array_equal(op.weighted_gram(c["D"]), c["weighted_gram"])
        assert np.array_equal(op.gram_vjp_weights(c["D"], c["G_bar"]), c["gram_vjp_weights"])


@pytest.mark.parametrize("case", sorted(load("scan.npz")))
def test_oracle_scan_matches_reference_golden(case):
    c = load("scan.npz")[case]
    pre, suf = O.decay_scan(c["values"], c["payload"], dtype=c["values"].dtype)
    assert np.array_equal(pre, c["prefix"]) and np.array_equal(suf, c["suffix"])


# ------------------------------------------- (c) live reference (dev only)
needs_ref = pytest.mark.skipif(not O.available("ref"), reason="oracle/_ref not built")


@needs_ref
def test_mt19937_64_matches_libstdcxx():
    import ctypes as C
    out = np.empty(2000)
    O._lib("ref").lxr_mt_uniform(C.c_uint64(42), C.c_size_t(2000), C.c_double(-100.0), C.c_double(100.0),
                                 out.ctypes.data_as(C.c_void_p))
    assert np.array_equal(out, O.Mt19937_64Uniform(42).uniform(2000, -100, 100))


@needs_ref
@pytest.mark.parametrize("dt", [F64, F32])
def test_oracle_vs_reference_random(dt):
    rng = np.random.default_rng(11)
    for trial in range(20):
        n, k = rng.integers(1, 400, 2)
        a = rng.uniform(-6, 6, n).astype(dt)
        b = rng.uniform(-6, 6, k).astype(dt)
        m = min(n, k) // 2 + 1
        b[rng.integers(0, k, m)] = a[rng.integers(0, n, m)]
        x = rng.uniform(-1, 1, k).astype(dt)
        g = rng.uniform(-1, 1, n).astype(dt)
        t = 1.0 if trial % 2 else 0.42
        oc, orf = O.OracleOp(a, b, t, dtype=dt), O.OracleOp(a, b, t, dtype=dt, backend="ref")
        for side in (0, 1):
            for u, v in zip(oc.sorted(side), orf.sorted(side)):
                assert np.array_equal(u, v)
            assert np.array_equal(oc.ranks(side), orf.ranks(side))
        for d in (0, 1, 2):
            assert np.array_equal(oc.matvec(x, d), orf.matvec(x, d))
        for u, v in zip(oc.vjp(x, g), orf.vjp(x, g)):
            assert np.array_equal(u, v)


# ------------------------------- (d) the at-scale oracle (given sort order)
@pytest.mark.parametrize("case", sorted(load("operator.npz")))
def test_sorted_oracle_matches_reference_golden(case):
    """OracleOp.from_sorted over the reference's own permutations reproduces
    every reference output bit for bit (the sort is the only step skipped)."""
    c = load("operator.npz")[case]
    dt = c["a"].dtype
    op = O.OracleOp.from_sorted(c["a"], c["b"], float(c["t"]), c["rows_perm"], c["cols_perm"],
                                c.get("phi"), c.get("psi"), dtype=dt)
    assert np.array_equal(op.ranks(0), c["j_of_row"]) and np.array_equal(op.ranks(1), c["r_of_col"])
    assert np.array_equal(op.sorted(0)[0].view(np.uint8), c["rows_values"].view(np.uint8))
    if "phi" in c:
        assert np.array_equal(op.phased_matvec(c["x"]), c["phased_matvec"])
        for g, key in zip(op.phased_vjp(c["x"], c["g"]), ("x_bar", "a_bar", "b_bar", "phi_bar", "psi_bar")):
            assert np.array_equal(g, c["pvjp_" + key])
    else:
        assert np.array_equal(op.matvec(c["x"], 1), c["matvec_A"])
        assert np.array_equal(op.matvec(c["x"], 2), c["matvec_B"])
        assert np.array_equal(op.matvec_transpose(c["g"]), c["matvec_transpose"])
        for g, key in zip(op.vjp(c["x"], c["g"]), ("x_bar", "a_bar", "b_bar")):
            assert np.array_equal(g, c["vjp_" + key])


@pytest.mark.parametrize("dt", [F64, F32])
def test_verify_sort_accepts_only_the_stable_sort(dt):
    rng = np.random.default_rng(5)
    raw = rng.integers(-20, 20, 5000).astype(dt)  # heavy ties
    raw[::7] = -0.0
    raw[::11] = 0.0
    for t in (1.0, 0.3):
        _, perm, _ = O.sort_anchors(raw / dt(t), dtype=dt)
        assert O.verify_sort(raw, t, perm, dtype=dt) == -1
        # a swapped tie pair keeps the values sorted but breaks stability
        v = (raw / dt(t))[perm.astype(np.int64)]
        i = int(np.flatnonzero(v[:-1] == v[1:])[0])
        bad = perm.copy()
        bad[i], bad[i + 1] = bad[i + 1], bad[i]
        assert O.verify_sort(raw, t, bad, dtype=dt) == i
        # -0 and +0 compare equal: they must stay in index order too
        z = np.flatnonzero(v == 0)
        assert O.verify_sort(raw, t, perm, dtype=dt) == -1 and len(z) > 2
        # not a permutation
        dup = perm.copy()
        dup[3] = dup[4]
        assert O.verify_sort(raw, t, dup, dtype=dt) == len(raw)


def test_sorted_oracle_rejects_a_wrong_order():
    rng = np.random.default_rng(6)
    a, b = rng.uniform(-5, 5, 300), rng.uniform(-5, 5, 200)
    pa = np.argsort(a, kind="stable")
    pb = np.argsort(b, kind="stable")
    O.OracleOp.from_sorted(a, b, 1.0, pa, pb)
    with pytest.raises(O.OracleError) as e:
        O.OracleOp.from_sorted(a, b, 1.0, pa[::-1], pb)
    assert e.value.code == 97


def test_sorted_oracle_equals_sorting_oracle_random():
    rng = np.random.default_rng(8)
    for dt in (F64, F32):
        n, k = 3000, 2000
        a = rng.uniform(-30, 30, n).astype(dt)
        b = rng.uniform(-30, 30, k).astype(dt)
        b[:500] = a[:500]
        x, g = rng.uniform(-1, 1, k).astype(dt), rng.uniform(-1, 1, n).astype(dt)
        ref = O.OracleOp(a, b, 0.7, dtype=dt)
        op = O.OracleOp.from_sorted(a, b, 0.7, ref.sorted(0)[1], ref.sorted(1)[1], dtype=dt)
        for side in (0, 1):
            assert np.array_equal(op.ranks(side), ref.ranks(side))
        assert np.array_equal(op.matvec(x), ref.matvec(x))
        for u, v in zip(op.vjp(x, g), ref.vjp(x, g)):
            assert np.array_equal(u, v)
