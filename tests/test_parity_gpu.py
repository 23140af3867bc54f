"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north_star): sort permutations and merge ranks bit-exact,
ties broken exactly as the reference; fp64 outputs within the reference's own
test tolerances (1e-12/1e-13); fp32 outputs within relative l2 <= 1e-5 of the
fp64 oracle on the same fp32 inputs.
"""
import math

import numpy as np
import pytest

import oracle as O
import paper_2605_24584_b200 as L
from _golden import load

pytestmark = pytest.mark.gpu
F64, F32 = np.float64, np.float32
TOL32 = 1e-5  # north_star: fp32 accumulation vs fp64 oracle, relative l2


def instance(rng, n, k, span=5.0, ties=True):
    a = rng.uniform(-span, span, n)
    b = rng.uniform(-span, span, k)
    if ties:
        m = min(n, k) // 2 + 1
        b[rng.integers(0, k, m)] = a[rng.integers(0, n, m)]
    return a, b


# ---------------------------------------------------------------- sort
@pytest.mark.parametrize("dt", [F64, F32])
@pytest.mark.parametrize("m", [1, 2, 3, 31, 4095, 4096, 4097, 6143, 6144, 6145, 12289, 100_003])
def test_sort_bit_exact(dt, m):
    rng = np.random.default_rng(m)
    raw = rng.uniform(-3, 3, m).astype(dt)
    if m > 8:
        raw[rng.integers(0, m, m // 3)] = raw[rng.integers(0, m, m // 3)]  # duplicates
        raw[:6] = [0.0, -0.0, 0.0, -0.0, 1.0, -1.0]
    s = L.sort_anchors(raw, dtype=dt)
    v, p, d = O.sort_anchors(raw, dtype=dt)
    assert np.array_equal(s.perm, p)
    assert np.array_equal(s.values.view(np.uint8), v.view(np.uint8))  # sign of zero kept
    assert O.rel_err_l2(s.decays, d) <= (1e-15 if dt == F64 else 1e-6)


@pytest.mark.parametrize("case", sorted(load("sort.npz")))
def test_sort_matches_reference_golden(case):
    c = load("sort.npz")[case]
    dt = c["raw"].dtype
    s = L.sort_anchors(c["raw"], dtype=dt)
    assert np.array_equal(s.perm, c["perm"])
    assert np.array_equal(s.values.view(np.uint8), c["values"].view(np.uint8))
    if dt == F64:
        # tests/test_scan.cpp:20: decays to 1e-15 relative
        assert np.allclose(s.decays, c["decays"], rtol=1e-15, atol=0)


def test_sort_signed_zero_and_spec_examples():
    s = L.sort_anchors([0.0, -0.0, 1.0, -0.0, 0.0])
    assert s.perm.tolist() == [0, 1, 3, 4, 2]
    assert np.signbit(s.values).tolist() == [False, True, True, False, False]
    s = L.sort_anchors([3.0, -1.0, 2.0, -1.0])
    assert s.values.tolist() == [-1.0, -1.0, 2.0, 3.0] and s.perm[:2].tolist() == [1, 3]
    assert s.decays[0] == 1.0 and s.decays[1] == pytest.approx(math.exp(-3.0), rel=1e-15)
    assert L.sort_anchors([0.0, 0.0, -1.0]).perm.tolist() == [2, 0, 1]


@pytest.mark.parametrize("dt", [F64, F32])
def test_sort_division_collisions_keep_input_order(dt):
    # raw/t rounds distinct raws onto the same key: ties must keep input order
    rng = np.random.default_rng(5)
    raw = (1.0 + rng.integers(0, 4, 20000) * np.finfo(dt).eps).astype(dt)
    t = 3.0
    op = L.LaplexOperator(raw, raw[:100], t, dtype=dt)
    oo = O.OracleOp(raw, raw[:100], t, dtype=dt)
    assert np.array_equal(op.sorted_rows().perm, oo.sorted(0)[1])
    assert np.array_equal(op.sorted_rows().values, oo.sorted(0)[0])


# ------------------------------------------------------------- co-ranks
@pytest.mark.parametrize("dt", [F64, F32])
def test_coranks_bit_exact(dt):
    rng = np.random.default_rng(9)
    for n, k in [(1, 1), (3, 5000), (5000, 3), (4096, 4096), (20000, 30000)]:
        a, b = instance(rng, n, k, 2.0)
        a = np.round(a, 2)  # dense ties inside both sides
        b = np.round(b, 2)
        op = L.LaplexOperator(a.astype(dt), b.astype(dt), 1.0, dtype=dt)
        oo = O.OracleOp(a.astype(dt), b.astype(dt), 1.0, dtype=dt)
        A, Bv = oo.sorted(0)[0], oo.sorted(1)[0]
        assert np.array_equal(op.row_buckets(), oo.ranks(0))        # j_of_row, operator.hpp:116-120
        assert np.array_equal(op.col_buckets(), oo.ranks(1))        # r_of_col, operator.hpp:111-115
        assert np.array_equal(op.ranks(0, True), np.searchsorted(Bv, A, "left"))
        assert np.array_equal(op.ranks(1, True), np.searchsorted(A, Bv, "left"))


def test_coranks_probe_signed_zero():
    op = L.LaplexOperator([-0.0, 1.0], [0.0, -0.0, 2.0])
    assert op.col_buckets().tolist() == [1, 1, 2]
    assert op.row_buckets().tolist() == [2, 2]


def test_transposed_view_ranks_and_sorted():
    rng = np.random.default_rng(10)
    a, b = instance(rng, 300, 200)
    op = L.LaplexOperator(a, b, 0.7)
    tr = op.transposed()
    oo = O.OracleOp(b, a, 0.7)
    assert np.array_equal(tr.row_buckets(), oo.ranks(0))
    assert np.array_equal(tr.col_buckets(), oo.ranks(1))
    assert np.array_equal(tr.sorted_rows().perm, oo.sorted(0)[1])


# -------------------------------------------------------- golden outputs
@pytest.mark.parametrize("case", sorted(load("operator.npz")))
def test_operator_matches_reference_golden(case):
    c = load("operator.npz")[case]
    dt = c["a"].dtype
    tol = 1e-12 if dt == F64 else 2e-5  # fp32 golden is the reference's own fp32
    op = L.LaplexOperator(c["a"], c["b"], float(c["t"]), c.get("phi"), c.get("psi"), dtype=dt)
    assert np.array_equal(op.sorted_rows().perm, c["rows_perm"])
    assert np.array_equal(op.sorted_cols().perm, c["cols_perm"])
    assert np.array_equal(op.sorted_rows().values, c["rows_values"])
    assert np.array_equal(op.row_buckets(), c["j_of_row"])
    assert np.array_equal(op.col_buckets(), c["r_of_col"])
    if "phi" in c:
        assert O.rel_err_l2(op.phased_matvec(c["x"]), c["phased_matvec"]) <= tol
        v = L.phased_matvec_vjp(op, c["x"], c["g"])
        for got, key in zip((v.x_bar, v.a_bar, v.b_bar, v.phi_bar, v.psi_bar),
                            ("x_bar", "a_bar", "b_bar", "phi_bar", "psi_bar")):
            assert O.rel_err_l2(got, c["pvjp_" + key]) <= 10 * tol, key
        assert O.rel_err_l2(op.phased_gram(c["D"]).matrix, c["phased_gram"]) <= 10 * tol
    else:
        assert O.rel_err_l2(op.matvec(c["x"]), c["matvec_B"]) <= tol
        assert O.rel_err_l2(op.matvec_transpose(c["g"]), c["matvec_transpose"]) <= tol
        assert O.rel_err_l2(op.batch_matvec(c["X"]), c["batch_matvec"]) <= tol
        v = L.matvec_vjp(op, c["x"], c["g"])
        for got, key in zip((v.x_bar, v.a_bar, v.b_bar), ("x_bar", "a_bar", "b_bar")):
            assert O.rel_err_l2(got, c["vjp_" + key]) <= 10 * tol, key
        M = op.weighted_gram(c["D"]).matrix
        assert O.rel_err_l2(M, c["weighted_gram"]) <= 10 * tol
        assert O.rel_err_l2(L.gram_vjp_weights(op, c["D"], c["G_bar"]), c["gram_vjp_weights"]) <= 10 * tol


@pytest.mark.parametrize("case", sorted(load("scan.npz")))
def test_scans_match_reference_golden(case):
    c = load("scan.npz")[case]
    dt = c["values"].dtype
    s = L.SortedAnchors(c["values"], np.arange(len(c["values"]), dtype=np.uint64), np.zeros(0, dt))
    tol = 1e-12 if dt == F64 else 1e-5
    assert O.rel_err_l2(L.prefix_decay_scan(s, c["payload"]), c["prefix"]) <= tol
    assert O.rel_err_l2(L.suffix_decay_scan(s, c["payload"]), c["suffix"]) <= tol


# ------------------------------------------ fp64 vs dense (reference tests)
def test_matvec_matches_dense_many_instances():
    # tests/test_operator.cpp:36-49 and acceptance check 1 (<= 1e-12, ties planted)
    rng = np.random.default_rng(21)
    worst = 0.0
    for trial in range(120):
        n, k = rng.integers(1, 257, 2)
        a, b = instance(rng, n, k, 6.0, ties=trial % 3 == 0)
        x = rng.uniform(-1, 1, k)
        t = 1.0 if trial % 2 else 0.42
        got = L.LaplexOperator(a, b, t).matvec(x)
        worst = max(worst, O.rel_err_l2(got, O.dense_matvec(a, b, t, x)))
    assert worst <= 1e-13


def test_transpose_and_vjp_fp64():
    rng = np.random.default_rng(24)
    for trial in range(30):
        n, k = rng.integers(1, 300, 2)
        a, b = instance(rng, n, k, ties=trial % 2 == 0)
        g = rng.uniform(-1, 1, n)
        x = rng.uniform(-1, 1, k)
        op = L.LaplexOperator(a, b, 0.9)
        tr = op.matvec_transpose(g)
        assert O.rel_err_l2(tr, O.dense_matvec(b, a, 0.9, g)) <= 1e-13
        v = L.matvec_vjp(op, x, g)
        assert np.array_equal(v.x_bar, tr)  # SPEC.md:242 bitwise
        want = O.OracleOp(a, b, 0.9).vjp(x, g)
        for got, w in zip((v.x_bar, v.a_bar, v.b_bar), want):
            assert O.rel_err_l2(got, w) <= 1e-12


def test_vjp_matches_finite_differences():
    # tests/test_gradients.cpp:41-68, acceptance check 4
    rng = np.random.default_rng(42)

    def separate(a, b, gap=1e-3):
        for i in range(len(a)):
            for j in range(len(b)):
                if abs(a[i] - b[j]) < gap:
                    a[i] += 2 * gap
    for trial in range(20):
        n, k = rng.integers(2, 25, 2)
        a, b = rng.uniform(-3, 3, n), rng.uniform(-3, 3, k)
        separate(a, b)
        x, g = rng.uniform(-1, 1, k), rng.uniform(-1, 1, n)
        t = 1.0 if trial % 2 else 0.5
        v = L.matvec_vjp(L.LaplexOperator(a, b, t), x, g)
        h = 1e-6
        fa = np.array([(g @ O.dense_matvec(a + h * np.eye(n)[i], b, t, x) -
                        g @ O.dense_matvec(a - h * np.eye(n)[i], b, t, x)) / (2 * h) for i in range(n)])
        fb = np.array([(g @ O.dense_matvec(a, b + h * np.eye(k)[j], t, x) -
                        g @ O.dense_matvec(a, b - h * np.eye(k)[j], t, x)) / (2 * h) for j in range(k)])
        assert O.rel_err_l2(v.a_bar, fa) <= 1e-5
        assert O.rel_err_l2(v.b_bar, fb) <= 1e-5
        s = v.a_bar.sum() + v.b_bar.sum()
        assert abs(s) <= 1e-10 * np.linalg.norm(g) * np.linalg.norm(x)


def test_exact_ties_zero_subgradient():
    # tests/test_gradients.cpp:85-106
    v = L.matvec_vjp(L.LaplexOperator([2.0], [2.0]), [1.5], [3.0])
    assert v.a_bar[0] == 0.0 and v.b_bar[0] == 0.0 and v.x_bar[0] == pytest.approx(3.0)
    v = L.matvec_vjp(L.LaplexOperator([0.0, 5.0], [5.0]), [1.0], [1.0, 1.0])
    assert v.a_bar[0] == pytest.approx(math.exp(-5)) and v.a_bar[1] == 0.0
    assert v.b_bar[0] == pytest.approx(-math.exp(-5))
    v = L.matvec_vjp(L.LaplexOperator([0.0], [5.0]), [1.0], [1.0])
    assert v.a_bar[0] == pytest.approx(math.exp(-5), rel=1e-14)
    assert v.b_bar[0] == pytest.approx(-math.exp(-5), rel=1e-14)


def test_degenerate_shapes():
    assert L.LaplexOperator([0.0], [0.0]).matvec([3.0]).tolist() == [3.0]
    y = L.LaplexOperator([0.0, math.log(2.0)], [0.0]).matvec([1.0])
    assert y.tolist() == pytest.approx([1.0, 0.5])
    z = L.LaplexOperator([1.0, 1.0, 1.0], [1.0, 1.0]).matvec([2.0, 3.0])
    assert z.tolist() == pytest.approx([5.0] * 3)
    # all anchors equal across several merge tiles
    n = 10_000
    y = L.LaplexOperator(np.ones(n), np.ones(n)).matvec(np.ones(n))
    assert np.allclose(y, n, rtol=1e-12)


def test_bitwise_contracts():
    rng = np.random.default_rng(25)
    a, b = instance(rng, 2000, 3500)
    op = L.LaplexOperator(a, b, 1.0)
    X = rng.uniform(-1, 1, (5, 3500))
    Y = op.batch_matvec(X)
    for r in range(5):  # tests/test_operator.cpp:120-132
        assert np.array_equal(Y[r], op.matvec(X[r]))
    t = 0.73  # tests/test_operator.cpp:98-108
    x = rng.uniform(-1, 1, 3500)
    y1 = L.LaplexOperator(a, b, t).matvec(x)
    y2 = L.LaplexOperator(a / t, b / t, 1.0).matvec(x)
    assert np.array_equal(y1, y2)


def test_linearity_and_permutation_equivariance():
    rng = np.random.default_rng(22)
    a, b = instance(rng, 400, 600)
    op = L.LaplexOperator(a, b, 1.0)
    x1, x2 = rng.uniform(-1, 1, 600), rng.uniform(-1, 1, 600)
    y1, y2 = op.matvec(x1), op.matvec(x2)
    yc = op.matvec(1.5 * x1 - 0.5 * x2)
    assert np.allclose(yc, 1.5 * y1 - 0.5 * y2, rtol=1e-12, atol=1e-12)
    yp = L.LaplexOperator(a[::-1].copy(), b, 1.0).matvec(x1)
    assert np.allclose(yp, y1[::-1], rtol=1e-13)


def test_phased_fp64():
    rng = np.random.default_rng(29)
    for trial in range(10):
        n, k = rng.integers(1, 300, 2)
        a, b = instance(rng, n, k)
        phi, psi = rng.uniform(0, 6.28, n), rng.uniform(0, 6.28, k)
        x, g = rng.uniform(-1, 1, k), rng.uniform(-1, 1, n)
        op = L.LaplexOperator(a, b, 1.1, phi, psi)
        assert O.rel_err_l2(op.phased_matvec(x), O.dense_matvec(a, b, 1.1, x, phi, psi)) <= 1e-12
        v = L.phased_matvec_vjp(op, x, g)
        want = O.OracleOp(a, b, 1.1, phi, psi).phased_vjp(x, g)
        for got, w in zip((v.x_bar, v.a_bar, v.b_bar, v.phi_bar, v.psi_bar), want):
            assert O.rel_err_l2(got, w) <= 1e-11
    # SPEC.md phased examples: zero phases == plain; phi - psi = pi/2 -> 0
    a, b = instance(rng, 50, 70)
    x = rng.uniform(-1, 1, 70)
    z = L.LaplexOperator(a, b, 1.0, np.zeros(50), np.zeros(70)).phased_matvec(x)
    assert O.rel_err_l2(z, L.LaplexOperator(a, b, 1.0).matvec(x)) <= 1e-14
    q = L.LaplexOperator(a, b, 1.0, np.full(50, np.pi / 2), np.zeros(70)).phased_matvec(x)
    assert np.max(np.abs(q)) <= 1e-12 * np.max(np.abs(z))


def test_gram_fp64_and_symmetry():
    # tests/test_operator.cpp:134-173, acceptance check 2
    rng = np.random.default_rng(26)
    for trial in range(25):
        n, k = rng.integers(1, 49), rng.integers(1, 4097)
        a, b = rng.uniform(-5, 5, n), rng.uniform(-5, 5, k)
        D = rng.uniform(-2, 2, k)
        t = 1.0 if trial % 2 else 1.6
        M = L.LaplexOperator(a, b, t).weighted_gram(D).matrix
        assert O.rel_err_l2(M, O.dense_gram(a, b, t, D)) <= 1e-10
        assert np.array_equal(M, M.T)
        diag = np.array([np.sum(D * np.exp(-2 * np.abs(a[i] - b) / t)) for i in range(n)])
        assert np.max(np.abs(np.diag(M) - diag) / np.maximum(1, np.abs(diag))) <= 1e-12
    phi, psi = rng.uniform(0, 6.28, 28), rng.uniform(0, 6.28, 70)
    a, b, D = rng.uniform(-5, 5, 28), rng.uniform(-5, 5, 70), rng.uniform(-1.5, 1.5, 70)
    M = L.LaplexOperator(a, b, 0.6, phi, psi).phased_gram(D).matrix
    assert O.rel_err_l2(M, O.dense_gram(a, b, 0.6, D, phi, psi)) <= 1e-10
    assert np.array_equal(M, M.T)


def test_gram_vjp_weights():
    rng = np.random.default_rng(45)
    n, k = 18, 30
    a, b = rng.uniform(-3, 3, n), rng.uniform(-3, 3, k)
    op = L.LaplexOperator(a, b, 1.2)
    G = rng.uniform(-1, 1, (n, n))
    G = np.tril(G) + np.tril(G, -1).T
    D = rng.uniform(-1, 1, k)
    got = L.gram_vjp_weights(op, D, G)
    K = np.exp(-np.abs(a[:, None] - b[None, :]) / 1.2)
    want = np.einsum("it,ij,jt->t", K, G, K)
    assert np.allclose(got, want, rtol=1e-11, atol=1e-13)
    G[0, 1] += 0.5
    with pytest.raises(L.AsymmetricCotangent):
        L.gram_vjp_weights(op, D, G)


def test_error_taxonomy_on_device_plans():
    op = L.LaplexOperator([0.0, 1.0], [0.5])
    with pytest.raises(L.DimensionMismatch):
        op.matvec([1.0, 2.0])
    with pytest.raises(L.DimensionMismatch):
        op.weighted_gram([1.0, 2.0])
    with pytest.raises(L.PhaseAbsent):
        op.phased_matvec([1.0])
    with pytest.raises(L.PhaseAbsent):
        op.phased_gram([1.0])
    with pytest.raises(L.NonFinite):
        op.matvec([float("nan")])
    with pytest.raises(L.DimensionMismatch):
        L.matvec_vjp(op, [1.0, 2.0], [1.0, 1.0])
    with pytest.raises(L.DimensionMismatch):
        L.matvec_vjp(op, [1.0], [1.0])
    ph = L.LaplexOperator([0.0], [0.5], 1.0, [0.2], [0.3])
    with pytest.raises(L.PhasePresent):
        ph.matvec([1.0])
    with pytest.raises(L.PhasePresent):
        ph.weighted_gram([1.0])
    with pytest.raises(L.PhasePresent):
        L.gram_vjp_weights(ph, [1.0], np.ones((1, 1)))


# ------------------------------------------------ fp32 at scale vs fp64
# 2^23 sides take the permutation-plan path (staged outputs, per-tile store order)
@pytest.mark.parametrize("lg,span", [(16, 100.0), (20, 100.0), (20, 3.0), (22, 100.0), (23, 100.0)])
def test_fp32_against_fp64_oracle(lg, span):
    rng = np.random.default_rng(lg)
    N = 1 << lg
    a = rng.uniform(-span, span, N).astype(F32)
    b = rng.uniform(-span, span, N).astype(F32)
    x = rng.uniform(-1, 1, N).astype(F32)
    g = rng.uniform(-1, 1, N).astype(F32)
    op = L.LaplexOperator(a, b, 1.0, dtype=F32)
    y = op.matvec(x)
    v = L.matvec_vjp(op, x, g)
    of = O.OracleOp(a, b, 1.0, dtype=F32)   # bit-exact permutations vs the fp32 reference path
    assert np.array_equal(op.sorted_rows().perm, of.sorted(0)[1])
    assert np.array_equal(op.sorted_cols().perm, of.sorted(1)[1])
    assert np.array_equal(op.col_buckets(), of.ranks(1))
    o64 = O.OracleOp(a.astype(F64), b.astype(F64), 1.0)
    assert O.rel_err_l2(y, o64.matvec(x.astype(F64), 2)) <= TOL32
    for got, w in zip((v.x_bar, v.a_bar, v.b_bar), o64.vjp(x.astype(F64), g.astype(F64))):
        assert O.rel_err_l2(got, w) <= TOL32


def test_fp32_accuracy_ordering_acceptance5():
    # acceptance check 5: f32 scan error <= f32 dense error, n=2^14, batch 8
    rng = np.random.default_rng(500)
    n = 1 << 14
    a, b = rng.uniform(-8, 8, n), rng.uniform(-8, 8, n)
    X = rng.uniform(-1, 1, (8, n))
    Yref = np.stack([O.dense_matvec(a, b, 1.0, X[r]) for r in range(8)])
    Ys = L.LaplexOperator(a.astype(F32), b.astype(F32), 1.0, dtype=F32).batch_matvec(X.astype(F32))
    Kf = np.exp(-np.abs(a.astype(F32)[:, None] - b.astype(F32)[None, :]), dtype=F32)
    Yd = (X.astype(F32) @ Kf.T).astype(F32)
    es = np.median([O.rel_err_l2(Ys[r], Yref[r]) for r in range(8)])
    ed = np.median([O.rel_err_l2(Yd[r], Yref[r]) for r in range(8)])
    assert es <= ed


# --------------------------------------------------- device-pointer API
def test_device_api_matches_host_api():
    import torch
    rng = np.random.default_rng(77)
    a, b = instance(rng, 50_000, 70_000, 50.0)
    x = rng.uniform(-1, 1, (3, 70_000))
    g = rng.uniform(-1, 1, (3, 50_000))
    dev = torch.device("cuda:0")
    T = lambda v: torch.tensor(v, dtype=torch.float64, device=dev)  # noqa: E731
    dop = L.DeviceOperator(T(a), T(b), 0.9)
    y = dop.apply(T(x))
    xb, ab, bb, _, _ = dop.backward(T(x), T(g))
    yt = dop.apply(T(g), transpose=True)
    torch.cuda.synchronize()
    op = L.LaplexOperator(a, b, 0.9)
    assert np.array_equal(y.cpu().numpy(), op.batch_matvec(x))
    v = L.matvec_vjp(op, x, g)
    assert np.array_equal(xb.cpu().numpy(), v.x_bar)
    assert np.array_equal(yt.cpu().numpy(), xb.cpu().numpy())
    assert np.array_equal(ab.cpu().numpy(), v.a_bar) and np.array_equal(bb.cpu().numpy(), v.b_bar)
    # batch a_bar/b_bar are sums of the per-row VJPs
    per = [L.matvec_vjp(op, x[r], g[r]) for r in range(3)]
    assert np.allclose(v.a_bar, sum(p.a_bar for p in per), rtol=1e-12, atol=1e-14)


def test_device_plan_reports_nonfinite_anchor():
    import torch
    a = torch.tensor([0.0, float("nan"), 1.0], device="cuda:0")
    b = torch.tensor([0.5], device="cuda:0")
    with pytest.raises(L.NonFinite):
        L.DeviceOperator(a, b)


# ------------------------------------------------ batch rows on the plan path
def test_batch_rows_on_plan_path():
    """Rows > 1 with sides above the direct-permutation limit (2^22): per-row
    payload staging, store order and the row-summed anchor cotangents."""
    import torch
    rng = np.random.default_rng(41)
    N, B = (1 << 23) + 1234, 3
    dev = torch.device("cuda:0")
    a = torch.tensor(rng.uniform(-100, 100, N).astype(F32), device=dev)
    b = torch.tensor(rng.uniform(-100, 100, N - 777).astype(F32), device=dev)
    X = torch.tensor(rng.uniform(-1, 1, (B, N - 777)).astype(F32), device=dev)
    G = torch.tensor(rng.uniform(-1, 1, (B, N)).astype(F32), device=dev)
    op = L.DeviceOperator(a, b, 1.0)
    Y = op.apply(X)
    xb, ab, bb, _, _ = op.backward(X, G)
    for r in range(B):  # batch row r == single-row call, bitwise (tests/test_operator.cpp:120-132)
        assert torch.equal(Y[r], op.apply(X[r:r + 1])[0])
        xr, ar, br, _, _ = op.backward(X[r:r + 1], G[r:r + 1])
        assert torch.equal(xb[r], xr[0])
    # anchor cotangents are sums over rows
    parts = [op.backward(X[r:r + 1], G[r:r + 1]) for r in range(B)]
    sa = sum(p[1].double() for p in parts)
    sb = sum(p[2].double() for p in parts)
    assert O.rel_err_l2(ab.double().cpu().numpy(), sa.cpu().numpy()) <= 1e-6
    assert O.rel_err_l2(bb.double().cpu().numpy(), sb.cpu().numpy()) <= 1e-6
    # x_bar of the VJP is the transpose, bitwise
    assert torch.equal(xb, op.apply(G, transpose=True))


# ------------------------------------------------ plan path: phases, transpose, fp64
def test_plan_path_phased_and_transpose_fp64():
    """Sides above the direct-permutation limit (2^22) in fp64: phased forward and
    VJP and the transpose against the reference oracle (staged outputs, per-tile
    store order, window scatters)."""
    rng = np.random.default_rng(43)
    n, k = (1 << 22) + 7, (1 << 22) + 1000
    a = rng.uniform(-100, 100, n)
    b = rng.uniform(-100, 100, k)
    b[:5000] = a[:5000]  # exact ties across the sides
    phi, psi = rng.uniform(0, 6.28, n), rng.uniform(0, 6.28, k)
    x, g = rng.uniform(-1, 1, k), rng.uniform(-1, 1, n)
    op = L.LaplexOperator(a, b, 0.9, phi, psi)
    oo = O.OracleOp(a, b, 0.9, phi, psi)
    assert O.rel_err_l2(op.phased_matvec(x), oo.phased_matvec(x)) <= 1e-12
    v = L.phased_matvec_vjp(op, x, g)
    for got, w in zip((v.x_bar, v.a_bar, v.b_bar, v.phi_bar, v.psi_bar), oo.phased_vjp(x, g)):
        assert O.rel_err_l2(got, w) <= 1e-11
    plain = L.LaplexOperator(a, b, 0.9)
    assert O.rel_err_l2(plain.matvec_transpose(g), O.OracleOp(a, b, 0.9).matvec_transpose(g)) <= 1e-12


# ------------------------------------------------ host API: device-side validation above 2^20
def test_host_api_large_inputs_nonfinite_order():
    """Above 2^20 elements the host-pointer API checks finiteness on the device
    after the upload; errors keep the reference order (operator.hpp:88-101,
    gradients.hpp:113-117) and no output is written."""
    import ctypes as C
    from paper_2605_24584_b200 import _lib
    lib = _lib.lib()
    rng = np.random.default_rng(44)
    n = k = (1 << 20) + 5
    a = rng.uniform(-10, 10, n)
    b = rng.uniform(-10, 10, k)
    bad_b = b.copy()
    bad_b[k // 2] = np.nan
    with pytest.raises(L.NonFinite, match="col anchors"):
        L.LaplexOperator(a, bad_b)
    with pytest.raises(L.NonFinite, match="row anchors"):
        L.LaplexOperator(np.where(np.arange(n) == 3, np.inf, a), bad_b, -1.0)  # anchors before temperature
    with pytest.raises(L.NonFinite, match="temperature"):
        L.LaplexOperator(a, b, 0.0)
    op = L.LaplexOperator(a, b)
    x = rng.uniform(-1, 1, k)
    g = rng.uniform(-1, 1, n)
    xb = x.copy()
    xb[7] = np.nan
    gb = g.copy()
    gb[n - 1] = np.inf
    y = np.full(n, 12345.0)
    rc = lib.laplex_apply(op._h, 0, xb.ctypes.data, 1, k, y.ctypes.data)
    assert rc == 2 and b"matvec x" in lib.laplex_last_error()
    assert np.all(y == 12345.0)  # untouched
    with pytest.raises(L.NonFinite, match="vjp g"):
        L.matvec_vjp(op, x, gb)
    with pytest.raises(L.NonFinite, match="vjp x"):
        L.matvec_vjp(op, xb, gb)  # x reported first
    # and the valid call still works afterwards
    assert O.rel_err_l2(op.matvec(x), O.OracleOp(a, b).matvec(x)) <= 1e-12


# ------------------------------------------------ batches over few tiles: row-split work items
@pytest.mark.parametrize("phased", [False, True])
def test_row_split_batches_fp64(phased):
    """A batch whose merge tiles are fewer than the resident CTA slots runs as
    (tile, row chunk) work items with per-chunk partial cotangents summed in
    chunk order (lx_main rsplit, lx_chunk_sum).  fp64 against the reference
    oracle row by row; a_bar/b_bar (and phi_bar/psi_bar) against the oracle's
    per-row cotangents summed over rows (reference gradients.hpp:122-133)."""
    import torch
    rng = np.random.default_rng(47 + phased)
    n, k, B = 3001, 150_000, 24
    a = rng.uniform(-50, 50, n)
    b = rng.uniform(-50, 50, k)
    b[:500] = a[:500]  # exact ties across the sides
    phi, psi = (rng.uniform(0, 6.28, n), rng.uniform(0, 6.28, k)) if phased else (None, None)
    X, G = rng.uniform(-1, 1, (B, k)), rng.uniform(-1, 1, (B, n))
    dev = torch.device("cuda:0")
    T = lambda v: None if v is None else torch.tensor(v, device=dev)
    op = L.DeviceOperator(T(a), T(b), 0.8, T(phi), T(psi))
    oo = O.OracleOp(a, b, 0.8, phi, psi)
    Y = op.apply(T(X)).cpu().numpy()
    cots = [c.cpu().numpy() if c is not None else None for c in op.backward(T(X), T(G))]
    sums = None
    for r in range(B):
        if phased:
            assert O.rel_err_l2(Y[r], oo.phased_matvec(X[r])) <= 1e-12
            w = oo.phased_vjp(X[r], G[r])
        else:
            assert O.rel_err_l2(Y[r], oo.matvec(X[r])) <= 1e-12
            w = oo.vjp(X[r], G[r])
        assert O.rel_err_l2(cots[0][r], w[0]) <= 1e-11
        sums = list(w[1:]) if sums is None else [s + v for s, v in zip(sums, w[1:])]
    for got, want in zip(cots[1:], sums):
        assert O.rel_err_l2(got, want) <= 1e-11


def test_row_split_batches_fp32_bitwise_rows():
    """fp32 unphased batch over few tiles (the 3-CTA batch kernels, carries of the
    next row prefetched): every row bitwise equal to its single-row call, x_bar
    bitwise the transpose, row-summed cotangents equal to the sum of single-row
    ones."""
    import torch
    rng = np.random.default_rng(53)
    n, k, B = 100_000, 90_000, 32
    dev = torch.device("cuda:0")
    a = torch.tensor(rng.uniform(-100, 100, n).astype(F32), device=dev)
    b = torch.tensor(rng.uniform(-100, 100, k).astype(F32), device=dev)
    X = torch.tensor(rng.uniform(-1, 1, (B, k)).astype(F32), device=dev)
    G = torch.tensor(rng.uniform(-1, 1, (B, n)).astype(F32), device=dev)
    op = L.DeviceOperator(a, b, 1.0)
    Y = op.apply(X)
    xb, ab, bb, _, _ = op.backward(X, G)
    parts = [op.backward(X[r:r + 1], G[r:r + 1]) for r in range(B)]
    for r in range(B):
        assert torch.equal(Y[r], op.apply(X[r:r + 1])[0])
        assert torch.equal(xb[r], parts[r][0][0])
    assert torch.equal(xb, op.apply(G, transpose=True))
    sa = sum(p[1].double() for p in parts)
    sb = sum(p[2].double() for p in parts)
    assert O.rel_err_l2(ab.double().cpu().numpy(), sa.cpu().numpy()) <= 1e-6
    assert O.rel_err_l2(bb.double().cpu().numpy(), sb.cpu().numpy()) <= 1e-6
