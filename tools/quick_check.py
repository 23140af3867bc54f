"""Quick GPU-vs-oracle sweep used while developing (the real gates are in tests/)."""
import sys
import time
import os

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import oracle as O  # noqa: E402
import paper_2605_24584_b200 as L  # noqa: E402

rng = np.random.default_rng(0)
fails = 0


def rep(name, ok, detail=""):
    global fails
    print(f"{'PASS' if ok else 'FAIL'} {name} {detail}", flush=True)
    if not ok:
        fails += 1


def inst(n, k, span=5.0, ties=True):
    a = rng.uniform(-span, span, n)
    b = rng.uniform(-span, span, k)
    if ties:
        m = min(n, k) // 2 + 1
        b[rng.integers(0, k, m)] = a[rng.integers(0, n, m)]
    return a, b


# sort
for dt in (np.float32, np.float64):
    for m in (1, 2, 5, 100, 4097, 100000):
        raw = rng.uniform(-3, 3, m).astype(dt)
        raw[rng.integers(0, m, m // 3 + 1)] = raw[rng.integers(0, m, m // 3 + 1)]
        if m > 4:
            raw[:4] = [0.0, -0.0, 0.0, -0.0]
        s = L.sort_anchors(raw, dtype=dt)
        v, p, d = O.sort_anchors(raw, dtype=dt)
        ok = np.array_equal(s.perm, p) and np.array_equal(s.values.view(np.uint8), v.view(np.uint8))
        rep(f"sort {dt.__name__} m={m}", ok)
raw = np.array([0.0, -0.0, 1.0, -0.0, 0.0])
s = L.sort_anchors(raw)
rep("sort +-0 golden", list(s.perm) == [0, 1, 3, 4, 2] and np.signbit(s.values).tolist() == [False, True, True, False, False],
    f"{s.perm} {np.signbit(s.values)}")

# plan / ranks / matvec (fp64 vs dense oracle)
for trial in range(30):
    n, k = rng.integers(1, 300, 2)
    a, b = inst(n, k, ties=trial % 3 == 0)
    t = 1.0 if trial % 2 else 0.37
    x = rng.uniform(-1, 1, k)
    g = rng.uniform(-1, 1, n)
    op = L.LaplexOperator(a, b, t)
    oo = O.OracleOp(a, b, t)
    ok = True
    for side in (0, 1):
        vv, pp, dd = oo.sorted(side)
        s = op._sorted(side)
        ok &= np.array_equal(s.perm, pp) and np.array_equal(s.values, vv)
    rep(f"plan sorted n={n} k={k}", ok)
    ok = np.array_equal(op.row_buckets(), oo.ranks(0)) and np.array_equal(op.col_buckets(), oo.ranks(1))
    A = oo.sorted(0)[0]
    Bv = oo.sorted(1)[0]
    ok &= np.array_equal(op.ranks(0, True), np.searchsorted(Bv, A, "left"))
    ok &= np.array_equal(op.ranks(1, True), np.searchsorted(A, Bv, "left"))
    rep(f"ranks n={n} k={k}", ok)
    y = op.matvec(x)
    want = O.dense_matvec(a, b, t, x)
    e = O.rel_err_l2(y, want)
    rep(f"matvec f64 n={n} k={k}", e <= 1e-13, f"{e:.2e}")
    yt = op.matvec_transpose(g)
    e = O.rel_err_l2(yt, O.dense_matvec(b, a, t, g))
    rep(f"transpose f64", e <= 1e-13, f"{e:.2e}")
    v = L.matvec_vjp(op, x, g)
    xb, ab, bb = oo.vjp(x, g)
    e1, e2, e3 = O.rel_err_l2(v.x_bar, xb), O.rel_err_l2(v.a_bar, ab), O.rel_err_l2(v.b_bar, bb)
    rep(f"vjp f64", max(e1, e2, e3) <= 1e-12, f"{e1:.2e} {e2:.2e} {e3:.2e}")
    rep("vjp xbar == transpose bitwise", np.array_equal(v.x_bar, yt))
    X = rng.uniform(-1, 1, (3, k))
    Y = op.batch_matvec(X)
    rep("batch bitwise", all(np.array_equal(Y[r], op.matvec(X[r])) for r in range(3)))

# phased
for trial in range(5):
    n, k = rng.integers(1, 200, 2)
    a, b = inst(n, k)
    phi = rng.uniform(0, 6.28, n)
    psi = rng.uniform(0, 6.28, k)
    x = rng.uniform(-1, 1, k)
    g = rng.uniform(-1, 1, n)
    op = L.LaplexOperator(a, b, 1.1, phi, psi)
    oo = O.OracleOp(a, b, 1.1, phi, psi)
    e = O.rel_err_l2(op.phased_matvec(x), oo.phased_matvec(x))
    rep("phased matvec", e <= 1e-12, f"{e:.2e}")
    v = L.phased_matvec_vjp(op, x, g)
    w = oo.phased_vjp(x, g)
    errs = [O.rel_err_l2(u, q) for u, q in zip((v.x_bar, v.a_bar, v.b_bar, v.phi_bar, v.psi_bar), w)]
    rep("phased vjp", max(errs) <= 1e-11, " ".join(f"{q:.1e}" for q in errs))
    D = rng.uniform(-1.5, 1.5, k)
    e = O.rel_err_l2(op.phased_gram(D).matrix, oo.phased_gram(D))
    rep("phased gram", e <= 1e-10, f"{e:.2e}")

# gram
for trial in range(5):
    n, k = rng.integers(1, 64), rng.integers(1, 2000)
    a, b = inst(n, k, 4.0)
    D = rng.uniform(-2, 2, k)
    op = L.LaplexOperator(a, b, 1.6)
    M = op.weighted_gram(D).matrix
    e = O.rel_err_l2(M, O.dense_gram(a, b, 1.6, D))
    rep("gram", e <= 1e-10 and np.array_equal(M, M.T), f"{e:.2e}")

# scans
s = L.sort_anchors(rng.uniform(-3, 3, 10000))
p = rng.uniform(-1, 1, 10000)
pre, suf = O.decay_scan(s.values, p)
rep("prefix scan", O.rel_err_l2(L.prefix_decay_scan(s, p), pre) <= 1e-12)
rep("suffix scan", O.rel_err_l2(L.suffix_decay_scan(s, p), suf) <= 1e-12)

# fp32 at scale vs fp64 oracle
for lg in (16, 20, 22):
    N = 1 << lg
    a = rng.uniform(-100, 100, N).astype(np.float32)
    b = rng.uniform(-100, 100, N).astype(np.float32)
    x = rng.uniform(-1, 1, N).astype(np.float32)
    g = rng.uniform(-1, 1, N).astype(np.float32)
    t0 = time.time()
    op = L.LaplexOperator(a, b, 1.0, dtype=np.float32)
    y = op.matvec(x)
    v = L.matvec_vjp(op, x, g)
    t1 = time.time()
    oo = O.OracleOp(a.astype(np.float64), b.astype(np.float64), 1.0)
    yw = oo.matvec(x.astype(np.float64), 2)
    xb, ab, bb = oo.vjp(x.astype(np.float64), g.astype(np.float64))
    of = O.OracleOp(a, b, 1.0, dtype=np.float32)
    ok = True
    for side in (0, 1):
        ok &= np.array_equal(op._sorted(side).perm, of.sorted(side)[1])
    rep(f"f32 perms 2^{lg}", ok)
    errs = [O.rel_err_l2(y, yw), O.rel_err_l2(v.x_bar, xb), O.rel_err_l2(v.a_bar, ab), O.rel_err_l2(v.b_bar, bb)]
    rep(f"f32 vs f64 oracle 2^{lg}", max(errs) <= 1e-5, " ".join(f"{q:.2e}" for q in errs) + f" gpu {t1-t0:.2f}s")

print("FAILS", fails)
sys.exit(1 if fails else 0)
