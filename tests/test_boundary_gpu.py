"""GPU: the boundary entry points added for SURVEY 8(b) -- device variants of
sort_anchors / decay scans / gram_vjp_weights, the Gram-vector product, async
plan creation, stream-ordered plan release from another stream -- against
the host-pointer entries (bitwise) and the oracle."""
import numpy as np
import pytest

import oracle as O
import paper_2605_24584_b200 as L

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("m", [1, 1000, 70001, (1 << 22) + 5])
def test_sort_dev_equals_host_sort_and_oracle(torch, dt, m):
    rng = np.random.default_rng(m)
    raw = rng.integers(-500, 500, m).astype(dt) / dt(7)  # ties
    raw[::13] = -0.0
    v, p, d = L.sort_anchors_dev(torch.from_numpy(raw).cuda())
    hv = L.sort_anchors(raw, dtype=dt)
    assert np.array_equal(v.cpu().numpy().view(np.uint8), hv.values.view(np.uint8))
    assert np.array_equal(p.cpu().numpy().view(np.uint32).astype(np.uint64), hv.perm)
    assert np.array_equal(d.cpu().numpy(), hv.decays)
    assert O.verify_sort(raw, 1.0, p.cpu().numpy().view(np.uint32), dtype=dt) == -1


def test_sort_dev_reports_nonfinite(torch):
    raw = torch.tensor([1.0, float("nan"), 2.0], device="cuda")
    with pytest.raises(L.NonFinite):
        L.sort_anchors_dev(raw)
    with pytest.raises(L.EmptyInput):
        L.sort_anchors_dev(torch.empty(0, device="cuda"))


@pytest.mark.parametrize("m", [1, 5000, 1 << 21])
def test_scan_dev_equals_host_scan(torch, m):
    rng = np.random.default_rng(m)
    vals = np.sort(rng.uniform(-50, 50, m))
    pay = rng.uniform(-1, 1, m)
    pre, suf = L.decay_scan_dev(torch.from_numpy(vals).cuda(), torch.from_numpy(pay).cuda())
    s = L.SortedAnchors(vals, np.arange(m, dtype=np.uint64), np.exp(vals[:-1] - vals[1:]))
    assert np.array_equal(pre.cpu().numpy(), L.prefix_decay_scan(s, pay))
    assert np.array_equal(suf.cpu().numpy(), L.suffix_decay_scan(s, pay))
    opre, osuf = O.decay_scan(vals, pay)
    assert O.rel_err_l2(pre.cpu().numpy(), opre) <= 1e-12 and O.rel_err_l2(suf.cpu().numpy(), osuf) <= 1e-12


def test_gram_vjp_weights_dev(torch):
    rng = np.random.default_rng(9)
    n, k = 40, 3000
    a, b = rng.uniform(-5, 5, n), rng.uniform(-5, 5, k)
    D = rng.uniform(0.1, 1, k)
    Gb = rng.uniform(-1, 1, (n, n))
    Gb = Gb + Gb.T
    host = L.gram_vjp_weights(L.LaplexOperator(a, b, 0.7), D, Gb)
    dop = L.DeviceOperator(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), 0.7)
    dev = dop.gram_vjp_weights(torch.from_numpy(Gb).cuda())
    assert np.array_equal(dev.cpu().numpy(), host)
    assert O.rel_err_l2(host, O.OracleOp(a, b, 0.7).gram_vjp_weights(D, Gb)) <= 1e-11
    Ga = Gb.copy()
    Ga[3, 1] += 1e-3
    with pytest.raises(L.AsymmetricCotangent):
        dop.gram_vjp_weights(torch.from_numpy(Ga).cuda())
    Gn = Gb.copy()
    Gn[2, 2] = np.inf
    with pytest.raises(L.NonFinite):
        dop.gram_vjp_weights(torch.from_numpy(Gn).cuda())


@pytest.mark.parametrize("n,k,rows", [(1, 1, 1), (3000, 2000, 3), ((1 << 22) + 3, (1 << 22) + 11, 2)])
def test_gram_apply_bitwise_composition_and_oracle(torch, n, k, rows):
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    a = torch.empty(n, device="cuda").uniform_(-30, 30, generator=g)
    b = torch.empty(k, device="cuda").uniform_(-30, 30, generator=g)
    b[: min(n, k) // 3] = a[: min(n, k) // 3]  # ties
    X = torch.empty(rows, k, device="cuda").uniform_(-1, 1, generator=g)
    dop = L.DeviceOperator(a, b, 0.9)
    Y = dop.gram_apply(X)
    assert torch.equal(Y, dop.apply(dop.apply(X), transpose=True))
    if n * k <= 10 ** 7:
        oo = O.OracleOp(a.double().cpu().numpy(), b.double().cpu().numpy(), float(np.float32(0.9)))
        for r in range(rows):
            want = oo.matvec_transpose(oo.matvec(X[r].double().cpu().numpy()))
            assert O.rel_err_l2(Y[r].cpu().numpy(), want) <= 1e-5
    # host entry and the C++-style wrapper path
    op = L.LaplexOperator(a.cpu().numpy(), b.cpu().numpy(), 0.9, dtype=np.float32)
    assert np.array_equal(op.batch_gram_matvec(X.cpu().numpy()), Y.cpu().numpy())


def test_gram_apply_errors(torch):
    op = L.LaplexOperator([0.0, 1.0], [0.5], 1.0, [0.1, 0.2], [0.3])
    with pytest.raises(L.PhasePresent):
        op.batch_gram_matvec([[1.0]])
    op = L.LaplexOperator([0.0, 1.0], [0.5, 2.0])
    with pytest.raises(L.DimensionMismatch):
        op.batch_gram_matvec([[1.0, 2.0, 3.0]])
    with pytest.raises(L.NonFinite):
        op.batch_gram_matvec([[1.0, np.nan]])


def test_async_plan_create_and_check(torch):
    import ctypes as C
    from paper_2605_24584_b200 import _lib
    lib = _lib.lib()
    a = torch.tensor([0.0, float("inf"), 1.0], device="cuda")
    b = torch.tensor([0.5, 1.5], device="cuda")
    h = C.c_void_p()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.laplex_plan_create_dev_async(0, a.data_ptr(), 3, b.data_ptr(), 2, 1.0, None, None, st, C.byref(h)) == 0
    assert lib.laplex_plan_check(h) == 2  # NonFinite, reported late
    assert lib.laplex_plan_release(h) == 0
    a[1] = 0.25
    assert lib.laplex_plan_create_dev_async(0, a.data_ptr(), 3, b.data_ptr(), 2, 1.0, None, None, st, C.byref(h)) == 0
    assert lib.laplex_plan_check(h) == 0
    assert lib.laplex_plan_release(h) == 0
    # fp32 plans reject a temperature that rounds to 0 or inf
    assert lib.laplex_plan_create_dev(0, a.data_ptr(), 3, b.data_ptr(), 2, 1e-300, None, None, st, C.byref(h)) == 2
    assert lib.laplex_plan_create_dev(0, a.data_ptr(), 3, b.data_ptr(), 2, 1e39, None, None, st, C.byref(h)) == 2
    assert lib.laplex_pool_trim() == 0


def test_plan_used_and_released_across_streams(torch):
    """A plan created on one stream, its role-swapped data built lazily on a
    second, used on a third and released while that work may still run: the
    results equal the single-stream ones (stream-ordered build and release)."""
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    n = (1 << 22) + 77
    a = torch.empty(n, device="cuda").uniform_(-50, 50, generator=g)
    b = torch.empty(n, device="cuda").uniform_(-50, 50, generator=g)
    x = torch.empty(2, n, device="cuda").uniform_(-1, 1, generator=g)
    ref_op = L.DeviceOperator(a, b, 1.0)
    want = ref_op.apply(x, transpose=True)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        op = L.DeviceOperator(a, b, 1.0, stream=s1)
    outs = []
    for s in (s2, s1):
        with torch.cuda.stream(s):
            outs.append(op.apply(x, transpose=True, stream=s))
    del op  # released while s1 / s2 may still be running
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, want)


def test_backward_zero_rows_zeroes_phase_cotangents(torch):
    a = torch.tensor([0.0, 1.0], device="cuda")
    b = torch.tensor([0.5, 2.0, 3.0], device="cuda")
    phi = torch.tensor([0.1, 0.2], device="cuda")
    psi = torch.tensor([0.3, 0.4, 0.5], device="cuda")
    dop = L.DeviceOperator(a, b, 1.0, phi, psi)
    X = torch.empty(0, 3, device="cuda")
    G = torch.empty(0, 2, device="cuda")
    outs = [torch.full((m,), 7.0, device="cuda") for m in (2, 3, 2, 3)]
    xb = torch.empty(0, 3, device="cuda")
    dop.backward(X, G, xb, *outs)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.count_nonzero(o) == 0


@pytest.mark.parametrize("phased,n", [(False, 5000), (True, 7000), (False, (1 << 22) + 9)])
def test_saved_forward_x_reuse_is_bitwise(torch, phased, n):
    """apply(save_x) + backward(reuse_x) == plain backward, bitwise; a reuse
    request for a different x (or after the saved x was consumed) recomputes."""
    g_ = torch.Generator(device="cuda")
    g_.manual_seed(n)
    u = lambda *s, lo=-1.0, hi=1.0: torch.empty(*s, device="cuda").uniform_(lo, hi, generator=g_)  # noqa: E731
    k = n + 31
    a, b = u(n, lo=-40, hi=40), u(k, lo=-40, hi=40)
    ph = (u(n, lo=0, hi=6), u(k, lo=0, hi=6)) if phased else (None, None)
    X, X2, G = u(2, k), u(2, k), u(2, n)
    dop = L.DeviceOperator(a, b, 1.0, *ph)
    want = dop.backward(X, G)
    y1 = dop.apply(X, save_x=True)
    got = dop.backward(X, G, reuse_x=True)
    for w, gg in zip(want, got):
        assert (w is None and gg is None) or torch.equal(w, gg)
    assert torch.equal(y1, dop.apply(X))
    dop.apply(X2, save_x=True)
    got2 = dop.backward(X, G, reuse_x=True)  # not the saved x: recomputed
    for w, gg in zip(want, got2):
        assert (w is None and gg is None) or torch.equal(w, gg)
    got3 = dop.backward(X2, G, reuse_x=True)
    want3 = dop.backward(X2, G)
    for w, gg in zip(want3, got3):
        assert (w is None and gg is None) or torch.equal(w, gg)


@pytest.mark.parametrize("phased,n", [(False, 6000), (True, 5000), (False, (1 << 21) + 5)])
def test_host_api_saved_x_reuse_is_bitwise(torch, phased, n):
    """Host-pointer API: laplex_apply(SAVE_X) + laplex_backward(REUSE_X) of the
    same host X skips the second upload of x and gives bitwise the results of
    a plain backward; a different host X is uploaded and recomputed."""
    from paper_2605_24584_b200 import laplex as LX
    rng = np.random.default_rng(n)
    k = n + 17
    a, b = rng.uniform(-30, 30, n).astype(np.float32), rng.uniform(-30, 30, k).astype(np.float32)
    ph = (rng.uniform(0, 6, n).astype(np.float32), rng.uniform(0, 6, k).astype(np.float32)) if phased else (None, None)
    X = rng.uniform(-1, 1, (2, k)).astype(np.float32)
    X2 = rng.uniform(-1, 1, (2, k)).astype(np.float32)
    G = rng.uniform(-1, 1, (2, n)).astype(np.float32)
    op = L.LaplexOperator(a, b, 1.0, *ph, dtype=np.float32)
    base = LX.PHASED if phased else 0
    want = LX._vjp(op, X, G, base)
    op._apply(base | LX.SAVE_X, X, 2, k, n)
    fields = ("x_bar", "a_bar", "b_bar", "phi_bar", "psi_bar")
    got = LX._vjp(op, X, G, base | LX.REUSE_X)
    for f in fields:
        assert np.array_equal(getattr(want, f), getattr(got, f)), f
    op._apply(base | LX.SAVE_X, X2, 2, k, n)
    got2 = LX._vjp(op, X, G, base | LX.REUSE_X)  # not the saved host x: uploaded again
    for f in fields:
        assert np.array_equal(getattr(want, f), getattr(got2, f)), f


def test_device_operator_without_creation_sync():
    """DeviceOperator(sync=False) (laplex_plan_create_dev_async): results bitwise those
    of a synchronously created plan; non-finite anchors reported by check()."""
    import torch
    import paper_2605_24584_b200 as L
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    a = torch.empty(70_001, device=dev).uniform_(-50, 50, generator=g)
    b = torch.empty(50_003, device=dev).uniform_(-50, 50, generator=g)
    X = torch.empty(3, 50_003, device=dev).uniform_(-1, 1, generator=g)
    G = torch.empty(3, 70_001, device=dev).uniform_(-1, 1, generator=g)
    s, q = L.DeviceOperator(a, b, 0.7), L.DeviceOperator(a, b, 0.7, sync=False)
    assert torch.equal(s.apply(X), q.apply(X))
    for u, v in zip(s.backward(X, G)[:3], q.backward(X, G)[:3]):
        assert torch.equal(u, v)
    q.check()
    a[123] = float("nan")
    bad = L.DeviceOperator(a, b, 0.7, sync=False)
    with pytest.raises(Exception):
        bad.check()
