"""GPU: the range-sharded operator with its CUDA data path, N shards simulated
by threads in one process on cuda:0 (SimComm), against the unsharded device
path and the fp64 oracle."""
import threading

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _run_sim(a, b, x, g, t, world, dtype):
    import torch
    from paper_2605_24584_b200.sharded import GpuBackend, ShardedOperator, SimComm, SimWorld
    w = SimWorld(world)
    out = [None] * world
    err = []
    dev = torch.device("cuda:0")
    n, k = len(a), len(b)

    def body(r):
        try:
            torch.cuda.set_device(0)
            T = lambda v: torch.tensor(np.ascontiguousarray(v), dtype=dtype, device=dev)  # noqa: E731
            sa = slice(r * n // world, (r + 1) * n // world)
            sb = slice(r * k // world, (r + 1) * k // world)
            op = ShardedOperator(T(a[sa]), T(b[sb]), t, SimComm(w, r), GpuBackend(), samples=256)
            y = op.apply(T(x[sb]))
            xb, ab, bb = op.backward(T(x[sb]), T(g[sa]))
            torch.cuda.synchronize()
            out[r] = [v.double().cpu().numpy() for v in (y, xb, ab, bb)] + [op.n_recv, op.k_recv]
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)
            w.barrier.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for h in th:
        h.start()
    for h in th:
        h.join()
    if err:
        raise err[0]
    return [np.concatenate([o[i] for o in out]) for i in range(4)], [o[4] for o in out], [o[5] for o in out]


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_sharded_fp64_matches_oracle(world):
    import torch
    rng = np.random.default_rng(world)
    n, k = 20_000, 17_000
    a, b = rng.uniform(-30, 30, n), rng.uniform(-30, 30, k)
    a[::7] = np.round(a[::7], 1)
    b[::5] = np.round(b[::5], 1)
    x, g = rng.uniform(-1, 1, k), rng.uniform(-1, 1, n)
    (y, xb, ab, bb), nr, kr = _run_sim(a, b, x, g, 0.9, world, torch.float64)
    assert sum(nr) == n and sum(kr) == k
    oo = O.OracleOp(a, b, 0.9)
    assert O.rel_err_l2(y, oo.matvec(x)) <= 1e-12
    for got, want in zip((xb, ab, bb), oo.vjp(x, g)):
        assert O.rel_err_l2(got, want) <= 1e-12


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_fp32_at_scale(world):
    import torch
    rng = np.random.default_rng(10 + world)
    N = 1 << 21
    a = rng.uniform(-100, 100, N).astype(np.float32)
    b = rng.uniform(-100, 100, N).astype(np.float32)
    x = rng.uniform(-1, 1, N).astype(np.float32)
    g = rng.uniform(-1, 1, N).astype(np.float32)
    (y, xb, ab, bb), nr, kr = _run_sim(a, b, x, g, 1.0, world, torch.float32)
    assert min(nr) > 0.5 * N / world and min(kr) > 0.5 * N / world  # balanced ranges
    o64 = O.OracleOp(a.astype(np.float64), b.astype(np.float64), 1.0)
    assert O.rel_err_l2(y, o64.matvec(x.astype(np.float64), 2)) <= 1e-5
    for got, want in zip((xb, ab, bb), o64.vjp(x.astype(np.float64), g.astype(np.float64))):
        assert O.rel_err_l2(got, want) <= 1e-5


# --------------------------------------------------- the C++ host layer (product)
def _run_cpp(fn, world):
    """fn(rank, comm, stream) on `world` threads of this process, one CUDA
    stream each, ranks joined by a laplex "local" communicator."""
    import torch
    from paper_2605_24584_b200.sharded import Comm
    key = np.random.default_rng().integers(1, 2 ** 62)
    out, err = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            comm = Comm.local(int(key), world, r)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[r] = fn(r, comm, st)
            st.synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for h in th:
        h.start()
    for h in th:
        h.join(timeout=600)
    if err:
        raise err[0]
    return out


def _cpp_sharded(a, b, x, g, t, world, dtype, rows=1, reuse=True):
    import torch
    from paper_2605_24584_b200.sharded import CppShardedOperator
    n, k = a.shape[-1], b.shape[-1]

    def fn(r, comm, st):
        T = lambda v: torch.tensor(np.ascontiguousarray(v), dtype=dtype, device="cuda:0")  # noqa: E731
        sa = slice(r * n // world, (r + 1) * n // world)
        sb = slice(r * k // world, (r + 1) * k // world)
        op = CppShardedOperator(T(a[sa]), T(b[sb]), t, comm, stream=st)
        xs = T(x[:, sb])
        y = op.apply(xs, stream=st)
        xb, ab, bb = op.backward(xs, T(g[:, sa]), reuse_x=reuse, stream=st)
        st.synchronize()
        return [v.double().cpu().numpy() for v in (y, xb, ab, bb)] + [op.n_recv, op.k_recv]
    out = _run_cpp(fn, world)
    y = np.concatenate([o[0] for o in out], axis=1)
    xb = np.concatenate([o[1] for o in out], axis=1)
    return y, xb, np.concatenate([o[2] for o in out]), np.concatenate([o[3] for o in out]), \
        [o[4] for o in out], [o[5] for o in out]


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_cpp_sharded_fp64_matches_oracle(world):
    import torch
    rng = np.random.default_rng(100 + world)
    n, k = 20_000, 17_000
    a, b = rng.uniform(-30, 30, n), rng.uniform(-30, 30, k)
    a[::7] = np.round(a[::7], 1)
    b[::5] = np.round(b[::5], 1)  # ties inside and across ranks
    x, g = rng.uniform(-1, 1, (2, k)), rng.uniform(-1, 1, (2, n))
    y, xb, ab, bb, nr, kr = _cpp_sharded(a, b, x, g, 0.9, world, torch.float64, rows=2)
    assert sum(nr) == n and sum(kr) == k
    oo = O.OracleOp(a, b, 0.9)
    want_ab, want_bb = 0, 0
    for r in range(2):
        assert O.rel_err_l2(y[r], oo.matvec(x[r])) <= 1e-12
        wx, wa, wb = oo.vjp(x[r], g[r])
        assert O.rel_err_l2(xb[r], wx) <= 1e-12
        want_ab, want_bb = want_ab + wa, want_bb + wb
    assert O.rel_err_l2(ab, want_ab) <= 1e-12 and O.rel_err_l2(bb, want_bb) <= 1e-12


@pytest.mark.parametrize("world", [2, 8])
def test_cpp_sharded_fp32_at_scale(world):
    import torch
    rng = np.random.default_rng(20 + world)
    N = 1 << 22
    a = rng.uniform(-100, 100, N).astype(np.float32)
    b = rng.uniform(-100, 100, N).astype(np.float32)
    x = rng.uniform(-1, 1, (1, N)).astype(np.float32)
    g = rng.uniform(-1, 1, (1, N)).astype(np.float32)
    y, xb, ab, bb, nr, kr = _cpp_sharded(a, b, x, g, 1.0, world, torch.float32, reuse=False)
    assert min(nr) > 0.5 * N / world and min(kr) > 0.5 * N / world
    o64 = O.OracleOp(a.astype(np.float64), b.astype(np.float64), 1.0)
    assert O.rel_err_l2(y[0], o64.matvec(x[0].astype(np.float64), 2)) <= 1e-5
    for got, want in zip((xb[0], ab, bb), o64.vjp(x[0].astype(np.float64), g[0].astype(np.float64))):
        assert O.rel_err_l2(got, want) <= 1e-5


@pytest.mark.parametrize("world", [2, 4])
def test_replica_backward_sums_anchor_cotangents_over_ranks(world):
    """Batch replicas: every rank holds the full plan and B/world rows; the
    a_bar / b_bar (and phi_bar / psi_bar) each rank returns are the sums over
    ALL rows, identical bitwise on every rank, and equal the single-GPU call."""
    import torch
    import paper_2605_24584_b200 as L
    from paper_2605_24584_b200.sharded import replica_backward
    rng = np.random.default_rng(world)
    n, k, B = 3000, 2500, 8
    a, b = rng.uniform(-10, 10, n), rng.uniform(-10, 10, k)
    phi, psi = rng.uniform(0, 6, n), rng.uniform(0, 6, k)
    X, G = rng.uniform(-1, 1, (B, k)), rng.uniform(-1, 1, (B, n))
    for phased in (False, True):
        def fn(r, comm, st):
            T = lambda v: torch.tensor(v, dtype=torch.float64, device="cuda:0")  # noqa: E731
            dop = L.DeviceOperator(T(a), T(b), 0.8, T(phi) if phased else None, T(psi) if phased else None,
                                   stream=st)
            rs = slice(r * B // world, (r + 1) * B // world)
            outs = replica_backward(dop, comm, T(X[rs]), T(G[rs]), stream=st)
            st.synchronize()
            return [None if v is None else v.cpu().numpy() for v in outs]
        out = _run_cpp(fn, world)
        for o in out[1:]:
            for u, v in zip(o[1:], out[0][1:]):
                assert (u is None and v is None) or np.array_equal(u, v)
        T = lambda v: torch.tensor(v, dtype=torch.float64, device="cuda:0")  # noqa: E731
        ref = L.DeviceOperator(T(a), T(b), 0.8, T(phi) if phased else None, T(psi) if phased else None)
        want = ref.backward(T(X), T(G))
        assert np.allclose(np.concatenate([o[0] for o in out]), want[0].cpu().numpy(), rtol=0, atol=1e-13)
        for got, w in zip(out[0][1:], want[1:]):
            if w is not None:
                assert O.rel_err_l2(got, w.cpu().numpy()) <= 1e-13
