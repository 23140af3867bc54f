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
