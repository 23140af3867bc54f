"""CPU, world_size 2 over gloo: the range-sharded operator's host logic
(splitters, stable partition, all-to-all routing, carry folding) with the
per-shard math restated densely (NumpyBackend), against the fp64 oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_24584_b200.sharded import NumpyBackend, ShardedOperator, TorchComm
    a, b, x, g, t = case
    n, k = len(a), len(b)
    sa = slice(rank * n // world, (rank + 1) * n // world)
    sb = slice(rank * k // world, (rank + 1) * k // world)
    T = lambda v: torch.from_numpy(np.ascontiguousarray(v))  # noqa: E731
    op = ShardedOperator(T(a[sa]), T(b[sb]), t, TorchComm(), NumpyBackend(), samples=64)
    y = op.apply(T(x[sb]))
    xb, ab, bb = op.backward(T(x[sb]), T(g[sa]))
    q.put((rank, y.numpy(), xb.numpy(), ab.numpy(), bb.numpy(), op.n_recv, op.k_recv))
    dist.barrier()
    dist.destroy_process_group()


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cat = lambda i: np.concatenate([r[i] for r in res])  # noqa: E731
    return cat(1), cat(2), cat(3), cat(4), [r[5] for r in res], [r[6] for r in res]


@pytest.mark.parametrize("ties", [False, True])
def test_sharded_world2_matches_oracle(ties):
    rng = np.random.default_rng(5)
    n, k = 300, 260
    a = rng.uniform(-6, 6, n)
    b = rng.uniform(-6, 6, k)
    if ties:
        a = np.round(a, 1)  # long runs of equal values: must not straddle shards
        b = np.round(b, 1)
    x, g = rng.uniform(-1, 1, k), rng.uniform(-1, 1, n)
    t = 0.8
    y, xb, ab, bb, nr, kr = _run((a, b, x, g, t))
    assert sum(nr) == n and sum(kr) == k and min(nr) > 0  # both shards got work
    oo = O.OracleOp(a, b, t)
    assert O.rel_err_l2(y, oo.matvec(x)) <= 1e-12
    for got, want in zip((xb, ab, bb), oo.vjp(x, g)):
        assert O.rel_err_l2(got, want) <= 1e-12


def test_fold_external_combines_in_scan_order():
    from paper_2605_24584_b200.sharded import fold_external
    # three shards with one element each at anchors 0, 1, 3 (prefix values = payloads)
    tots = np.zeros((3, 3 + 2 * 2))
    for s, (anc, v) in enumerate([(0.0, 1.0), (1.0, 2.0), (3.0, 4.0)]):
        tots[s, :3] = [anc, anc, 1.0]
        tots[s, 3] = v          # prefix inc
        tots[s, 3 + 2] = v      # suffix inc
    ext = fold_external(tots, 2, 2, 1, [False], [False])
    assert ext[2] == 1 and ext[0] == 1.0
    assert np.isclose(ext[3], 2.0 + np.exp(-1.0) * 1.0)
    ext = fold_external(tots, 0, 2, 1, [False], [False])
    assert ext[2] == 2 and ext[1] == 1.0
    assert np.isclose(ext[3 + 2], 2.0 + np.exp(1.0 - 3.0) * 4.0)
