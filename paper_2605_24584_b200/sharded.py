"""Range-sharded LAPLEX over N ranks: one long vector, split
by VALUE across GPUs.

Per rank (SPMD), with user slices a_r, b_r, x_r, g_r (contiguous global index
ranges, rank order = global index order):

1. splitters: every rank samples a/t and b/t; one all-gather; the same N-1
   splitter VALUES everywhere.  shard(v) = #{splitters < v}, so a run of equal
   values never straddles shards (the reference's tie-inclusive co-ranks stay
   shard-local).
2. exchange: stable partition by shard (laplex_shard_partition_dev) and one
   all-to-all of the raw anchors (b carries x; in the VJP a carries g).  The
   received elements arrive in global-index order, so the local stable sort
   reproduces std::stable_sort of the whole vector.
3. local plan on the received anchors; begin = tile aggregates + local carries
   -> this shard's totals; one all-gather of the totals; every rank folds the
   totals of the shards below (prefix) and above (suffix) with
   exp(anchor difference) -> external carries; end = main kernel with them.
4. outputs travel back along the reverse all-to-all and are scattered into
   the caller's slice order.

The PRODUCT path is the C++ host layer in the library (lx_dist.inc:
laplex_sharded_* over a laplex_comm -- NCCL or in-process "local" ranks),
wrapped here by `Comm` and `CppShardedOperator`; it folds the external carries
on the device and synchronises the host only once, at creation.  The Python
`ShardedOperator` below is its restatement over pluggable backends: with
NumpyBackend (dense per-shard math on the CPU) and TorchComm over gloo it
tests the host logic (splitters, routing, carry folding) without a GPU; with
GpuBackend it drives the same kernels from Python.  Communicators for it:
TorchComm (torch.distributed) and SimComm (threads in one process).
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import List, Optional, Sequence

import numpy as np

from . import laplex as _lx
from ._lib import lib

F32, F64 = 0, 1


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
class TorchComm:
    """torch.distributed process group (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather(self, t):
        import torch
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return out

    def all_to_all(self, send, send_counts: Sequence[int], recv_counts: Sequence[int]):
        import torch
        out = torch.empty(int(sum(recv_counts)), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(out, send.contiguous(), output_split_sizes=list(map(int, recv_counts)),
                                    input_split_sizes=list(map(int, send_counts)), group=self.group)
        return out


class SimWorld:
    """Shared state of an in-process simulated world (one thread per rank)."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots: List[object] = [None] * world


class SimComm:
    def __init__(self, world: SimWorld, rank: int):
        self.w = world
        self.rank = rank
        self.world = world.world

    def _exchange(self, item):
        self.w.slots[self.rank] = item
        self.w.barrier.wait()
        got = list(self.w.slots)
        self.w.barrier.wait()
        return got

    def all_gather(self, t):
        return [x.clone() for x in self._exchange(t)]

    def all_to_all(self, send, send_counts, recv_counts):
        import torch
        offs = np.concatenate([[0], np.cumsum(send_counts)]).astype(np.int64)
        parts = self._exchange([send[offs[i]:offs[i + 1]] for i in range(self.world)])
        pieces = [parts[src][self.rank].to(send.device) for src in range(self.world)]
        assert [len(p) for p in pieces] == list(map(int, recv_counts))
        return torch.cat(pieces) if pieces else send[:0]


# ---------------------------------------------------------------------------
# carry folding (host, fp64): combine the totals of the other shards
# ---------------------------------------------------------------------------
def fold_external(all_totals: np.ndarray, rank: int, slots: int, rows: int, pst: Sequence[bool],
                  qst: Sequence[bool]) -> np.ndarray:
    """all_totals[s] = [last, first, has, prefix[slot][rows], suffix[slot][rows]].

    Prefix carry of rank r = shards 0..r-1 combined left to right (anchor = the
    last of them); suffix carry = shards r+1..N-1 combined right to left
    (anchor = the first of them).  Combine of segments L then R (scan order):
    inc = inc_R + e * inc_L, strict = st_R + (s_L < s_R ? e * inc_L : st_L),
    with e = exp(-|s_L - s_R|).  Returns the ext array for laplex_*_end."""
    per = slots * rows
    out = np.zeros(3 + 2 * per)
    ch = slots // 2

    def vals(tot, off):
        v = tot[3 + off:3 + off + per].reshape(slots, rows)
        return v[0::2].astype(np.float64), v[1::2].astype(np.float64)  # inc, strict  [ch][rows]

    flags = 0
    run = None  # (anchor, inc, st)
    for s in range(rank):
        tot = all_totals[s]
        if tot[2] == 0:
            continue
        a_s = float(tot[0])
        inc, st = vals(tot, 0)
        if run is None:
            run = (a_s, inc, st)
        else:
            A, I, S = run
            e = np.exp(A - a_s)
            lt = A < a_s
            st = np.where(np.array(pst)[:, None], st + (e * I if lt else S), 0.0)
            run = (a_s, inc + e * I, st)
    if run is not None:
        flags |= 1
        out[0] = run[0]
        v = np.zeros((slots, rows))
        v[0::2] = run[1]
        v[1::2] = run[2]
        out[3:3 + per] = v.ravel()
    run = None
    for s in range(len(all_totals) - 1, rank, -1):
        tot = all_totals[s]
        if tot[2] == 0:
            continue
        a_s = float(tot[1])
        inc, st = vals(tot, per)
        if run is None:
            run = (a_s, inc, st)
        else:
            A, I, S = run  # running segment is to the right; prepend shard s
            e = np.exp(a_s - A)
            lt = a_s < A
            st = np.where(np.array(qst)[:, None], st + (e * I if lt else S), 0.0)
            run = (a_s, inc + e * I, st)
    if run is not None:
        flags |= 2
        out[1] = run[0]
        v = np.zeros((slots, rows))
        v[0::2] = run[1]
        v[1::2] = run[2]
        out[3 + per:] = v.ravel()
    out[2] = flags
    return out


# ---------------------------------------------------------------------------
# backends: the per-shard device work
# ---------------------------------------------------------------------------
def _dt(t):
    import torch
    return F64 if t.dtype == torch.float64 else F32


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _check(rc):
    _lx._check(rc)


class GpuBackend:
    """The CUDA library (C-ABI device entry points) on the current torch stream."""

    def __init__(self):
        import torch
        self.torch = torch

    def _st(self):
        return C.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def partition(self, raw, t, splitters):
        torch = self.torch
        m = raw.numel()
        perm = torch.empty(max(m, 1), dtype=torch.int32, device=raw.device)
        counts = torch.zeros(splitters.numel() + 1, dtype=torch.int32, device=raw.device)
        _check(lib().laplex_shard_partition_dev(_dt(raw), _ptr(raw), m, float(t), _ptr(splitters),
                                                splitters.numel(), _ptr(perm), _ptr(counts), self._st()))
        return perm[:m], counts

    def gather(self, src, idx, rows=1):
        torch = self.torch
        m = idx.numel()
        out = torch.empty((rows, m), dtype=src.dtype, device=src.device)
        _check(lib().laplex_gather_dev(_dt(src), _ptr(src), src.shape[-1], _ptr(idx), m, rows, _ptr(out),
                                       self._st()))
        return out

    def scatter(self, src, idx, ld, rows=1):
        torch = self.torch
        out = torch.empty((rows, ld), dtype=src.dtype, device=src.device)
        _check(lib().laplex_scatter_dev(_dt(src), _ptr(src), _ptr(idx), idx.numel(), rows, _ptr(out), ld,
                                        self._st()))
        return out

    def plan(self, a, b, t):
        h = C.c_void_p()
        _check(lib().laplex_shard_plan_create_dev(_dt(a), _ptr(a), a.numel(), _ptr(b), b.numel(), float(t),
                                                  None, None, self._st(), C.byref(h)))
        return h

    def release(self, plan):
        lib().laplex_plan_release(plan)

    def totals_count(self, plan, backward, rows):
        c = C.c_size_t()
        _check(lib().laplex_shard_totals_count(plan, 0, int(backward), rows, C.byref(c)))
        return c.value

    def fwd_begin(self, plan, x, rows, dtype):
        torch = self.torch
        tot = torch.empty(self.totals_count(plan, False, rows), dtype=dtype, device=x.device)
        w = C.c_void_p()
        _check(lib().laplex_shard_apply_begin(plan, 0, _ptr(x), rows, _ptr(tot), C.byref(w), self._st()))
        return w, tot

    def fwd_end(self, w, ext, n, rows, dtype, device):
        torch = self.torch
        y = torch.empty((rows, n), dtype=dtype, device=device)
        _check(lib().laplex_shard_apply_end(w, _ptr(ext), _ptr(y), self._st()))
        return y

    def bwd_begin(self, plan, x, g, rows, dtype):
        torch = self.torch
        tot = torch.empty(self.totals_count(plan, True, rows), dtype=dtype, device=x.device)
        w = C.c_void_p()
        _check(lib().laplex_shard_backward_begin(plan, 0, _ptr(x), _ptr(g), rows, _ptr(tot), C.byref(w),
                                                 self._st()))
        return w, tot

    def bwd_end(self, w, ext, n, k, rows, dtype, device):
        torch = self.torch
        xb = torch.empty((rows, k), dtype=dtype, device=device)
        ab = torch.empty(max(n, 1), dtype=dtype, device=device)
        bb = torch.empty(max(k, 1), dtype=dtype, device=device)
        _check(lib().laplex_shard_backward_end(w, _ptr(ext), _ptr(xb), _ptr(ab), _ptr(bb), None, None, self._st()))
        return xb, ab[:n], bb[:k]

    def to_device(self, arr, like):
        return self.torch.as_tensor(arr, dtype=like.dtype, device=like.device)


class NumpyBackend:
    """Dense CPU restatement of the per-shard work (tests of the host logic)."""

    def __init__(self):
        import torch
        self.torch = torch

    def partition(self, raw, t, splitters):
        torch = self.torch
        key = raw.numpy() / raw.numpy().dtype.type(t)
        sh = np.searchsorted(splitters.numpy(), key, side="left")  # #{splitters < key}
        perm = np.argsort(sh, kind="stable").astype(np.int32)
        counts = np.bincount(sh, minlength=splitters.numel() + 1).astype(np.int32)
        return torch.from_numpy(perm), torch.from_numpy(counts)

    def gather(self, src, idx, rows=1):
        return src.reshape(rows, -1)[:, idx.long()].clone()

    def scatter(self, src, idx, ld, rows=1):
        out = self.torch.zeros((rows, ld), dtype=src.dtype)
        out[:, idx.long()] = src.reshape(rows, -1)
        return out

    def plan(self, a, b, t):
        dt = a.numpy().dtype.type
        return {"a": a.numpy().astype(np.float64), "b": b.numpy().astype(np.float64),
                "sa": (a.numpy() / dt(t)).astype(np.float64), "sb": (b.numpy() / dt(t)).astype(np.float64),
                "t": float(t)}

    def release(self, plan):
        pass

    @staticmethod
    def _edges(P):
        anchors = np.concatenate([P["sa"], P["sb"]])
        return float(anchors.max()), float(anchors.min())

    def fwd_begin(self, P, x, rows, dtype):
        x = x.reshape(rows, -1).numpy().astype(np.float64)
        last, first = self._edges(P)
        sb = P["sb"]
        pre = x @ np.exp(sb - last)
        suf = x @ np.exp(first - sb)
        tot = np.zeros(3 + 2 * 2 * rows)
        tot[:3] = [last, first, 1.0]
        tot[3:3 + rows] = pre            # slot 0 (inc); slot 1 (strict) unused
        tot[3 + 2 * rows:3 + 3 * rows] = suf
        return (P, x), self.torch.from_numpy(tot)

    def fwd_end(self, w, ext, n, rows, dtype, device):
        P, x = w
        ext = ext.numpy()
        sa, sb = P["sa"], P["sb"]
        y = x @ np.exp(-np.abs(sa[:, None] - sb[None, :])).T
        per = 2 * rows
        if int(ext[2]) & 1:
            y += np.exp(ext[0] - sa)[None, :] * ext[3:3 + rows][:, None]
        if int(ext[2]) & 2:
            y += np.exp(sa - ext[1])[None, :] * ext[3 + per:3 + per + rows][:, None]
        return self.torch.from_numpy(y.astype(np.dtype(str(dtype).replace("torch.", ""))))

    def bwd_begin(self, P, x, g, rows, dtype):
        assert rows == 1
        x = x.reshape(-1).numpy().astype(np.float64)
        g = g.reshape(-1).numpy().astype(np.float64)
        last, first = self._edges(P)
        sa, sb = P["sa"], P["sb"]
        per = 4  # slots (g inc, g strict, x inc, x strict) x rows(1)
        tot = np.zeros(3 + 2 * per)
        tot[:3] = [last, first, 1.0]
        tot[3 + 0] = np.sum(np.exp(sa - last) * g)
        tot[3 + 1] = np.sum(np.where(sa < last, np.exp(sa - last) * g, 0.0))
        tot[3 + 2] = np.sum(np.exp(sb - last) * x)
        tot[3 + per + 0] = np.sum(np.exp(first - sa) * g)
        tot[3 + per + 2] = np.sum(np.exp(first - sb) * x)
        tot[3 + per + 3] = np.sum(np.where(sb > first, np.exp(first - sb) * x, 0.0))
        return (P, x, g), self.torch.from_numpy(tot)

    def bwd_end(self, w, ext, n, k, rows, dtype, device):
        P, x, g = w
        ext = ext.numpy()
        sa, sb, t = P["sa"], P["sb"], P["t"]
        K = np.exp(-np.abs(sa[:, None] - sb[None, :]))
        xb = K.T @ g
        below = (np.where(sa[:, None] < sb[None, :], K, 0.0) * g[:, None]).sum(0)   # a < b
        above = (np.where(sa[:, None] > sb[None, :], K, 0.0) * g[:, None]).sum(0)   # a > b
        right = (np.where(sb[None, :] > sa[:, None], K, 0.0) * x[None, :]).sum(1)   # b > a
        left = (np.where(sb[None, :] < sa[:, None], K, 0.0) * x[None, :]).sum(1)    # b < a
        per = 4
        fl = int(ext[2])
        if fl & 1:  # lower shards: every element is below every local anchor
            eg = np.exp(ext[0] - sb)
            xb += eg * ext[3 + 0]
            below += np.where(ext[0] < sb, eg * ext[3 + 0], ext[3 + 1])
            left += np.exp(ext[0] - sa) * ext[3 + 2]
        if fl & 2:
            eq = np.exp(sb - ext[1])
            xb += eq * ext[3 + per + 0]
            above += eq * ext[3 + per + 0]
            ea = np.exp(sa - ext[1])
            right += np.where(sa < ext[1], ea * ext[3 + per + 2], ext[3 + per + 3])
        ab = g / t * (right - left)
        bb = x / t * (above - below)
        T = self.torch
        cast = np.dtype(str(dtype).replace("torch.", ""))
        return T.from_numpy(xb[None, :].astype(cast)), T.from_numpy(ab.astype(cast)), T.from_numpy(bb.astype(cast))

    def to_device(self, arr, like):
        return self.torch.as_tensor(arr, dtype=like.dtype)


# ---------------------------------------------------------------------------
# the sharded operator (one instance per rank)
# ---------------------------------------------------------------------------
class ShardedOperator:
    """LAPLEX over a value-range-sharded long vector (B = 1)."""

    def __init__(self, a, b, t: float, comm, backend=None, samples: int = 4096):
        import torch
        self.torch = torch
        self.comm = comm
        self.be = backend or GpuBackend()
        self.t = float(t)
        self.dtype = a.dtype
        self.n_local, self.k_local = a.numel(), b.numel()
        W, r = comm.world, comm.rank
        # 1. splitters from a gathered sample of a/t and b/t (values only)
        tt = torch.tensor(self.t, dtype=a.dtype, device=a.device)

        def sample(v):
            if v.numel() == 0:
                return torch.full((samples,), float("nan"), dtype=v.dtype, device=v.device)
            # integer arithmetic: a float32 linspace rounds its endpoint past the last index
            # once numel > 2^24 (e.g. 2^29 elements per rank)
            idx = (torch.arange(samples, device=v.device, dtype=torch.int64) * (v.numel() - 1)) // max(1, samples - 1)
            return v[idx] / tt
        s = torch.cat([sample(a), sample(b)])
        allsamp = torch.cat(comm.all_gather(s))
        allsamp = allsamp[~torch.isnan(allsamp)].sort().values
        if W > 1 and allsamp.numel():
            q = (torch.arange(1, W, device=allsamp.device) * allsamp.numel()) // W
            self.splitters = allsamp[q.clamp(max=allsamp.numel() - 1)].contiguous()
        else:
            self.splitters = torch.empty(0, dtype=a.dtype, device=a.device)
        # 2. partition + exchange
        self.perm_a, ca = self.be.partition(a, self.t, self.splitters)
        self.perm_b, cb = self.be.partition(b, self.t, self.splitters)
        cnt = torch.stack([ca, cb]).to(torch.int64)
        allc = torch.stack(comm.all_gather(cnt)).cpu().numpy()  # [src][side][dst]
        self.send_a, self.send_b = allc[r, 0].tolist(), allc[r, 1].tolist()
        self.recv_a, self.recv_b = allc[:, 0, r].tolist(), allc[:, 1, r].tolist()
        ra = comm.all_to_all(self.be.gather(a, self.perm_a).reshape(-1), self.send_a, self.recv_a)
        rb = comm.all_to_all(self.be.gather(b, self.perm_b).reshape(-1), self.send_b, self.recv_b)
        self.n_recv, self.k_recv = ra.numel(), rb.numel()
        # 3. local plan on the received anchors (stable order = global index order)
        self.plan = self.be.plan(ra, rb, self.t) if self.n_recv + self.k_recv > 0 else None

    def __del__(self):
        if getattr(self, "plan", None) is not None:
            self.be.release(self.plan)
            self.plan = None

    def _route_in(self, v, perm, send, recv):
        return self.comm.all_to_all(self.be.gather(v.reshape(1, -1), perm).reshape(-1), send, recv)

    def _route_out(self, v, perm, send, recv, ld):
        back = self.comm.all_to_all(v.reshape(-1), recv, send)
        return self.be.scatter(back, perm, ld).reshape(-1)

    def _exchange_ext(self, tot, slots, pst, qst, count):
        torch = self.torch
        if tot is None:
            tot = torch.zeros(count, dtype=self.dtype, device=self.splitters.device)
        allt = torch.stack(self.comm.all_gather(tot)).double().cpu().numpy()
        return fold_external(allt, self.comm.rank, slots, 1, pst, qst)

    def apply(self, x):
        """y = A x for this rank's slice of x; returns this rank's slice of y."""
        torch = self.torch
        xr = self._route_in(x, self.perm_b, self.send_b, self.recv_b)
        work = None
        count = 3 + 2 * 2 * 1
        tot = None
        if self.plan is not None:
            work, tot = self.be.fwd_begin(self.plan, xr, 1, self.dtype)
        ext = self._exchange_ext(tot, 2, [False], [False], count)
        if work is not None:
            y_recv = self.be.fwd_end(work, self.be.to_device(ext, xr if xr.numel() else self.splitters),
                                     self.n_recv, 1, self.dtype, xr.device).reshape(-1)
        else:
            y_recv = torch.empty(0, dtype=self.dtype, device=self.splitters.device)
        return self._route_out(y_recv, self.perm_a, self.send_a, self.recv_a, self.n_local)

    def backward(self, x, g):
        """Cotangents of L = g^T A x: (x_bar, a_bar, b_bar) for this rank's slices."""
        torch = self.torch
        xr = self._route_in(x, self.perm_b, self.send_b, self.recv_b)
        gr = self._route_in(g, self.perm_a, self.send_a, self.recv_a)
        count = 3 + 2 * 4 * 1
        work, tot = (None, None)
        if self.plan is not None:
            work, tot = self.be.bwd_begin(self.plan, xr, gr, 1, self.dtype)
        ext = self._exchange_ext(tot, 4, [True, False], [False, True], count)
        dev = self.splitters.device
        if work is not None:
            like = xr if xr.numel() else gr
            xb, ab, bb = self.be.bwd_end(work, self.be.to_device(ext, like), self.n_recv, self.k_recv, 1,
                                         self.dtype, like.device)
        else:
            xb = torch.empty((1, 0), dtype=self.dtype, device=dev)
            ab = torch.empty(0, dtype=self.dtype, device=dev)
            bb = torch.empty(0, dtype=self.dtype, device=dev)
        x_bar = self._route_out(xb.reshape(-1), self.perm_b, self.send_b, self.recv_b, self.k_local)
        a_bar = self._route_out(ab, self.perm_a, self.send_a, self.recv_a, self.n_local)
        b_bar = self._route_out(bb, self.perm_b, self.send_b, self.recv_b, self.k_local)
        return x_bar, a_bar, b_bar


# ---------------------------------------------------------------------------
# the C++ host layer (product path): communicators + sharded operator
# ---------------------------------------------------------------------------
class Comm:
    """A laplex_comm: NCCL (`Comm.nccl`) or in-process ranks (`Comm.local`)."""

    def __init__(self, handle, rank, world):
        self.h, self.rank, self.world = handle, rank, world

    @classmethod
    def local(cls, key: int, world: int, rank: int) -> "Comm":
        h = C.c_void_p()
        _check(lib().laplex_comm_init_local(C.c_uint64(key), world, rank, C.byref(h)))
        return cls(h, rank, world)

    @classmethod
    def nccl(cls, world: int, rank: int, broadcast) -> "Comm":
        """broadcast(bytes_or_None) -> bytes: rank 0's 128-byte id to every rank
        (e.g. torch.distributed.broadcast_object_list)."""
        uid = None
        if rank == 0:
            buf = C.create_string_buffer(128)
            _check(lib().laplex_nccl_unique_id(buf))
            uid = buf.raw
        uid = broadcast(uid)
        h = C.c_void_p()
        _check(lib().laplex_comm_init_nccl(C.create_string_buffer(uid, 128), world, rank, C.byref(h)))
        return cls(h, rank, world)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            lib().laplex_comm_destroy(h)
            self.h = None


class CppShardedOperator:
    """laplex_sharded_*: this rank's slices a_r, b_r of one long vector (any
    rows per call); outputs come back in the slice order."""

    REUSE_X = 4

    def __init__(self, a, b, t: float, comm: Comm, stream=None):
        import torch
        self.torch, self.comm = torch, comm
        self.dtype = a.dtype
        self.n_local, self.k_local = a.numel(), b.numel()
        h = C.c_void_p()
        _check(lib().laplex_sharded_create_dev(comm.h, _dt(a), _ptr(a), self.n_local, _ptr(b), self.k_local,
                                               float(t), self._st(stream), C.byref(h)))
        self.h = h
        nr, kr = C.c_size_t(), C.c_size_t()
        _check(lib().laplex_sharded_shape(h, C.byref(nr), C.byref(kr)))
        self.n_recv, self.k_recv = nr.value, kr.value

    def _st(self, stream):
        s = stream if stream is not None else self.torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            lib().laplex_sharded_release(h)
            self.h = None

    def apply(self, x, out=None, stream=None):
        rows = x.shape[0] if x.dim() == 2 else 1
        if out is None:
            out = self.torch.empty((rows, self.n_local), dtype=self.dtype, device=x.device)
        _check(lib().laplex_sharded_apply_dev(self.h, _ptr(x), rows, _ptr(out), self._st(stream)))
        return out

    def backward(self, x, g, reuse_x=False, stream=None):
        torch = self.torch
        rows = x.shape[0] if x.dim() == 2 else 1
        xb = torch.empty((rows, self.k_local), dtype=self.dtype, device=x.device)
        ab = torch.empty(max(self.n_local, 1), dtype=self.dtype, device=x.device)
        bb = torch.empty(max(self.k_local, 1), dtype=self.dtype, device=x.device)
        _check(lib().laplex_sharded_backward_dev(self.h, self.REUSE_X if reuse_x else 0, _ptr(x), _ptr(g), rows,
                                                 _ptr(xb), _ptr(ab), _ptr(bb), self._st(stream)))
        return xb, ab[:self.n_local], bb[:self.k_local]


def replica_backward(dop, comm: Comm, X, G, stream=None):
    """Batch replicas: this rank's rows X, G over the replicated DeviceOperator
    `dop`; anchor cotangents summed over all ranks' rows (deterministic)."""
    import torch
    rows = X.shape[0]
    dev = X.device
    xb = torch.empty((rows, dop.k), dtype=dop.dtype, device=dev)
    ab = torch.empty(dop.n, dtype=dop.dtype, device=dev)
    bb = torch.empty(dop.k, dtype=dop.dtype, device=dev)
    pb = torch.empty(dop.n, dtype=dop.dtype, device=dev) if dop.phased else None
    qb = torch.empty(dop.k, dtype=dop.dtype, device=dev) if dop.phased else None
    s = stream if stream is not None else torch.cuda.current_stream()
    _check(lib().laplex_replica_backward_dev(dop._h, comm.h, 2 if dop.phased else 0, _ptr(X), _ptr(G), rows,
                                             _ptr(xb), _ptr(ab), _ptr(bb), _ptr(pb), _ptr(qb),
                                             C.c_void_p(s.cuda_stream)))
    return xb, ab, bb, pb, qb
