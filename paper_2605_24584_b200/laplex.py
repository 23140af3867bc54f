"""Python mirror of the reference LAPLEX interface, backed by the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/laplex/):

  LaplexOperator            operator.hpp:75-437  (matvec, matvec_transpose,
                            batch_matvec, weighted_gram, phased_matvec,
                            phased_gram, transposed, sorted_rows/cols,
                            col_buckets/row_buckets)
  matvec_vjp, phased_matvec_vjp, gram_vjp_weights     gradients.hpp:110-219
  sort_anchors, prefix_decay_scan, suffix_decay_scan,
  symmetric_matvec                                    scan.hpp:27-86
  Error and its subclasses                            errors.hpp:8-50

Host arrays are numpy.  `DeviceOperator` is the device-resident entry
(torch CUDA tensors in, torch CUDA tensors out, stream-ordered) used by the
benchmark; it calls the *_dev entry points.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum
from typing import Optional

import numpy as np

from ._lib import lib

F32, F64 = 0, 1
ROWS, COLS = 0, 1
TRANSPOSE, PHASED, REUSE_X, SAVE_X = 1, 2, 4, 8


class Error(RuntimeError):
    pass


class EmptyInput(Error):
    pass


class NonFinite(Error):
    pass


class DimensionMismatch(Error):
    pass


class PhasePresent(Error):
    pass


class PhaseAbsent(Error):
    pass


class AsymmetricCotangent(Error):
    pass


class NumericalBreakdown(Error):
    """errors.hpp:36 (raised by host-side callers such as FactorGaussian)."""


class InvalidSize(Error):
    pass


class InvalidArgument(Error):
    pass


class CudaError(Error):
    pass


_CODES = {1: EmptyInput, 2: NonFinite, 3: DimensionMismatch, 4: PhasePresent, 5: PhaseAbsent,
          6: AsymmetricCotangent, 7: InvalidSize, 8: InvalidArgument, 100: CudaError}


def _check(rc: int):
    if rc != 0:
        msg = lib().laplex_last_error().decode(errors="replace")
        raise _CODES.get(rc, Error)(msg)


class Dispatch(IntEnum):
    """operator.hpp:64-68.  Accepted and ignored: the B200 path has one algorithm."""
    Auto = 0
    ForceA = 1
    ForceB = 2


@dataclass
class SortedAnchors:
    values: np.ndarray
    perm: np.ndarray
    decays: np.ndarray

    def size(self) -> int:
        return len(self.values)


@dataclass
class MatvecCotangents:
    x_bar: np.ndarray
    a_bar: np.ndarray
    b_bar: np.ndarray
    phi_bar: np.ndarray
    psi_bar: np.ndarray


@dataclass
class GramResult:
    matrix: np.ndarray


def _dt(dtype) -> int:
    return F64 if np.dtype(dtype) == np.float64 else F32


def _host(x, dtype, name="x"):
    a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
    return a


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class LaplexOperator:
    """Implicit n x k kernel A_ij = exp(-|a_i - b_j|/t) cos(phi_i - psi_j)."""

    def __init__(self, row_anchors, col_anchors, temperature: float = 1.0, row_phases=None, col_phases=None,
                 dtype=np.float64, _handle=None, _raw=None):
        self.dtype = np.dtype(dtype)
        if _handle is not None:
            self._h = _handle
            (self._a, self._b, self._t, self._phi, self._psi) = _raw
            return
        a = _host(row_anchors, self.dtype)
        b = _host(col_anchors, self.dtype)
        phi = None if row_phases is None or len(row_phases) == 0 else _host(row_phases, self.dtype)
        psi = None if col_phases is None or len(col_phases) == 0 else _host(col_phases, self.dtype)
        if phi is not None and psi is not None and (len(phi) != len(a) or len(psi) != len(b)):
            # operator.hpp:96-98: lengths checked after emptiness/finiteness of anchors
            if len(a) == 0 or len(b) == 0:
                raise EmptyInput("LaplexOperator: empty anchor set")
            if not (np.all(np.isfinite(a)) and np.all(np.isfinite(b))):
                raise NonFinite("LaplexOperator: non-finite anchor")
            raise DimensionMismatch("LaplexOperator: phase lengths")
        h = C.c_void_p()
        _check(lib().laplex_plan_create(_dt(self.dtype), _p(a), len(a), _p(b), len(b), float(temperature),
                                        _p(phi), _p(psi), C.byref(h)))
        self._h = h
        self._a, self._b, self._t, self._phi, self._psi = a, b, float(temperature), phi, psi

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().laplex_plan_release(h)
            except Exception:
                pass
            self._h = None

    # ---- shape / accessors (operator.hpp:139-154) ----
    def n(self) -> int:
        return len(self._a)

    def k(self) -> int:
        return len(self._b)

    def temperature(self) -> float:
        return self._t

    def has_phases(self) -> bool:
        return self._phi is not None

    def row_anchors(self):
        return self._a

    def col_anchors(self):
        return self._b

    def _sorted(self, side: int) -> SortedAnchors:
        m = self.n() if side == ROWS else self.k()
        vals = np.empty(m, self.dtype)
        perm = np.empty(m, np.uint64)
        dec = np.empty(max(m - 1, 1), self.dtype)
        _check(lib().laplex_plan_sorted(self._h, side, _p(vals), _p(perm), _p(dec)))
        return SortedAnchors(vals, perm, dec[: max(m - 1, 0)])

    def sorted_rows(self) -> SortedAnchors:
        return self._sorted(ROWS)

    def sorted_cols(self) -> SortedAnchors:
        return self._sorted(COLS)

    def ranks(self, side: int, strict: bool = False) -> np.ndarray:
        m = self.n() if side == ROWS else self.k()
        out = np.empty(m, np.uint64)
        _check(lib().laplex_plan_ranks(self._h, side, int(strict), _p(out)))
        return out

    def col_buckets(self) -> np.ndarray:
        """r_of_col[j] = #{i : A_i <= B_j} (operator.hpp:111-115)."""
        return self.ranks(COLS, False)

    def row_buckets(self) -> np.ndarray:
        """j_of_row[i] = #{j : B_j <= A_i} (operator.hpp:116-120)."""
        return self.ranks(ROWS, False)

    def transposed(self) -> "LaplexOperator":
        """Role-swapped operator sharing the device plan (no re-sort)."""
        h = C.c_void_p()
        _check(lib().laplex_plan_transposed(self._h, C.byref(h)))
        return LaplexOperator(None, None, dtype=self.dtype, _handle=h,
                              _raw=(self._b, self._a, self._t, self._psi, self._phi))

    # ---- products ----
    def _apply(self, flags: int, X: np.ndarray, rows: int, cols: int, out_len: int) -> np.ndarray:
        Y = np.empty((rows, out_len), self.dtype)
        _check(lib().laplex_apply(self._h, flags, _p(X), rows, cols, _p(Y)))
        return Y

    def matvec(self, x, dispatch: Dispatch = Dispatch.Auto) -> np.ndarray:
        x = _host(x, self.dtype)
        return self._apply(0, x, 1, len(x), self.n())[0]

    def matvec_transpose(self, g, dispatch: Dispatch = Dispatch.Auto) -> np.ndarray:
        g = _host(g, self.dtype)
        if self.has_phases():
            raise PhasePresent("matvec_transpose: operator has phases, use phased path")
        return self._apply(TRANSPOSE, g, 1, len(g), self.k())[0]

    def batch_matvec(self, X, dispatch: Dispatch = Dispatch.Auto) -> np.ndarray:
        X = _host(X, self.dtype)
        if X.ndim != 2:
            raise DimensionMismatch("batch_matvec: X must be 2-D")
        return self._apply(0, X, X.shape[0], X.shape[1], self.n())

    def batch_gram_matvec(self, X) -> np.ndarray:
        """Y = A^T (A X^T) row by row: the Gram-vector composition
        matvec_transpose(matvec(x)) of SPEC.md:187 in one device call (the
        intermediate stays in sorted order on the device; bitwise equal to
        the composition).  Extension: not a member of the reference class."""
        X = np.atleast_2d(_host(X, self.dtype))
        rows, cols = X.shape
        Y = np.empty((rows, self.k()), self.dtype)
        _check(lib().laplex_gram_apply(self._h, _p(X), rows, cols, _p(Y)))
        return Y

    def phased_matvec(self, x, dispatch: Dispatch = Dispatch.Auto) -> np.ndarray:
        x = _host(x, self.dtype)
        return self._apply(PHASED, x, 1, len(x), self.n())[0]

    def weighted_gram(self, D) -> GramResult:
        D = _host(D, self.dtype)
        M = np.empty((self.n(), self.n()), self.dtype)
        _check(lib().laplex_gram(self._h, 0, _p(D), len(D), _p(M)))
        return GramResult(M)

    def phased_gram(self, D) -> GramResult:
        D = _host(D, self.dtype)
        M = np.empty((self.n(), self.n()), self.dtype)
        _check(lib().laplex_gram(self._h, PHASED, _p(D), len(D), _p(M)))
        return GramResult(M)


def _vjp(op: LaplexOperator, x, g, flags: int) -> MatvecCotangents:
    x = _host(x, op.dtype)
    g = _host(g, op.dtype)
    batched = x.ndim == 2
    X = x if batched else x[None, :]
    G = g if g.ndim == 2 else g[None, :]
    rows = X.shape[0]
    n, k = op.n(), op.k()
    xb = np.empty((rows, k), op.dtype)
    ab = np.empty(n, op.dtype)
    bb = np.empty(k, op.dtype)
    pb = np.empty(n, op.dtype) if flags & PHASED else np.empty(0, op.dtype)
    qb = np.empty(k, op.dtype) if flags & PHASED else np.empty(0, op.dtype)
    _check(lib().laplex_backward(op._h, flags, _p(X), rows, X.shape[1], _p(G), G.shape[1], _p(xb), _p(ab), _p(bb),
                                 _p(pb) if flags & PHASED else None, _p(qb) if flags & PHASED else None))
    return MatvecCotangents(xb if batched else xb[0], ab, bb, pb, qb)


def matvec_vjp(op: LaplexOperator, x, g) -> MatvecCotangents:
    """gradients.hpp:110-135 (x may also be a batch; a_bar/b_bar then sum over rows)."""
    return _vjp(op, x, g, 0)


def phased_matvec_vjp(op: LaplexOperator, x, g) -> MatvecCotangents:
    """gradients.hpp:139-184."""
    return _vjp(op, x, g, PHASED)


def gram_vjp_weights(op: LaplexOperator, D, G_bar) -> np.ndarray:
    """gradients.hpp:190-219."""
    D = _host(D, op.dtype)
    G = _host(G_bar, op.dtype)
    out = np.empty(op.k(), op.dtype)
    _check(lib().laplex_gram_vjp_weights(op._h, _p(D), len(D), _p(G), G.shape[0], G.shape[1] if G.ndim == 2 else 0,
                                         _p(out)))
    return out


def sort_anchors(raw, dtype=np.float64) -> SortedAnchors:
    """scan.hpp:27-46 (device onesweep radix sort, t = 1)."""
    r = _host(raw, dtype)
    m = len(r)
    vals = np.empty(max(m, 1), dtype)
    perm = np.empty(max(m, 1), np.uint64)
    dec = np.empty(max(m - 1, 1), dtype)
    _check(lib().laplex_sort(_dt(dtype), _p(r), m, _p(vals), _p(perm), _p(dec)))
    return SortedAnchors(vals[:m], perm[:m], dec[: max(m - 1, 0)])


def _scan(anchors: SortedAnchors, payload, which: str):
    dtype = anchors.values.dtype
    p = _host(payload, dtype)
    m = anchors.size()
    if len(p) != m:
        raise DimensionMismatch(f"{which}: payload length")
    out = np.empty(m, dtype)
    if m == 0:
        return out
    vals = np.ascontiguousarray(anchors.values)
    args = (_p(out), None) if which == "prefix_decay_scan" else (None, _p(out))
    _check(lib().laplex_scan(_dt(dtype), _p(vals), m, _p(p), *args))
    return out


def prefix_decay_scan(anchors: SortedAnchors, payload) -> np.ndarray:
    """scan.hpp:50-60."""
    return _scan(anchors, payload, "prefix_decay_scan")


def suffix_decay_scan(anchors: SortedAnchors, payload) -> np.ndarray:
    """scan.hpp:63-73."""
    return _scan(anchors, payload, "suffix_decay_scan")


def symmetric_matvec(anchors: SortedAnchors, x) -> np.ndarray:
    """scan.hpp:77-86: prefix + suffix - x."""
    x = _host(x, anchors.values.dtype)
    if len(x) != anchors.size():
        raise DimensionMismatch("symmetric_matvec: x length")
    y = prefix_decay_scan(anchors, x)
    s = suffix_decay_scan(anchors, x)
    return y + (s - x)


# ---------------------------------------------------------------------------
# device-resident entry (benchmark / framework integration)
# ---------------------------------------------------------------------------
class DeviceOperator:
    """Plan built from CUDA tensors; apply/backward on CUDA tensors, stream-ordered."""

    def __init__(self, a, b, temperature: float = 1.0, phi=None, psi=None, stream=None, sync=True):
        """sync=False: no host synchronisation at creation (laplex_plan_create_dev_async);
        non-finite anchors are then reported by check(), e.g. once per training step."""
        import torch
        assert a.is_cuda and b.is_cuda and a.dtype == b.dtype
        self.torch = torch
        self.dtype = a.dtype
        self.n, self.k = a.numel(), b.numel()
        st = self._stream(stream)
        h = C.c_void_p()
        dt = F64 if a.dtype == torch.float64 else F32
        create = lib().laplex_plan_create_dev if sync else lib().laplex_plan_create_dev_async
        _check(create(dt, a.data_ptr(), self.n, b.data_ptr(), self.k, float(temperature),
                      phi.data_ptr() if phi is not None else None,
                      psi.data_ptr() if psi is not None else None, st, C.byref(h)))
        self._h = h
        self.phased = phi is not None

    def check(self):
        """Raise the creation errors of a sync=False plan (waits for its build)."""
        _check(lib().laplex_plan_check(self._h))

    def _stream(self, stream):
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().laplex_plan_release(h)
            except Exception:
                pass
            self._h = None

    def apply(self, X, out=None, transpose=False, stream=None, save_x=False):
        """Y = A X (or A^T X).  save_x: keep the sorted x for backward(..., reuse_x=True)
        (LAPLEX_SAVE_X, the autograd "save for backward" of x)."""
        torch = self.torch
        rows = X.shape[0] if X.dim() == 2 else 1
        out_len = self.k if transpose else self.n
        if out is None:
            out = torch.empty((rows, out_len), dtype=self.dtype, device=X.device)
        flags = (TRANSPOSE if transpose else 0) | (PHASED if self.phased else 0) | (SAVE_X if save_x else 0)
        _check(lib().laplex_apply_dev(self._h, flags, X.data_ptr(), rows, out.data_ptr(), self._stream(stream)))
        return out

    def transposed(self) -> "DeviceOperator":
        """Role-swapped operator sharing the device plan (operator.hpp:157-159; no re-sort)."""
        h = C.c_void_p()
        _check(lib().laplex_plan_transposed(self._h, C.byref(h)))
        t = DeviceOperator.__new__(DeviceOperator)
        t.torch, t.dtype, t._h, t.phased = self.torch, self.dtype, h, self.phased
        t.n, t.k = self.k, self.n
        return t

    def weighted_gram(self, D, stream=None):
        """M = A diag(D) A^T (n x n; phased_gram for a phased operator), operator.hpp:191-248."""
        M = self.torch.empty((self.n, self.n), dtype=self.dtype, device=D.device)
        _check(lib().laplex_gram_dev(self._h, PHASED if self.phased else 0, D.data_ptr(), M.data_ptr(),
                                     self._stream(stream)))
        return M

    def gram_vjp_weights(self, G_bar, stream=None):
        """D_bar (k) of gram_vjp_weights (gradients.hpp:190-219) for a symmetric
        n x n CUDA tensor G_bar; raises AsymmetricCotangent / NonFinite."""
        out = self.torch.empty(self.k, dtype=self.dtype, device=G_bar.device)
        _check(lib().laplex_gram_vjp_weights_dev(self._h, G_bar.data_ptr(), out.data_ptr(), self._stream(stream)))
        return out

    def gram_apply(self, X, out=None, stream=None):
        """Y = A^T (A X) per row (rows x k -> rows x k), stream-ordered."""
        torch = self.torch
        rows = X.shape[0] if X.dim() == 2 else 1
        if out is None:
            out = torch.empty((rows, self.k), dtype=self.dtype, device=X.device)
        _check(lib().laplex_gram_apply_dev(self._h, X.data_ptr(), rows, out.data_ptr(), self._stream(stream)))
        return out

    def backward(self, X, G, x_bar=None, a_bar=None, b_bar=None, phi_bar=None, psi_bar=None, stream=None,
                 reuse_x=False):
        """(x_bar, a_bar, b_bar, phi_bar, psi_bar).  reuse_x: X is the (unchanged) tensor of
        the preceding apply(..., save_x=True); its sorted copy is reused (bitwise same results)."""
        torch = self.torch
        rows = X.shape[0] if X.dim() == 2 else 1
        dev = X.device
        if x_bar is None:
            x_bar = torch.empty((rows, self.k), dtype=self.dtype, device=dev)
        if a_bar is None:
            a_bar = torch.empty(self.n, dtype=self.dtype, device=dev)
        if b_bar is None:
            b_bar = torch.empty(self.k, dtype=self.dtype, device=dev)
        if self.phased:
            if phi_bar is None:
                phi_bar = torch.empty(self.n, dtype=self.dtype, device=dev)
            if psi_bar is None:
                psi_bar = torch.empty(self.k, dtype=self.dtype, device=dev)
        flags = (PHASED if self.phased else 0) | (REUSE_X if reuse_x else 0)
        _check(lib().laplex_backward_dev(self._h, flags, X.data_ptr(), G.data_ptr(), rows, x_bar.data_ptr(),
                                         a_bar.data_ptr(), b_bar.data_ptr(),
                                         phi_bar.data_ptr() if phi_bar is not None else None,
                                         psi_bar.data_ptr() if psi_bar is not None else None, self._stream(stream)))
        return x_bar, a_bar, b_bar, phi_bar, psi_bar


    # ---- accessors (operator.hpp:151-154), copied to the host ----
    def sorted(self, side: int):
        """(values, perm) of one side in sorted order: numpy arrays of the plan's
        dtype and uint32 (the device layout; the reference's size_t values fit)."""
        m = self.n if side == ROWS else self.k
        vals = np.empty(m, np.float64 if self.dtype == self.torch.float64 else np.float32)
        perm = np.empty(m, np.uint64)
        _check(lib().laplex_plan_sorted(self._h, side, _p(vals), _p(perm), None))
        return vals, perm.astype(np.uint32)

    def ranks(self, side: int, strict: bool = False) -> np.ndarray:
        """side ROWS: j_of_row (J<=), COLS: r_of_col (R<=) -- operator.hpp:111-120."""
        m = self.n if side == ROWS else self.k
        out = np.empty(m, np.uint64)
        _check(lib().laplex_plan_ranks(self._h, side, int(strict), _p(out)))
        return out


def sort_anchors_dev(raw, stream=None):
    """sort_anchors (scan.hpp:27-46) on a CUDA tensor: (values, perm int32
    tensor holding the uint32 device permutation, decays); stream-ordered
    except for the one synchronisation that reports NonFinite."""
    import torch
    m = raw.numel()
    vals = torch.empty_like(raw)
    perm = torch.empty(m, dtype=torch.int32, device=raw.device)
    dec = torch.empty(max(m - 1, 1), dtype=raw.dtype, device=raw.device)
    s = stream if stream is not None else torch.cuda.current_stream()
    _check(lib().laplex_sort_dev(F64 if raw.dtype == torch.float64 else F32, raw.data_ptr(), m, vals.data_ptr(),
                                 perm.data_ptr(), dec.data_ptr(), None, C.c_void_p(s.cuda_stream)))
    return vals, perm, dec[: max(m - 1, 0)]


def decay_scan_dev(sorted_values, payload, stream=None):
    """(prefix, suffix) decay scans (scan.hpp:50-73) of CUDA tensors."""
    import torch
    m = sorted_values.numel()
    pre = torch.empty_like(payload)
    suf = torch.empty_like(payload)
    s = stream if stream is not None else torch.cuda.current_stream()
    _check(lib().laplex_scan_dev(F64 if payload.dtype == torch.float64 else F32, sorted_values.data_ptr(), m,
                                 payload.data_ptr(), pre.data_ptr(), suf.data_ptr(), C.c_void_p(s.cuda_stream)))
    return pre, suf


def pool_trim() -> None:
    """Return every unused byte of the library's device memory pool (it caches
    freed blocks for reuse, like torch's allocator; cf. torch.cuda.empty_cache)."""
    _check(lib().laplex_pool_trim())


def kernel_launches() -> int:
    return int(lib().laplex_kernel_launches())
