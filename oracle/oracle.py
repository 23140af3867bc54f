"""oracle/oracle.py -- ctypes front-end for the CPU CHECKERS.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product package.

Two backends with one interface:

* ``backend="c"``   -- oracle/liblaplex_oracle.so, the plain-C restatement of
  the reference algorithms (oracle/lxo_impl.inc, each function citing the
  reference file:line).  Travels to the GPU box.
* ``backend="ref"`` -- oracle/_ref/libref_laplex.so, the UNMODIFIED reference
  headers (/root/reference/proj/include) compiled by oracle/Makefile.  Built
  in the dev container; the built .so travels to the GPU box too.

All arrays are numpy; outputs are freshly allocated numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIBS = {"c": os.path.join(HERE, "liblaplex_oracle.so"),
         "ref": os.path.join(HERE, "_ref", "libref_laplex.so")}
_PREFIX = {"c": "lxo_", "ref": "lxr_"}
_handles = {}

ERRORS = {0: None, 1: "EmptyInput", 2: "NonFinite", 3: "DimensionMismatch", 4: "PhasePresent",
          5: "PhaseAbsent", 6: "AsymmetricCotangent", 97: "UnverifiedOrder", 99: "Error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {ERRORS.get(code, code)}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


def available(backend: str) -> bool:
    return os.path.exists(_LIBS[backend])


def _lib(backend: str):
    if backend not in _handles:
        path = _LIBS[backend]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle backend {backend!r} not built: {path} (run make -C oracle)")
        _handles[backend] = C.CDLL(path)
    return _handles[backend]


def _sfx(dtype) -> str:
    return "_f64" if np.dtype(dtype) == np.float64 else "_f32"


def _ctype(dtype):
    return C.c_double if np.dtype(dtype) == np.float64 else C.c_float


def _p(arr):
    return None if arr is None else arr.ctypes.data_as(C.c_void_p)


def _fn(backend, name, dtype):
    return getattr(_lib(backend), _PREFIX[backend] + name + _sfx(dtype))


def _arr(x, dtype):
    return None if x is None else np.ascontiguousarray(np.asarray(x, dtype=dtype))


def _check(rc, where):
    if rc != 0:
        raise OracleError(rc, where)


class OracleOp:
    """The reference ``LaplexOperator<Real>`` (operator.hpp:75-437) on the CPU."""

    def __init__(self, a, b, t=1.0, phi=None, psi=None, dtype=np.float64, backend="c"):
        self.dtype = np.dtype(dtype)
        self.backend = backend
        self.a = _arr(a, dtype)
        self.b = _arr(b, dtype)
        self.phi = _arr(phi, dtype)
        self.psi = _arr(psi, dtype)
        self.n, self.k = len(self.a), len(self.b)
        self.t = t
        h = C.c_void_p()
        f = _fn(backend, "op_create", dtype)
        f.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, _ctype(dtype), C.c_void_p,
                      C.c_void_p, C.POINTER(C.c_void_p)]
        _check(f(_p(self.a), self.n, _p(self.b), self.k, t, _p(self.phi), _p(self.psi), C.byref(h)),
               "LaplexOperator")
        self._h = h

    @classmethod
    def from_sorted(cls, a, b, t, perm_rows, perm_cols, phi=None, psi=None, dtype=np.float64):
        """The at-scale oracle: the same operator built over a GIVEN sort order
        (e.g. the GPU's), which lxo_op_create_sorted first proves equal to the
        reference's std::stable_sort (see lxo_verify_sort); only the sort itself
        is skipped, and the co-ranks come from one merge walk.  Raises
        OracleError(97) when a permutation is not the stable sort."""
        self = cls.__new__(cls)
        self.dtype = np.dtype(dtype)
        self.backend = "c"
        self.a, self.b = _arr(a, dtype), _arr(b, dtype)
        self.phi, self.psi = _arr(phi, dtype), _arr(psi, dtype)
        self.n, self.k = len(self.a), len(self.b)
        self.t = t
        pr = np.ascontiguousarray(perm_rows, dtype=np.uint32)
        pc = np.ascontiguousarray(perm_cols, dtype=np.uint32)
        h = C.c_void_p()
        f = _fn("c", "op_create_sorted", dtype)
        f.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, _ctype(dtype), C.c_void_p,
                      C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        _check(f(_p(self.a), self.n, _p(self.b), self.k, t, _p(self.phi), _p(self.psi), _p(pr), _p(pc),
                 C.byref(h)), "LaplexOperator(sorted)")
        self._h = h
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            f = _fn(self.backend, "op_destroy", self.dtype)
            f.argtypes = [C.c_void_p]
            f(h)
            self._h = None

    def _call(self, name, *args):
        f = _fn(self.backend, name, self.dtype)
        return f(self._h, *args)

    def transposed(self):
        """operator.hpp:157-159 (reference backend: the reference's own
        transposed(), which rebuilds the role-swapped operator)."""
        if self.backend != "ref":
            raise NotImplementedError("transposed() is exposed for the compiled reference only")
        h = C.c_void_p()
        f = _fn("ref", "op_transposed", self.dtype)
        f.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
        _check(f(self._h, C.byref(h)), "transposed")
        t = OracleOp.__new__(OracleOp)
        t.dtype, t.backend, t.a, t.b, t.phi, t.psi = self.dtype, "ref", self.b, self.a, None, None
        t.n, t.k, t.t, t._h = self.k, self.n, self.t, h
        return t

    def sorted(self, side: int):
        m = self.n if side == 0 else self.k
        vals = np.empty(m, self.dtype)
        perm = np.empty(m, np.uint64)
        dec = np.empty(max(m - 1, 1), self.dtype)
        self._call("op_sorted", C.c_int(side), _p(vals), _p(perm), _p(dec))
        return vals, perm, dec[: m - 1]

    def ranks(self, side: int):
        """side 0: j_of_row (J<=), side 1: r_of_col (R<=)."""
        m = self.n if side == 0 else self.k
        r = np.empty(m, np.uint64)
        self._call("op_ranks", C.c_int(side), _p(r))
        return r

    def matvec(self, x, dispatch=0):
        x = _arr(x, self.dtype)
        y = np.empty(self.n, self.dtype)
        _check(self._call("matvec", _p(x), C.c_size_t(len(x)), C.c_int(dispatch), _p(y)), "matvec")
        return y

    def matvec_transpose(self, g, dispatch=0):
        g = _arr(g, self.dtype)
        y = np.empty(self.k, self.dtype)
        _check(self._call("matvec_transpose", _p(g), C.c_size_t(len(g)), C.c_int(dispatch), _p(y)),
               "matvec_transpose")
        return y

    def batch_matvec(self, X, dispatch=0):
        X = _arr(X, self.dtype)
        B, cols = X.shape
        Y = np.empty((B, self.n), self.dtype)
        _check(self._call("batch_matvec", _p(X), C.c_size_t(B), C.c_size_t(cols), C.c_int(dispatch),
                          _p(Y)), "batch_matvec")
        return Y

    def phased_matvec(self, x, dispatch=0):
        x = _arr(x, self.dtype)
        y = np.empty(self.n, self.dtype)
        _check(self._call("phased_matvec", _p(x), C.c_size_t(len(x)), C.c_int(dispatch), _p(y)),
               "phased_matvec")
        return y

    def vjp(self, x, g):
        x = _arr(x, self.dtype)
        g = _arr(g, self.dtype)
        xb = np.empty(self.k, self.dtype)
        ab = np.empty(self.n, self.dtype)
        bb = np.empty(self.k, self.dtype)
        _check(self._call("matvec_vjp", _p(x), C.c_size_t(len(x)), _p(g), C.c_size_t(len(g)), _p(xb),
                          _p(ab), _p(bb)), "matvec_vjp")
        return xb, ab, bb

    def phased_vjp(self, x, g):
        x = _arr(x, self.dtype)
        g = _arr(g, self.dtype)
        xb = np.empty(self.k, self.dtype)
        ab = np.empty(self.n, self.dtype)
        bb = np.empty(self.k, self.dtype)
        pb = np.empty(self.n, self.dtype)
        qb = np.empty(self.k, self.dtype)
        _check(self._call("phased_matvec_vjp", _p(x), C.c_size_t(len(x)), _p(g), C.c_size_t(len(g)),
                          _p(xb), _p(ab), _p(bb), _p(pb), _p(qb)), "phased_matvec_vjp")
        return xb, ab, bb, pb, qb

    def weighted_gram(self, D):
        D = _arr(D, self.dtype)
        M = np.empty((self.n, self.n), self.dtype)
        _check(self._call("weighted_gram", _p(D), C.c_size_t(len(D)), _p(M)), "weighted_gram")
        return M

    def phased_gram(self, D):
        D = _arr(D, self.dtype)
        M = np.empty((self.n, self.n), self.dtype)
        _check(self._call("phased_gram", _p(D), C.c_size_t(len(D)), _p(M)), "phased_gram")
        return M

    def gram_vjp_weights(self, D, Gbar):
        D = _arr(D, self.dtype)
        Gbar = _arr(Gbar, self.dtype)
        out = np.empty(self.k, self.dtype)
        _check(self._call("gram_vjp_weights", _p(D), C.c_size_t(len(D)), _p(Gbar),
                          C.c_size_t(Gbar.shape[0]), C.c_size_t(Gbar.shape[1]), _p(out)),
               "gram_vjp_weights")
        return out


def sort_anchors(raw, dtype=np.float64, backend="c"):
    """scan.hpp:27-46 -> (values, perm(uint64), decays)."""
    raw = _arr(raw, dtype)
    m = len(raw)
    vals = np.empty(max(m, 1), dtype)
    perm = np.empty(max(m, 1), np.uint64)
    dec = np.empty(max(m - 1, 1), dtype)
    f = _fn(backend, "sort_anchors", dtype)
    _check(f(_p(raw), C.c_size_t(m), _p(vals), _p(perm), _p(dec)), "sort_anchors")
    return vals[:m], perm[:m], dec[: max(m - 1, 0)]


def verify_sort(raw, t, perm, dtype=np.float64, values=None) -> int:
    """-1 when perm is exactly std::stable_sort of raw/t (scan.hpp:37-40) in
    `dtype` arithmetic (and, if given, values == (raw/t)[perm] bitwise), else
    the first offending sorted position (len(raw) when perm is not a
    permutation).  O(m): see lxo_verify_sort."""
    raw = _arr(raw, dtype)
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    values = None if values is None else _arr(values, dtype)
    f = _fn("c", "verify_sort", dtype)
    f.argtypes = [C.c_void_p, C.c_size_t, _ctype(dtype), C.c_void_p, C.c_void_p]
    f.restype = C.c_int64
    return int(f(_p(raw), len(raw), t, _p(perm), _p(values)))


def coranks(sorted_rows, sorted_cols, dtype=np.float64):
    """(j_of_row, r_of_col) of two sorted anchor arrays: std::upper_bound
    per element (operator.hpp:111-120) as one merge walk each."""
    A, B = _arr(sorted_rows, dtype), _arr(sorted_cols, dtype)
    jr = np.empty(len(A), np.uint64)
    rc = np.empty(len(B), np.uint64)
    f = _fn("c", "coranks", dtype)
    f.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
    f(_p(A), len(A), _p(B), len(B), _p(jr), _p(rc))
    return jr, rc


def decay_scan(sorted_values, payload, dtype=np.float64, backend="c"):
    """prefix_decay_scan / suffix_decay_scan (scan.hpp:50-73) on sorted anchors."""
    v = _arr(sorted_values, dtype)
    p = _arr(payload, dtype)
    pre = np.empty(len(v), dtype)
    suf = np.empty(len(v), dtype)
    f = _fn(backend, "decay_scan", dtype)
    _check(f(_p(v), C.c_size_t(len(v)), _p(p), _p(pre), _p(suf)), "decay_scan")
    return pre, suf


def dense_matvec(a, b, t, x, phi=None, psi=None, dtype=np.float64):
    """oracle.hpp:86-93 (C restatement; no size cap -- keep n*k small)."""
    a, b, x = _arr(a, dtype), _arr(b, dtype), _arr(x, dtype)
    phi, psi = _arr(phi, dtype), _arr(psi, dtype)
    y = np.empty(len(a), dtype)
    f = _fn("c", "dense_matvec", dtype)
    f.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, _ctype(dtype), C.c_void_p,
                  C.c_void_p, C.c_void_p, C.c_void_p]
    f(_p(a), len(a), _p(b), len(b), t, _p(phi), _p(psi), _p(x), _p(y))
    return y


def dense_gram(a, b, t, D, phi=None, psi=None, dtype=np.float64):
    """oracle.hpp:96-121."""
    a, b, D = _arr(a, dtype), _arr(b, dtype), _arr(D, dtype)
    phi, psi = _arr(phi, dtype), _arr(psi, dtype)
    G = np.empty((len(a), len(a)), dtype)
    f = _fn("c", "dense_gram", dtype)
    f.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, _ctype(dtype), C.c_void_p,
                  C.c_void_p, C.c_void_p, C.c_void_p]
    f(_p(a), len(a), _p(b), len(b), t, _p(D), _p(phi), _p(psi), _p(G))
    return G


def map_rows(fn, items, workers=None):
    """[fn(item) for item in items] on a thread pool: each worker runs the
    oracle single-threaded (ctypes releases the GIL, so calls overlap).  For
    per-row oracle calls of a batch; results are identical to a serial loop."""
    import concurrent.futures as cf
    workers = workers or max(1, min(len(items), os.cpu_count() or 1))
    lib = _lib("c")

    def run(it):
        lib.lxo_set_num_threads(1)
        return fn(it)

    with cf.ThreadPoolExecutor(workers) as ex:
        return list(ex.map(run, items))


def rel_err_l2(got, want) -> float:
    """tests/helpers.hpp:27-35 (relative l2 in double, absolute when ||want|| = 0)."""
    got = np.asarray(got, np.float64).ravel()
    want = np.asarray(want, np.float64).ravel()
    num = float(np.sum((got - want) ** 2))
    den = float(np.sum(want ** 2))
    return float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num))


class Mt19937_64Uniform:
    """std::mt19937_64 + uniform_real_distribution<double> (libstdc++), the
    reference's input recipe (tests/helpers.hpp:12-24, laplex_bench.cpp:114-120).

    libstdc++'s generate_canonical<double,53> draws ONE 64-bit word and
    returns (w * 2^-64), clamped below 1; uniform(lo,hi) = lo + u*(hi-lo).
    numpy has no mt19937_64, so the generator is implemented here (vectorised
    per block of 312 words)."""

    NN, MM = 312, 156
    MATRIX_A = np.uint64(0xB5026F5AA96619E9)
    UM = np.uint64(0xFFFFFFFF80000000)
    LM = np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = np.zeros(self.NN, np.uint64)
        mt[0] = np.uint64(seed)
        with np.errstate(over="ignore"):
            for i in range(1, self.NN):
                prev = int(mt[i - 1])
                mt[i] = np.uint64((6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
        self.mt = mt
        self.idx = self.NN

    def _twist(self):
        mt = self.mt
        NN, MM = self.NN, self.MM
        for i in range(NN):
            x = (int(mt[i]) & 0xFFFFFFFF80000000) | (int(mt[(i + 1) % NN]) & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = np.uint64(int(mt[(i + MM) % NN]) ^ xa)
        self.idx = 0

    def words(self, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        o = 0
        while o < count:
            if self.idx >= self.NN:
                self._twist()
            take = min(self.NN - self.idx, count - o)
            y = self.mt[self.idx:self.idx + take].copy()
            y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
            y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
            y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
            y ^= y >> np.uint64(43)
            out[o:o + take] = y
            o += take
            self.idx += take
        return out

    def uniform(self, count: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        w = self.words(count).astype(np.float64) * (2.0 ** -64)
        w = np.where(w >= 1.0, np.nextafter(1.0, 0.0), w)
        return lo + w * (hi - lo)
