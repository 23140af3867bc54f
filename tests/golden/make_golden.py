"""Generate tests/golden/*.npz from the UNMODIFIED reference.

Runs in the dev container only (needs oracle/_ref/libref_laplex.so, which
oracle/Makefile compiles from /root/reference/proj/include).  The fixtures are
small and committed; tests on the GPU box read them without the reference.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402


def mt(seed, n, lo=-1.0, hi=1.0):
    """std::mt19937_64 + uniform_real_distribution (tests/helpers.hpp:12-24)."""
    return O.Mt19937_64Uniform(seed).uniform(n, lo, hi)


def sort_cases():
    cases = {}
    raws = {
        "ref_test_scan": np.array([3.0, -1.0, 2.0, -1.0]),            # tests/test_scan.cpp:11
        "spec_swap": np.array([1.0, 0.0]),
        "spec_stable_tie": np.array([0.0, 0.0, -1.0]),
        "signed_zero": np.array([0.0, -0.0, 1.0, -0.0, 0.0]),         # SURVEY 8(c) probe
        "singleton": np.array([3.0]),
    }
    g = mt(901, 5000, -3, 3)
    g[::11] = g[1::7][: len(g[::11])]  # planted duplicates
    raws["random_ties_5000"] = g
    raws["tile_edge_4097"] = np.round(mt(902, 4097, -50, 50), 1)  # heavy ties across a sort tile
    for name, raw in raws.items():
        for dt in (np.float64, np.float32):
            r = raw.astype(dt)
            v, p, d = O.sort_anchors(r, dtype=dt, backend="ref")
            cases[f"{name}_{np.dtype(dt).name}"] = dict(raw=r, values=v, perm=p, decays=d)
    return cases


def operator_cases():
    cases = {}
    seed = 1000
    specs = [
        # (n, k, span, t, ties, phased)
        (1, 1, 1.0, 1.0, False, False),
        (2, 1, 1.0, 1.0, False, False),
        (7, 13, 5.0, 1.0, True, False),
        (13, 7, 5.0, 0.37, True, False),
        (64, 96, 5.0, 0.42, True, False),
        (96, 64, 2.0, 1.0, False, False),
        (160, 120, 8.0, 0.73, True, False),
        (40, 55, 10.0, 1.1, False, True),
        (9, 14, 3.0, 0.8, True, True),
    ]
    for (n, k, span, t, ties, phased) in specs:
        seed += 1
        a = mt(seed, n, -span, span)
        b = mt(seed + 500, k, -span, span)
        if ties:
            m = min(n, k) // 2 + 1
            idx_a = (mt(seed + 700, m, 0, 1) * n).astype(int) % n
            idx_b = (mt(seed + 800, m, 0, 1) * k).astype(int) % k
            b[idx_b] = a[idx_a]
        x = mt(seed + 900, k)
        gv = mt(seed + 950, n)
        X = mt(seed + 960, 3 * k).reshape(3, k)
        D = mt(seed + 970, k, -2, 2)
        phi = mt(seed + 980, n, 0, 6.28) if phased else None
        psi = mt(seed + 990, k, 0, 6.28) if phased else None
        for dt in (np.float64, np.float32):
            name = f"op_n{n}_k{k}_t{t}_{'ph' if phased else 'pl'}_{np.dtype(dt).name}"
            cast = lambda v: None if v is None else np.asarray(v, dt)  # noqa: E731
            op = O.OracleOp(cast(a), cast(b), t, cast(phi), cast(psi), dtype=dt, backend="ref")
            rec = dict(a=cast(a), b=cast(b), t=np.array(t), x=cast(x), g=cast(gv), X=cast(X), D=cast(D))
            rv, rp, rd = op.sorted(0)
            cv, cp, cd = op.sorted(1)
            rec.update(rows_values=rv, rows_perm=rp, rows_decays=rd, cols_values=cv, cols_perm=cp,
                       cols_decays=cd, j_of_row=op.ranks(0), r_of_col=op.ranks(1))
            if phased:
                rec.update(phi=cast(phi), psi=cast(psi))
                rec["phased_matvec"] = op.phased_matvec(cast(x))
                xb, ab, bb, pb, qb = op.phased_vjp(cast(x), cast(gv))
                rec.update(pvjp_x_bar=xb, pvjp_a_bar=ab, pvjp_b_bar=bb, pvjp_phi_bar=pb, pvjp_psi_bar=qb)
                rec["phased_gram"] = op.phased_gram(cast(D))
            else:
                rec["matvec_A"] = op.matvec(cast(x), 1)
                rec["matvec_B"] = op.matvec(cast(x), 2)
                rec["matvec_transpose"] = op.matvec_transpose(cast(gv))
                rec["batch_matvec"] = op.batch_matvec(cast(X))
                xb, ab, bb = op.vjp(cast(x), cast(gv))
                rec.update(vjp_x_bar=xb, vjp_a_bar=ab, vjp_b_bar=bb)
                rec["weighted_gram"] = op.weighted_gram(cast(D))
                Gb = mt(seed + 999, n * n).reshape(n, n)
                Gb = np.tril(Gb) + np.tril(Gb, -1).T
                rec["G_bar"] = cast(Gb)
                rec["gram_vjp_weights"] = op.gram_vjp_weights(cast(D), cast(Gb))
            cases[name] = rec
    return cases


def scan_cases():
    cases = {}
    for m, seed in ((1, 11), (2, 12), (64, 13), (5000, 14)):
        for dt in (np.float64, np.float32):
            raw = mt(seed, m, -3, 3).astype(dt)
            v, _, _ = O.sort_anchors(raw, dtype=dt, backend="ref")
            p = mt(seed + 100, m).astype(dt)
            pre, suf = O.decay_scan(v, p, dtype=dt, backend="ref")
            cases[f"scan_m{m}_{np.dtype(dt).name}"] = dict(values=v, payload=p, prefix=pre, suffix=suf)
    return cases


def main():
    if not O.available("ref"):
        sys.exit("oracle/_ref/libref_laplex.so missing: run `make -C oracle ref` (needs /root/reference)")
    for fname, cases in (("sort.npz", sort_cases()), ("operator.npz", operator_cases()),
                         ("scan.npz", scan_cases())):
        flat = {f"{c}::{k}": v for c, rec in cases.items() for k, v in rec.items() if v is not None}
        np.savez_compressed(os.path.join(HERE, fname), **flat)
        print(fname, len(cases), "cases")


if __name__ == "__main__":
    main()
