#!/usr/bin/env python
"""LAPLEX fwd+bwd benchmark (BASELINE.json metric, config C5: n = k = 2^30, B = 1).

One step = plan build (scale by 1/t, device radix sort of both anchor sets,
merge-path partition) + forward y = A x + backward (x_bar, a_bar, b_bar) for a
synthetic cotangent g, all through the library's C-ABI device entry points,
inputs resident in HBM.  `value` is elements/s = n / step time (whole job:
sum over ranks).  `e2e` is the same step through the host-buffer C-ABI entry
points (host -> device copies and result read-back inside the timed region).

--impl reference times the reference's own CPU implementation (the UNMODIFIED
reference headers compiled by oracle/Makefile into oracle/_ref) on a bounded
sample of the same workload, on all host threads.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "elements/sec and % HBM roofline, LAPLEX fwd+bwd n=2^30, 1/2/4/8 B200 vs CPU ref"
UNIT = "elements/s"
SPEC_PEAK_GBS = 8000.0  # B200 HBM3e spec (report beside the measured copy peak)
REUSE_X, SAVE_X = 4, 8  # include/laplex_c.h flags

# BASELINE.json configs: shape, the timed work unit and
# what counts as an "element".
CONFIGS = {
    "C1": dict(n=1 << 20, k=1 << 20, B=1, kind="fwd", units="n",
               workload="C1 LAPLEX forward matvec incl. plan build, n=k=2^20, batch 1"),
    "C2": dict(n=1 << 24, k=1 << 24, B=64, kind="fwdbwd", units="Bn",
               workload="C2 LAPLEX fwd+bwd (x_bar, a_bar, b_bar) incl. plan build, n=k=2^24, batch 64"),
    "C3": dict(n=1000, k=1 << 20, B=256, kind="phased", units="Bk",
               workload="C3 phased LAPLEX head training step (phased_matvec + phased_matvec_vjp) incl. plan, "
                        "n=1000 classes, k=2^20 features, batch 256"),
    "C4": dict(n=3 << 20, k=3 << 20, B=32, kind="gram", units="Bn",
               workload="C4 Gram-vector A^T(A X) incl. plan build, n=k=3*1024*1024, batch 32"),
    "C5": dict(n=1 << 30, k=1 << 30, B=1, kind="fwdbwd", units="n",
               workload="C5 LAPLEX fwd+bwd incl. plan build, n=k=2^30, batch 1"),
}


def units_of(c):
    return {"n": c["n"], "Bn": c["B"] * c["n"], "Bk": c["B"] * c["k"]}[c["units"]]


# Algorithmic bytes of one step: fp32 values, u32 indices,
# 4-pass 8-bit LSD sort at 64 B per element per side, co-ranks 8 B per element
# per side, anchor metadata read once per step.
def step_model_bytes(c):
    n, k, B = c["n"], c["k"], c["B"]
    return {"fwd": 84 * n + 80 * k + B * (4 * n + 4 * k),
            "fwdbwd": 100 * n + 96 * k + B * (8 * n + 12 * k),
            "phased": 112 * n + 108 * k + B * (8 * n + 12 * k),
            "gram": 84 * n + 92 * k + B * (8 * n + 8 * k)}[c["kind"]]


STEP_MODEL_TEXT = {"fwd": "84n+80k+B(4n+4k)", "fwdbwd": "100n+96k+B(8n+12k)", "phased": "112n+108k+B(8n+12k)",
                   "gram": "84n+92k+B(8n+8k)"}


# Algorithmic bytes per kernel over one step (summed over its launches),
# what each kernel must read and write at minimum for its
# role in this pipeline (fp32 values, u32 indices, u16 store order).
def row_split(T, B, phased):
    """Row chunks of a batched main-kernel launch (launch_main_mb, lx_capi.cu): the chunk count
    minimising rounds of the resident CTA slots per chunk (phased kernels only; 148 SMs x 2 CTAs)."""
    slots = 148 * 2
    if not phased or B < 16 or T >= 4 * slots:
        return 1
    best, rc = math.ceil(T / slots), 1
    for c in range(2, 9):
        if c * 4 > B:
            break
        m = math.ceil(T * c / slots) / c
        if m < best - 1e-9:
            best, rc = m, c
    chunk = (B + rc - 1) // rc
    return (B + chunk - 1) // chunk


def kernel_model_bytes(name, c):
    n, k, B, kind = c["n"], c["k"], c["B"], c["kind"]
    m2 = n + k
    # sides permuted through the two-pass plans: larger than kDirectMax (2^22),
    # or any side above 2^16 in a batch whose rows x side exceeds 48 MB
    # (kBatchStageBytes, lx_capi.cu)
    def is_staged(m):
        return m > (1 << 22) or (B > 1 and m > (1 << 16) and B * m * 4 > (48 << 20))
    big = 0
    staged = [m for m in (n, k) if is_staged(m)]
    T = (m2 + 2047) // 2048
    ST = 6144  # radix-sort tile (lx_sort.cuh kTile: 256 threads x 24 keys)
    tiles = (n + ST - 1) // ST + (k + ST - 1) // ST
    phased = kind == "phased"
    # payload arrays per step, by side: (rows side element count, cols side)
    pay_rows = {"fwd": 0, "fwdbwd": B, "phased": B, "gram": B}[kind]  # g (bwd) / z (gram)
    out_rows = {"fwd": B, "fwdbwd": B + 1, "phased": B + 2, "gram": B}[kind]  # y, a_bar, phi_bar / z
    out_cols = {"fwd": 0, "fwdbwd": B + 1, "phased": B + 2, "gram": B}[kind]  # x_bar, b_bar, psi_bar / y
    ch = 2 if phased else 1
    model = {
        "lx_sort_hist": 4 * m2 + 2 * 4 * 256 * 4,         # keys once; 4 digit histograms per side
        "lx_sort_bases": 2 * 2 * 4 * 256 * 4,
        "lx_sort_count": 3 * 4 * m2 + 3 * tiles * 1024,  # passes 2-4: keys in, per-tile digit counts out
        "lx_sort_scan": 4 * tiles * 2048 + sum((m + ST - 1) // ST for m in staged) * 2048,
        "lx_sort_pass": (12 + 16 + 16 + 16) * m2,          # pass 1: r4 w8; passes 2-4: r8 w8
        "lx_splan_count": sum(4 * m + (m + ST - 1) // ST * 1024 for m in staged),
        "lx_splan": sum(12 * m for m in staged),            # perm in; pos (sequential), dst (bucket streams) out
        "lx_gather_sorted": 8 * m2 if phased else 0,        # phases into sorted order
        "cos_sin": 12 * m2 if phased else 0,
        "lx_partition": 4 * (T + 1),
        "lx_tiledesc": (T + 1) * 32,
        # output positions and anchors in; u16 store order and the merge words (4 B per 16 merged) out
        "lx_group_plan": 10 * m2 + T * 512,
        "lx_iota": 4 * n,
        # x once (the backward reuses the forward's sorted x), g in the backward
        "lx_perm_gather": 12 * ((B * k if is_staged(k) else 0) + ((B if kind in ("fwdbwd", "phased") else 0) * n
                                                                if is_staged(n) else 0)),
        "lx_gather_agg": 16 * (B * k + pay_rows * n) + 8 * m2 * (ch - 1),
        "lx_carry": 2 * 2 * 4 * ch * max(B, 1) * T * 4,
        # (+ the tile's merge words, 512 B per 2048 merged elements, T * 512)
        "lx_main_fwd": 4 * m2 + B * 4 * k + 6 * n + B * 4 * n + T * 512,
        "lx_main_fwd_phased": 4 * m2 + 16 * m2 + B * 4 * k + 6 * n + B * 4 * n + T * 512,
        "lx_main_trn": 4 * m2 + B * 4 * n + 6 * k + B * 4 * k + T * 512,
        "lx_main_bwd": 4 * m2 + B * (4 * n + 4 * k) + 6 * m2 + B * 4 * k + 4 * n + 4 * k + T * 512,
        "lx_main_bwd_phased": 4 * m2 + 16 * m2 + B * (4 * n + 4 * k) + 6 * m2 + B * 4 * k + 8 * n + 8 * k + T * 512,
        "lx_perm_scatter": 12 * ((out_rows * n if is_staged(n) else 0) + (out_cols * k if is_staged(k) else 0)),
        # row-split backward: per-chunk partial a_bar/b_bar (+ phi_bar/psi_bar) summed in chunk order
        "lx_chunk_sum": 4 * ch * m2 * (row_split(T, B, phased) + 1),
    }
    v = model.get(name)
    return v if v else None


def measured_traffic(kernel, cfg):
    """ncu DRAM bytes per launch of `kernel` for this config (profiles/*_traffic.json, written by
    tools/traffic_json.py from the committed launch list), or None."""
    import glob
    c = CONFIGS[cfg]
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")), reverse=True):
        try:
            d = json.load(open(path))
        except Exception:
            continue
        same = d.get("config") == cfg if "config" in d else (cfg == "C5" and d.get("log2n") == c["n"].bit_length() - 1)
        if same and kernel in d.get("kernels", {}):
            return d["kernels"][kernel]
    return None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled during the timed region by one
    `nvidia-smi -lms` process started before it (polling from inside this process, by
    fork + exec or by NVML, was measured to stall the enqueue thread: some runs showed
    20-60 ms/step of GPU idle).  Only samples taken inside the timed window count."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, interval=1.0):
        self.index = index
        self.interval = interval
        self.samples = []
        self._p = None
        self._t0 = self._t1 = None
        self._lines = []
        self._first = threading.Event()
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                                        "--format=csv,noheader,nounits", "-lms", str(int(interval * 1000))],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self._p = None

    def _read(self):
        for line in self._p.stdout:
            self._lines.append(line)
            self._first.set()

    def __enter__(self):
        # nvidia-smi's start-up (driver / NVML initialisation) must not overlap the
        # timed window: wait for its first sample
        self._first.wait(timeout=30)
        self._t0 = time.time()
        return self

    def __exit__(self, *a):
        self._t1 = time.time()
        if self._p is None:
            return
        time.sleep(min(2.0, self.interval + 0.2))  # let the sample covering the window's end arrive
        self._p.terminate()
        try:
            self._p.wait(timeout=10)
        except Exception:
            self._p.kill()
        import datetime
        for line in list(self._lines):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                continue
            if self._t0 - 0.05 <= ts <= self._t1 + 0.05:
                self.samples.append(f[1:])

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# reference CPU arm / cpu_baseline (BASELINE.md section 3 protocol)
# ---------------------------------------------------------------------------
# Each config's reference call sequence runs on a
# bounded sample: ctor, then the per-row work of `rows_s` rows, each piece timed
# separately (2 warm-ups + 5 trials, median).  Sizes above the sample are
# extrapolated: the ctor (two std::stable_sorts) and the VJP (which re-sorts in
# matvec_transpose) by n log n, matvec / batch_matvec by n; rows by B / rows_s.
# Row-parallel pieces (the API is thread-safe, operator.hpp:266-272) run one
# row per thread when threads > 1; the ctor of one operator is single-threaded.
REF_SAMPLE = {  # sample n, k (log2 or exact) per config
    "C1": (1 << 20, 1 << 20), "C2": (1 << 20, 1 << 20), "C3": (1000, 1 << 20), "C4": (1 << 20, 1 << 20),
    "C5": (1 << 21, 1 << 21)}


def _nlogn(m):
    import math
    return m * math.log2(max(m, 2))


def host_cpu():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count() or 1


def reference_pieces(cfg_name, threads, seed=42):
    """One timed sample of the config's reference call sequence.  Returns
    {piece: seconds} for: ctor, (transposed), fwd (rows_s rows), bwd (rows_s rows)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle as O

    c = CONFIGS[cfg_name]
    ns, ks = REF_SAMPLE[cfg_name]
    rows_s = threads if c["B"] > 1 else 1
    lib = O._lib("ref")
    buf = np.empty(2 * (ns + ks) + 2 * rows_s * (ns + ks))
    lib.lxr_mt_uniform(C.c_uint64(seed), C.c_size_t(len(buf)), C.c_double(-1.0), C.c_double(1.0),
                       buf.ctypes.data_as(C.c_void_p))
    o = 0

    def take(m, scale=1.0, shift=0.0):
        nonlocal o
        v = (buf[o:o + m] * scale + shift).astype(np.float32)
        o += m
        return v
    a, b = take(ns, 100), take(ks, 100)
    X = [take(ks) for _ in range(rows_s)]
    G = [take(ns) for _ in range(rows_s)]
    phi = psi = None
    if c["kind"] == "phased":
        phi, psi = take(ns, 3.14, 3.14), take(ks, 3.14, 3.14)
    out = {}
    t0 = time.perf_counter()
    op = O.OracleOp(a, b, 1.0, phi, psi, dtype=np.float32, backend="ref")
    out["ctor"] = time.perf_counter() - t0
    opT = None
    if c["kind"] == "gram":  # build op.transposed() once
        t0 = time.perf_counter()
        opT = op.transposed()
        out["transposed"] = time.perf_counter() - t0

    def wave(fn):
        res = [None] * rows_s
        ths = [threading.Thread(target=lambda r=r: res.__setitem__(r, fn(r))) for r in range(rows_s)]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return time.perf_counter() - t0, res
    kind = c["kind"]
    if kind in ("fwd", "fwdbwd"):
        out["fwd"], _ = wave(lambda r: op.matvec(X[r]))
        if kind == "fwdbwd":
            out["bwd"], _ = wave(lambda r: op.vjp(X[r], G[r]))
    elif kind == "phased":
        out["fwd"], _ = wave(lambda r: op.phased_matvec(X[r]))
        out["bwd"], _ = wave(lambda r: op.phased_vjp(X[r], G[r]))
    else:
        out["fwd"], Z = wave(lambda r: op.batch_matvec(X[r][None, :]))
        out["bwd"], _ = wave(lambda r: opT.batch_matvec(Z[r]))
    return out, rows_s


def reference_step_seconds(cfg_name, pieces, rows_s):
    """Extrapolate one sample's piece times to the config's full step."""
    c = CONFIGS[cfg_name]
    ns, ks = REF_SAMPLE[cfg_name]
    f_sort = (_nlogn(c["n"]) + _nlogn(c["k"])) / (_nlogn(ns) + _nlogn(ks))
    f_lin = (c["n"] + c["k"]) / (ns + ks)
    f_rows = c["B"] / rows_s
    kind = c["kind"]
    total = pieces["ctor"] * f_sort + pieces.get("transposed", 0.0) * f_sort
    total += pieces["fwd"] * f_lin * f_rows
    if "bwd" in pieces:  # VJPs re-sort (matvec_transpose, gradients.hpp:118); the Gram half is a batch_matvec
        total += pieces["bwd"] * (f_lin if kind == "gram" else f_sort) * f_rows
    return total


def reference_measure(cfg_name, threads, warmups, trials):
    for i in range(warmups):
        reference_pieces(cfg_name, threads, seed=7 + i)
    runs = [reference_pieces(cfg_name, threads, seed=42 + i) for i in range(trials)]
    rows_s = runs[0][1]
    med = {p: statistics.median(r[0][p] for r in runs) for p in runs[0][0]}
    return med, rows_s, reference_step_seconds(cfg_name, med, rows_s)


def reference_sample_text(cfg_name, med, rows_s, threads, warmups, trials):
    c = CONFIGS[cfg_name]
    ns, ks = REF_SAMPLE[cfg_name]
    model, nproc = host_cpu()
    pieces = ", ".join(f"{p} {1000 * v:.1f} ms" for p, v in med.items())
    extra = "" if (ns, ks) == (c["n"], c["k"]) else (
        f"; sampled at n={ns}, k={ks} and extrapolated to n={c['n']}, k={c['k']} (ctor and VJP by n log n, "
        f"matvec by n)")
    return (f"unmodified reference (proj/include headers compiled -O3 -DNDEBUG into oracle/_ref), fp32, "
            f"BASELINE.md section 3 call sequence for {cfg_name}; {warmups} warm-ups + {trials} trials, median "
            f"per piece ({pieces}); {rows_s} of {c['B']} rows timed, {threads} thread(s) (one row per thread), "
            f"rows extrapolated by B/{rows_s}{extra}; host: {model}, nproc {nproc}")


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = args.config
    c = CONFIGS[cfg]
    # all host threads the library can use: rows run concurrently on a shared
    # operator; one vector (B = 1) is single-threaded in the reference
    threads = max(1, min(os.cpu_count() or 1, args.ref_threads, c["B"]))
    for i in range(args.warmup):
        reference_pieces(cfg, threads, seed=7 + i)
    steps = []
    meds = []
    for i in range(args.steps):
        pieces, rows_s = reference_pieces(cfg, threads, seed=42 + i)
        steps.append(reference_step_seconds(cfg, pieces, rows_s))
        meds.append(pieces)
    sec = statistics.median(steps)
    med = {p: statistics.median(m[p] for m in meds) for p in meds[0]}
    value = units_of(c) / sec
    sample = reference_sample_text(cfg, med, rows_s, threads, args.warmup, args.steps)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sec, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (mt19937_64 recipe)",
        "config": {"workload": c["workload"], "n": c["n"], "k": c["k"], "batch": c["B"],
                   "parallelism": f"cpu, {threads} thread(s)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline(args):
    """Rank 0, N = 1: the compiled reference on one core, bounded sample of the config."""
    cfg = args.config
    med, rows_s, sec = reference_measure(cfg, 1, 2, args.ref_trials)
    return {"value": units_of(CONFIGS[cfg]) / sec, "unit": UNIT, "cores": 1, "kind": "reference",
            "seconds_per_step": sec,
            "sample": reference_sample_text(cfg, med, rows_s, 1, 2, args.ref_trials)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def make_inputs(torch, c, dev, seed):
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    n, k, B = c["n"], c["k"], c["B"]
    u = lambda shape, lo, hi: torch.empty(shape, device=dev).uniform_(lo, hi, generator=gen)  # noqa: E731
    t = dict(a=u(n, -100, 100), b=u(k, -100, 100), X=u((B, k), -1, 1))
    if c["kind"] in ("fwdbwd", "phased"):
        t["G"] = u((B, n), -1, 1)
    if c["kind"] == "phased":
        t["phi"], t["psi"] = u(n, 0, 6.28), u(k, 0, 6.28)
    return t


def make_step(L, torch, c, t):
    """One step of the config through the device C-ABI (DeviceOperator)."""
    n, k, B, kind = c["n"], c["k"], c["B"], c["kind"]
    dev = t["a"].device
    o = dict(Y=torch.empty((B, k if kind == "gram" else n), device=dev))
    if kind in ("fwdbwd", "phased"):
        o.update(xb=torch.empty((B, k), device=dev), ab=torch.empty(n, device=dev), bb=torch.empty(k, device=dev))
    if kind == "phased":
        o.update(pb=torch.empty(n, device=dev), qb=torch.empty(k, device=dev))

    def step():
        # a training loop's plan: no host synchronisation at creation; the
        # finiteness errors are checked once per step, after its work is queued
        if kind == "phased":
            op = L.DeviceOperator(t["a"], t["b"], 1.0, t["phi"], t["psi"], sync=False)
        else:
            op = L.DeviceOperator(t["a"], t["b"], 1.0, sync=False)
        if kind == "gram":
            op.gram_apply(t["X"], out=o["Y"])
            op.check()
            return op
        # a training step: the forward saves its sorted x for the backward (LAPLEX_SAVE_X / REUSE_X)
        op.apply(t["X"], out=o["Y"], save_x=kind != "fwd")
        if kind == "fwdbwd":
            op.backward(t["X"], t["G"], x_bar=o["xb"], a_bar=o["ab"], b_bar=o["bb"], reuse_x=True)
        elif kind == "phased":
            op.backward(t["X"], t["G"], x_bar=o["xb"], a_bar=o["ab"], b_bar=o["bb"], phi_bar=o["pb"],
                        psi_bar=o["qb"], reuse_x=True)
        op.check()
        return op
    return step, o


def run_ours(args, rank, world, dist):
    import torch

    import paper_2605_24584_b200 as L
    from paper_2605_24584_b200 import _lib

    lib = _lib.lib()
    cfg = args.config
    c = CONFIGS[cfg]
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n, k, B = c["n"], c["k"], c["B"]
    t = make_inputs(torch, c, dev, 42 + rank)
    step, outs = make_step(L, torch, c, t)
    stream = torch.cuda.current_stream()
    in_bytes = sum(v.numel() * v.element_size() for v in t.values())
    flush = in_bytes < (512 << 20)  # working set near the 126 MB L2: flush between timed steps
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local, args.clock_interval)  # started before the warm-up steps
    for _ in range(args.warmup):
        step()
    barrier()
    launches0 = L.kernel_launches()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps if flush else 1)]
    with sampler as clk:
        barrier()
        if flush:  # per-step events; the L2 scrub between steps is outside them
            for e0, e1 in evs:
                scrub.zero_()
                e0.record(stream)
                step()
                e1.record(stream)
        else:
            evs[0][0].record(stream)
            for _ in range(args.steps):
                step()
            evs[0][1].record(stream)
        barrier()
    launches = L.kernel_launches() - launches0
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps
    if dist is not None:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    check = {}
    if "ab" in outs:  # translation conservation sum(a_bar) + sum(b_bar) ~ 0 (unphased)
        ab, bb = outs["ab"], outs["bb"]
        if c["kind"] == "fwdbwd":
            check["conservation_rel"] = float((ab.double().sum() + bb.double().sum()).abs() /
                                              (ab.double().abs().sum() + bb.double().abs().sum()))

    # per-kernel CUDA-event timing over extra (untimed) steps
    lib.laplex_profile_enable(1)
    prof_steps = 2
    for _ in range(prof_steps):
        if flush:
            scrub.zero_()
        step()
    torch.cuda.synchronize()
    buf = C.create_string_buffer(1 << 16)
    lib.laplex_profile_dump(buf, len(buf))
    lib.laplex_profile_enable(0)
    prof = json.loads(buf.value.decode())
    for v in prof.values():
        v["ms"] /= prof_steps
        v["launches"] //= prof_steps
    hbm, peak_kind = peaks()
    roof = None
    kern_table = {}
    for name, v in prof.items():
        mb = kernel_model_bytes(name, c)
        gbs = mb / (v["ms"] / 1000) / 1e9 if mb else None
        kern_table[name] = {"ms_per_step": round(v["ms"], 4), "launches_per_step": v["launches"],
                            "model_bytes": mb, "achieved_gbs": round(gbs, 1) if gbs else None,
                            "frac": round(gbs / hbm, 4) if gbs else None,
                            "frac_spec": round(gbs / SPEC_PEAK_GBS, 4) if gbs else None}
    dom = max(prof.items(), key=lambda kv: kv[1]["ms"])[0] if prof else None
    if dom:
        d = kern_table[dom]
        per_launch_bytes = d["model_bytes"] / max(1, d["launches_per_step"]) if d["model_bytes"] else None
        roof = {"bound": "hbm", "kernel": dom, "achieved": d["achieved_gbs"], "peak": hbm, "unit": "GB/s",
                "frac": d["frac"], "traffic": measured_traffic(dom, cfg), "peak_kind": peak_kind,
                "frac_spec": d["frac_spec"], "spec_peak": SPEC_PEAK_GBS,
                "bytes_per_launch": per_launch_bytes,
                "avg_launch_ms": d["ms_per_step"] / max(1, d["launches_per_step"])}

    value = units_of(c) * world / (ms / 1000)
    step_bytes = step_model_bytes(c)
    step_gbs = step_bytes / (ms / 1000) / 1e9

    e2e = None
    if args.e2e and rank == 0:
        # the host-pointer path runs on its own: the device-path inputs, outputs
        # and torch's cached blocks (~8 arrays of the config's size) are freed
        # first, as in a process that only uses the host API
        del step, outs, t, scrub
        ab = bb = None  # noqa: F841 (the conservation check's references)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        e2e = run_e2e(args, torch, lib, c)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: anchors U(-100,100), x and g U(-1,1), phases U(0,6.28), t=1 "
                    "(torch.Generator seed 42+rank)",
            "config": {"workload": c["workload"], "name": cfg, "n": n, "k": k, "batch": B, "temperature": 1.0,
                       "elements": f"{c['units']} = {units_of(c)} per step",
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": ("inputs smaller than L2 scale: a 256 MB buffer is written between timed steps "
                              "(outside the per-step events)") if flush else
                             "inputs larger than the 126 MB L2; no flush needed"},
            "gpu_launches": launches,
            "roofline": roof,
            "step_roofline": {"model": f"SURVEY 8(d) {c['kind']} incl. plan: {STEP_MODEL_TEXT[c['kind']]} bytes",
                              "bytes": step_bytes, "achieved": round(step_gbs, 1), "peak": hbm, "unit": "GB/s",
                              "frac": round(step_gbs / hbm, 4), "frac_spec": round(step_gbs / SPEC_PEAK_GBS, 4)},
            "kernels": kern_table,
            "check": check,
            "clocks": clk.summary(),
            "e2e": e2e,
        }
        if world == 1 and args.cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(line), flush=True)


def run_sharded(args, rank, world, dist, comm_factory):
    """N > 1, C5: one long vector (n = k = 2^log2n in total) range-sharded over
    the ranks by the library's C++ host layer (laplex_sharded_*); each rank
    starts from its contiguous slice of a, b, x, g.  comm_factory() -> Comm."""
    import torch

    import paper_2605_24584_b200 as L
    from paper_2605_24584_b200.sharded import CppShardedOperator

    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not args.sim:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", torch.cuda.current_device())
    c = CONFIGS[args.config]
    n, k = c["n"], c["k"]
    nl, kl = n // world, k // world
    gen = torch.Generator(device=dev)
    gen.manual_seed(42 + rank)
    a = torch.empty(nl, device=dev).uniform_(-100, 100, generator=gen)
    b = torch.empty(kl, device=dev).uniform_(-100, 100, generator=gen)
    x = torch.empty(1, kl, device=dev).uniform_(-1, 1, generator=gen)
    g = torch.empty(1, nl, device=dev).uniform_(-1, 1, generator=gen)
    comm = comm_factory()
    stream = torch.cuda.Stream() if args.sim else torch.cuda.current_stream()

    def step():
        op = CppShardedOperator(a, b, 1.0, comm, stream=stream)
        y = op.apply(x, stream=stream)
        xb, ab, bb = op.backward(x, g, reuse_x=True, stream=stream)
        return op, (y, xb, ab, bb)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        elif args.sim:
            args.sim_barrier.wait()
        torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        sampler = ClockSampler(local if not args.sim else 0, args.clock_interval)  # before the warm-up
        for _ in range(args.warmup):
            step()
        barrier()
        launches0 = L.kernel_launches()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with sampler as clk:
            barrier()
            ev0.record(stream)
            for _ in range(args.steps):
                _, outs = step()
            ev1.record(stream)
            barrier()
        ms = ev0.elapsed_time(ev1) / args.steps
    if dist is not None:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    elif args.sim:
        args.sim_ms[rank] = ms
        args.sim_barrier.wait()
        ms = max(args.sim_ms)
    launches = L.kernel_launches() - launches0
    y, xb, ab, bb = outs
    part = torch.stack([ab.double().sum() + bb.double().sum(), ab.double().abs().sum() + bb.double().abs().sum()])
    if dist is not None:
        dist.all_reduce(part)
    cons = float(part[0].abs() / part[1]) if not args.sim else None
    if rank == 0:
        hbm, peak_kind = peaks()
        step_bytes = step_model_bytes(c)
        print(json.dumps({
            "metric": METRIC, "value": n / (ms / 1000), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: anchors U(-100,100), x and g U(-1,1), t=1; rank r holds the r-th contiguous slice",
            "config": {"workload": f"{c['workload']} [total, range-sharded]", "name": args.config,
                       "n": n, "k": k, "batch": 1, "temperature": 1.0,
                       "parallelism": f"range-sharded x{world}: value splitters + all-to-all (a, b, x, g, outputs) "
                                      f"+ all-gather of shard totals folded on the device (C++ laplex_sharded_*, "
                                      f"NCCL)" + (" [SIMULATED: local ranks on one GPU]" if args.sim else ""),
                       "l2": "inputs larger than L2"},
            "gpu_launches": launches,
            "roofline": None,
            "step_roofline": {"model": "SURVEY 8(d) fwd+bwd incl. plan: 100n+96k+8n+12k bytes (whole job)",
                              "bytes": step_bytes, "achieved": round(step_bytes / (ms / 1000) / 1e9, 1),
                              "peak": hbm * world, "unit": "GB/s",
                              "frac": round(step_bytes / (ms / 1000) / 1e9 / (hbm * world), 4)},
            "check": {"conservation_rel": cons},
            "clocks": clk.summary(),
            "e2e": None,
        }), flush=True)


def run_replicas(args, rank, world, dist, comm):
    """N > 1, batch configs (C2-C4): global batch B split over the ranks, the
    plan replicated on each; the anchor cotangents all-gathered and summed in
    rank order (laplex_replica_backward_dev).  Strong scaling."""
    import torch

    import paper_2605_24584_b200 as L
    from paper_2605_24584_b200.sharded import replica_backward

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    c = dict(CONFIGS[args.config])
    B = c["B"]
    rows = B // world + (1 if rank < B % world else 0)
    t = make_inputs(torch, dict(c, B=rows), dev, 42 + rank)
    gen = torch.Generator(device=dev)
    gen.manual_seed(42)  # identical anchors on every rank
    t["a"] = torch.empty(c["n"], device=dev).uniform_(-100, 100, generator=gen)
    t["b"] = torch.empty(c["k"], device=dev).uniform_(-100, 100, generator=gen)
    if c["kind"] == "phased":
        t["phi"] = torch.empty(c["n"], device=dev).uniform_(0, 6.28, generator=gen)
        t["psi"] = torch.empty(c["k"], device=dev).uniform_(0, 6.28, generator=gen)
    Y = torch.empty((rows, c["k"] if c["kind"] == "gram" else c["n"]), device=dev)

    def step():
        ph = c["kind"] == "phased"
        op = L.DeviceOperator(t["a"], t["b"], 1.0, t.get("phi") if ph else None, t.get("psi") if ph else None)
        if c["kind"] == "gram":
            op.gram_apply(t["X"], out=Y)
            return op
        op.apply(t["X"], out=Y)
        if c["kind"] != "fwd":
            replica_backward(op, comm, t["X"], t["G"])
        return op

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = L.kernel_launches()
    sampler = ClockSampler(local, args.clock_interval)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler as clk:
        torch.cuda.synchronize()
        dist.barrier()
        ev0.record()
        for _ in range(args.steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    tt = torch.tensor([ms], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    if rank == 0:
        hbm, _ = peaks()
        step_bytes = step_model_bytes(c)
        print(json.dumps({
            "metric": METRIC, "value": units_of(c) / (ms / 1000), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": c["workload"], "name": args.config, "n": c["n"], "k": c["k"], "batch": B,
                       "parallelism": f"batch replicas x{world}: rows split, plan replicated, anchor cotangents "
                                      f"all-gathered and summed in rank order"},
            "gpu_launches": L.kernel_launches() - launches0,
            "roofline": None,
            "step_roofline": {"model": f"SURVEY 8(d) {c['kind']} incl. plan (whole job)", "bytes": step_bytes,
                              "achieved": round(step_bytes / (ms / 1000) / 1e9, 1), "peak": hbm * world,
                              "unit": "GB/s", "frac": round(step_bytes / (ms / 1000) / 1e9 / (hbm * world), 4)},
            "clocks": clk.summary(),
            "e2e": None,
        }), flush=True)


def run_e2e(args, torch, lib, c):
    """The same step through the host-buffer C-ABI (the reference-facing
    entry points): pinned host inputs in, host outputs out, copies inside."""
    import paper_2605_24584_b200 as L  # noqa: F401
    n, k, B, kind = c["n"], c["k"], c["B"], c["kind"]
    pin = dict(dtype=torch.float32, pin_memory=True)
    gen = torch.Generator()
    gen.manual_seed(7)
    h = dict(a=torch.empty(n, **pin).uniform_(-100, 100, generator=gen),
             b=torch.empty(k, **pin).uniform_(-100, 100, generator=gen),
             X=torch.empty((B, k), **pin).uniform_(-1, 1, generator=gen))
    if kind in ("fwdbwd", "phased"):
        h["G"] = torch.empty((B, n), **pin).uniform_(-1, 1, generator=gen)
    if kind == "phased":
        h["phi"] = torch.empty(n, **pin).uniform_(0, 6.28, generator=gen)
        h["psi"] = torch.empty(k, **pin).uniform_(0, 6.28, generator=gen)
    o = dict(Y=torch.empty((B, k if kind == "gram" else n), **pin))
    if kind in ("fwdbwd", "phased"):
        o.update(xb=torch.empty((B, k), **pin), ab=torch.empty(n, **pin), bb=torch.empty(k, **pin))
    if kind == "phased":
        o.update(pb=torch.empty(n, **pin), qb=torch.empty(k, **pin))
    P = lambda key: o[key].data_ptr() if key in o else None  # noqa: E731
    flags = 2 if kind == "phased" else 0

    def step():
        hp = C.c_void_p()
        rc = lib.laplex_plan_create(0, h["a"].data_ptr(), n, h["b"].data_ptr(), k, 1.0,
                                    h["phi"].data_ptr() if "phi" in h else None,
                                    h["psi"].data_ptr() if "psi" in h else None, C.byref(hp))
        assert rc == 0, lib.laplex_last_error()
        if kind == "gram":
            rc = lib.laplex_gram_apply(hp, h["X"].data_ptr(), B, k, o["Y"].data_ptr())
            assert rc == 0, lib.laplex_last_error()
        else:
            # fwd+bwd: the apply keeps its sorted x (LAPLEX_SAVE_X) and the
            # backward of the same host X reuses it (LAPLEX_REUSE_X): x crosses
            # PCIe once; results are bitwise those of separate calls
            fb = kind != "fwd"
            rc = lib.laplex_apply(hp, flags | (SAVE_X if fb else 0), h["X"].data_ptr(), B, k, o["Y"].data_ptr())
            assert rc == 0, lib.laplex_last_error()
            if fb:
                rc = lib.laplex_backward(hp, flags | REUSE_X, h["X"].data_ptr(), B, k, h["G"].data_ptr(), n,
                                         P("xb"), P("ab"), P("bb"), P("pb"), P("qb"))
                assert rc == 0, lib.laplex_last_error()
        lib.laplex_plan_release(hp)

    step()
    times = []
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    sec = statistics.median(times)
    # bytes crossing PCIe per step: every input once per call that takes it
    uploads = {"fwd": ["a", "b", "X"], "fwdbwd": ["a", "b", "X", "G"],
               "phased": ["a", "b", "phi", "psi", "X", "G"], "gram": ["a", "b", "X"]}[kind]
    h2d = sum(h[key].numel() * 4 for key in uploads)
    d2h = sum(v.numel() * 4 for v in o.values())
    calls = {"fwd": "laplex_plan_create + laplex_apply", "fwdbwd": "laplex_plan_create + laplex_apply(SAVE_X) + "
             "laplex_backward(REUSE_X)", "phased": "laplex_plan_create(phases) + laplex_apply(PHASED|SAVE_X) + "
             "laplex_backward(PHASED|REUSE_X)", "gram": "laplex_plan_create + laplex_gram_apply"}[kind]
    return {"value": units_of(c) / sec, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": 1000 * sec,
            "path": f"{calls} (host pointers, pinned torch buffers; inputs checked for finiteness in the "
                    f"reference's order), median of {args.e2e_steps} steps"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS),
                    help="BASELINE.json config (C5, the metric's own config, by default)")
    ap.add_argument("--log2n", type=int, default=None, help="override n = k = 2^log2n (C5 / C2 shapes)")
    ap.add_argument("--ref-trials", type=int, default=5)
    ap.add_argument("--ref-threads", type=int, default=64)
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--sim", type=int, default=0,
                    help="simulate N range shards with threads on one GPU (functional check only)")
    ap.add_argument("--clock-interval", type=float, default=1.0,
                    help="seconds between nvidia-smi samples during the timed region")
    args = ap.parse_args()
    if args.log2n is not None:
        CONFIGS[args.config] = dict(CONFIGS[args.config], n=1 << args.log2n, k=1 << args.log2n)
        CONFIGS[args.config]["workload"] += f" [resized: n=k=2^{args.log2n}]"
        if args.config in ("C5", "C2"):
            REF_SAMPLE[args.config] = tuple(min(v, 1 << 21) for v in REF_SAMPLE[args.config])
    args.log2n = (CONFIGS[args.config]["n"]).bit_length() - 1

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.sim > 1:  # N range shards as threads on one GPU (functional path check, C5 shape)
        from paper_2605_24584_b200.sharded import Comm
        args.sim_barrier = threading.Barrier(args.sim)
        args.sim_ms = [0.0] * args.sim
        key = int(time.time() * 1e6)
        ths = [threading.Thread(target=run_sharded, args=(args, r, args.sim, None,
                                                          lambda r=r: Comm.local(key, args.sim, r)))
               for r in range(args.sim)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return
    if world > 1:
        import torch
        import torch.distributed as tdist
        from paper_2605_24584_b200.sharded import Comm
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        tdist.init_process_group("nccl")

        def bcast(uid):
            box = [uid]
            tdist.broadcast_object_list(box, src=0)
            return box[0]
        comm = Comm.nccl(world, rank, bcast)
        if CONFIGS[args.config]["B"] == 1:
            run_sharded(args, rank, world, tdist, lambda: comm)
        else:
            run_replicas(args, rank, world, tdist, comm)
        del comm
        tdist.destroy_process_group()
        return
    run_ours(args, rank, world, None)


if __name__ == "__main__":
    main()
