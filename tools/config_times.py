"""Device time of the other BASELINE configs (C2-C4) through DeviceOperator, CUDA events, median of 5
(diagnostics; the bench line is C5).  C2: fwd+bwd n=k=2^24, 64 rows.  C3: phased head n=1000 classes,
k=2^20 features, 256 rows, phased_matvec + phased VJP.  C4: Gram-vector A^T(A X) on n=k=3*2^20, 32 rows."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_24584_b200 as L

dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(3)


def U(*shape, lo=-1.0, hi=1.0):
    return torch.empty(*shape, device=dev).uniform_(lo, hi, generator=g)


def timeit(f, reps=5):
    ts = []
    for i in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


which = [w for w in sys.argv[1:] if not w.startswith("--")] or ["C2", "C3", "C4"]
if "C2" in which:
    n = k = 1 << 24
    B = 64
    a, b = U(n, lo=-100, hi=100), U(k, lo=-100, hi=100)
    X, G = U(B, k), U(B, n)

    def c2():
        op = L.DeviceOperator(a, b, 1.0)
        op.apply(X)
        op.backward(X, G)
    ms = timeit(c2)
    print(f"C2 fwd+bwd n=k=2^24 B=64 incl. plan: {ms:.2f} ms  {B * n / ms * 1e3:.3e} elem/s  "
          f"model 24.76 GB -> {24.76e9 / (ms / 1e3) / 1e9:.0f} GB/s")
if "C3" in which:
    n, k, B = 1000, 1 << 20, 256
    a, b = U(n, lo=-100, hi=100), U(k, lo=-100, hi=100)
    phi, psi = U(n, lo=0, hi=6.28), U(k, lo=0, hi=6.28)
    X, G = U(B, k), U(B, n)

    def c3():
        op = L.DeviceOperator(a, b, 1.0, phi, psi)
        op.apply(X)
        op.backward(X, G)
    ms = timeit(c3)
    print(f"C3 phased head n=1000 k=2^20 B=256 incl. plan: {ms:.2f} ms  {B * k / ms * 1e3:.3e} elem/s  "
          f"model 3.337 GB -> {3.337e9 / (ms / 1e3) / 1e9:.0f} GB/s")
if "C4" in which:
    n = k = 3 * (1 << 20)
    B = 32
    a, b = U(n, lo=-100, hi=100), U(k, lo=-100, hi=100)
    X = U(B, k)

    def c4():
        op = L.DeviceOperator(a, b, 1.0)
        z = op.apply(X)
        op.apply(z, transpose=True)
    ms = timeit(c4)
    print(f"C4 Gram-vector n=k=3*2^20 B=32 incl. plan: {ms:.2f} ms  {B * n / ms * 1e3:.3e} elem/s  "
          f"model 2.164 GB -> {2.164e9 / (ms / 1e3) / 1e9:.0f} GB/s")

if "--kernels" in sys.argv:
    import ctypes
    import json
    from paper_2605_24584_b200 import _lib
    lib = _lib.lib()
    lib.laplex_profile_enable(1)
    for f in [v for k_, v in list(globals().items()) if k_ in ("c2", "c3", "c4")]:
        f()
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.laplex_profile_dump(buf, len(buf))
    d = json.loads(buf.value.decode())
    for k_, v in sorted(d.items(), key=lambda kv: -kv[1]["ms"]):
        print("%-22s %4d %9.3f" % (k_, v["launches"], v["ms"]))
