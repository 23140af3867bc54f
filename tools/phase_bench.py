"""Diagnostics: CUDA-event time of each API phase of the C5 step (not a bench line)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2605_24584_b200 as L

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
N = 1 << lg
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(1)
a = torch.empty(N, device=dev).uniform_(-100, 100, generator=g)
b = torch.empty(N, device=dev).uniform_(-100, 100, generator=g)
x = torch.empty(1, N, device=dev).uniform_(-1, 1, generator=g)
gg = torch.empty(1, N, device=dev).uniform_(-1, 1, generator=g)
y = torch.empty(1, N, device=dev)
xb = torch.empty(1, N, device=dev)
ab = torch.empty(N, device=dev)
bb = torch.empty(N, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for it in range(6):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    ev[0].record()
    op = L.DeviceOperator(a, b, 1.0)
    ev[1].record()
    w1 = time.perf_counter()
    op.apply(x, out=y)
    ev[2].record()
    w2 = time.perf_counter()
    op.backward(x, gg, x_bar=xb, a_bar=ab, b_bar=bb)
    ev[3].record()
    w3 = time.perf_counter()
    del op
    torch.cuda.synchronize()
    w4 = time.perf_counter()
    print(f"it{it}: create {ev[0].elapsed_time(ev[1]):.1f} ms  apply {ev[1].elapsed_time(ev[2]):.1f}  "
          f"backward {ev[2].elapsed_time(ev[3]):.1f}  | host: create {1e3*(w1-w0):.1f} apply-enq {1e3*(w2-w1):.1f} "
          f"bwd-enq {1e3*(w3-w2):.1f} drain+free {1e3*(w4-w3):.1f}", flush=True)
