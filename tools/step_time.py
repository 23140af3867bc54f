"""Device time of one C5 step (plan + apply + backward) at 2^LG by CUDA events, median of 5 (diagnostics)."""
import statistics
import sys

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
ts = []
for it in range(7):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    e0.record()
    op = L.DeviceOperator(a, b, 1.0)
    e1.record()
    op.apply(x, out=y)
    op.backward(x, gg, x_bar=xb, a_bar=ab, b_bar=bb)
    e2.record()
    torch.cuda.synchronize()
    del op
    if it >= 2:
        ts.append((e0.elapsed_time(e1), e0.elapsed_time(e2)))
print("plan %.2f ms  step %.2f ms" % (statistics.median(t[0] for t in ts), statistics.median(t[1] for t in ts)))
