"""One C5-style step at a given size, for ncu captures (never a bench number)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2605_24584_b200 as L

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
N = 1 << lg
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(1)
a = torch.empty(N, device=dev).uniform_(-100, 100, generator=g)
b = torch.empty(N, device=dev).uniform_(-100, 100, generator=g)
x = torch.empty(1, N, device=dev).uniform_(-1, 1, generator=g)
gg = torch.empty(1, N, device=dev).uniform_(-1, 1, generator=g)
for _ in range(steps):
    op = L.DeviceOperator(a, b, 1.0)
    y = op.apply(x)
    op.backward(x, gg)
torch.cuda.synchronize()
print("done")
