"""fp32 path vs fp64 device path: relative l2 errors of y, x_bar, a_bar, b_bar at scale (diagnostics)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2605_24584_b200 as L
for lg, span in ((28, 100.0), (29, 100.0), (27, 3.0)):
    N = 1 << lg
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev); g.manual_seed(lg)
    a = torch.empty(N, device=dev).uniform_(-span, span, generator=g)
    b = torch.empty(N, device=dev).uniform_(-span, span, generator=g)
    x = torch.empty(1, N, device=dev).uniform_(-1, 1, generator=g)
    gg = torch.empty(1, N, device=dev).uniform_(-1, 1, generator=g)
    op = L.DeviceOperator(a, b, 1.0); r32 = [op.apply(x)] + list(op.backward(x, gg)[:3]); del op
    op = L.DeviceOperator(a.double(), b.double(), 1.0); r64 = [op.apply(x.double())] + list(op.backward(x.double(), gg.double())[:3]); del op
    rel = lambda u, w: float(torch.linalg.vector_norm(u.double() - w) / torch.linalg.vector_norm(w))
    print(f"2^{lg} span {span}: y {rel(r32[0], r64[0]):.2e} x_bar {rel(r32[1], r64[1]):.2e} a_bar {rel(r32[2], r64[2]):.2e} b_bar {rel(r32[3], r64[3]):.2e}", flush=True)
    del r32, r64, a, b, x, gg; torch.cuda.empty_cache()
