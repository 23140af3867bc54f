"""Stream-ordered pool footprint across C5 steps at 2^30 (diagnostics)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2605_24584_b200 as L
from cuda.bindings import runtime as rt
N = 1 << 30
dev = torch.device("cuda:0")
g = torch.Generator(device=dev); g.manual_seed(1)
a = torch.empty(N, device=dev).uniform_(-100, 100, generator=g)
b = torch.empty(N, device=dev).uniform_(-100, 100, generator=g)
x = torch.empty(1, N, device=dev).uniform_(-1, 1, generator=g)
gg = torch.empty(1, N, device=dev).uniform_(-1, 1, generator=g)
y = torch.empty(1, N, device=dev); xb = torch.empty(1, N, device=dev); ab = torch.empty(N, device=dev); bb = torch.empty(N, device=dev)
err, pool = rt.cudaDeviceGetDefaultMemPool(0)
def attr(a):
    return rt.cudaMemPoolGetAttribute(pool, a)[1]
for it in range(5):
    op = L.DeviceOperator(a, b, 1.0); op.apply(x, out=y); op.backward(x, gg, x_bar=xb, a_bar=ab, b_bar=bb); del op
    torch.cuda.synchronize()
    print(it, "reserved", int(attr(rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent))/2**30, "high", int(attr(rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemHigh))/2**30, "used high", int(attr(rt.cudaMemPoolAttr.cudaMemPoolAttrUsedMemHigh))/2**30, flush=True)
print("torch allocated GB", torch.cuda.memory_allocated()/2**30, "free GB", torch.cuda.mem_get_info()[0]/2**30)
