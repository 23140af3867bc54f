"""Break the host-pointer e2e step into its parts (PCIe copies, host finiteness scans, API calls)."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_24584_b200 import _lib

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n = k = 1 << lg
lib = _lib.lib()
pin = dict(dtype=torch.float32, pin_memory=True)
ha = torch.empty(n, **pin).uniform_(-100, 100)
hb = torch.empty(k, **pin).uniform_(-100, 100)
hx = torch.empty(k, **pin).uniform_(-1, 1)
hg = torch.empty(n, **pin).uniform_(-1, 1)
hy, hxb, hab, hbb = (torch.empty(n, **pin) for _ in range(4))
d = torch.empty(n, device="cuda")
torch.cuda.synchronize()


def tm(f, reps=2):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


print("h2d 4 B x n ms", tm(lambda: d.copy_(ha, non_blocking=True)))
print("d2h 4 B x n ms", tm(lambda: hy.copy_(d, non_blocking=True)))
print("np isfinite ms", tm(lambda: bool(np.isfinite(ha.numpy()).all())))
h = C.c_void_p()


def create_release():
    lib.laplex_plan_create(0, ha.data_ptr(), n, hb.data_ptr(), k, 1.0, None, None, C.byref(h))
    lib.laplex_plan_release(h)


print("plan_create+release ms", tm(create_release))
lib.laplex_plan_create(0, ha.data_ptr(), n, hb.data_ptr(), k, 1.0, None, None, C.byref(h))
print("apply ms", tm(lambda: lib.laplex_apply(h, 0, hx.data_ptr(), 1, k, hy.data_ptr())))
print("backward ms", tm(lambda: lib.laplex_backward(h, 0, hx.data_ptr(), 1, k, hg.data_ptr(), n, hxb.data_ptr(),
                                                   hab.data_ptr(), hbb.data_ptr(), None, None)))


def fwd_bwd_reuse():  # the bench's e2e pair: apply(SAVE_X) + backward(REUSE_X)
    lib.laplex_apply(h, 8, hx.data_ptr(), 1, k, hy.data_ptr())
    lib.laplex_backward(h, 4, hx.data_ptr(), 1, k, hg.data_ptr(), n, hxb.data_ptr(), hab.data_ptr(), hbb.data_ptr(),
                        None, None)


print("apply(SAVE_X)+backward(REUSE_X) ms", tm(fwd_bwd_reuse))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty(n, device="cuda")


def duplex():  # H2D and D2H at once on two streams
    with torch.cuda.stream(s1):
        d.copy_(ha, non_blocking=True)
    with torch.cuda.stream(s2):
        hy.copy_(d2, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


print("h2d || d2h 4 B x n each ms", tm(duplex))
import os
print("cpus", os.cpu_count())
