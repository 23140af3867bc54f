"""Host-pointer step repeated: per-call wall times (diagnostics for e2e variance)."""
import ctypes as C, sys, time, statistics, torch
sys.path.insert(0, ".")
from paper_2605_24584_b200 import _lib
n = k = 1 << 30
lib = _lib.lib()
pin = dict(dtype=torch.float32, pin_memory=True)
ha = torch.empty(n, **pin).uniform_(-100, 100); hb = torch.empty(k, **pin).uniform_(-100, 100)
hx = torch.empty(k, **pin).uniform_(-1, 1); hg = torch.empty(n, **pin).uniform_(-1, 1)
hy, hxb, hab, hbb = (torch.empty(n, **pin) for _ in range(4))
for it in range(6):
    h = C.c_void_p()
    t0 = time.perf_counter(); lib.laplex_plan_create(0, ha.data_ptr(), n, hb.data_ptr(), k, 1.0, None, None, C.byref(h))
    t1 = time.perf_counter(); lib.laplex_apply(h, 0, hx.data_ptr(), 1, k, hy.data_ptr())
    t2 = time.perf_counter(); lib.laplex_backward(h, 0, hx.data_ptr(), 1, k, hg.data_ptr(), n, hxb.data_ptr(), hab.data_ptr(), hbb.data_ptr(), None, None)
    t3 = time.perf_counter(); lib.laplex_plan_release(h); t4 = time.perf_counter()
    print(f"it{it}: create {1e3*(t1-t0):.0f} apply {1e3*(t2-t1):.0f} backward {1e3*(t3-t2):.0f} release {1e3*(t4-t3):.0f} total {1e3*(t4-t0):.0f}", flush=True)
