"""Per-rank device time of the C++ range-sharded step (laplex_sharded_*, local communicators: W ranks as
threads on one GPU, n = k = 2^LG in total), per kernel via the profile API, next to the unsharded step at
the per-rank size (diagnostics for the multi-GPU path; kernel times of all ranks summed, then / W)."""
import ctypes
import json
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_2605_24584_b200 as L
from paper_2605_24584_b200 import _lib
from paper_2605_24584_b200.sharded import Comm, CppShardedOperator

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
lib = _lib.lib()
n = 1 << lg
nl = n // W
gen = torch.Generator(device="cuda:0")
gen.manual_seed(5)
data = [[torch.empty(nl, device="cuda:0").uniform_(lo, hi, generator=gen) for lo, hi in
         ((-100, 100), (-100, 100), (-1, 1), (-1, 1))] for _ in range(W)]


def dump(tag, div):
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.laplex_profile_dump(buf, len(buf))
    lib.laplex_profile_enable(0)
    d = json.loads(buf.value.decode())
    print(f"== {tag}: {sum(v['ms'] for v in d.values()) / div:.2f} ms of kernels per rank")
    for k, v in sorted(d.items(), key=lambda kv: -kv[1]["ms"])[:16]:
        print("   %-24s %5d %8.3f" % (k, v["launches"] // div, v["ms"] / div))


def sharded(profile):
    key = int(time.time() * 1e6)

    def body(r):
        torch.cuda.set_device(0)
        comm = Comm.local(key, W, r)
        st = torch.cuda.Stream()
        a, b, x, g = data[r]
        with torch.cuda.stream(st):
            op = CppShardedOperator(a, b, 1.0, comm, stream=st)
            y = op.apply(x[None], stream=st)
            op.backward(x[None], g[None], reuse_x=True, stream=st)
        st.synchronize()
        del op, y
    th = [threading.Thread(target=body, args=(r,)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join()


sharded(False)
lib.laplex_profile_enable(1)
sharded(True)
dump(f"sharded step, {W} ranks x (2^{lg - W.bit_length() + 1} + 2^{lg - W.bit_length() + 1})", W)
a, b, x, g = (torch.cat([d[i] for d in data]) for i in range(4))
for it in range(2):
    if it == 1:
        lib.laplex_profile_enable(1)
    op = L.DeviceOperator(a[:nl], b[:nl], 1.0)
    op.apply(x[None, :nl], save_x=True)
    op.backward(x[None, :nl], g[None, :nl], reuse_x=True)
    del op
dump(f"unsharded step at the per-rank size", 1)
