"""Per-kernel device time of one range-sharded step (SimComm, world W on one GPU, n = k = 2^LG in total)
next to the unsharded step at the per-shard size (diagnostics for the multi-GPU path)."""
import ctypes
import json
import sys
import threading

import torch

sys.path.insert(0, ".")
import paper_2605_24584_b200 as L
from paper_2605_24584_b200 import _lib
from paper_2605_24584_b200.sharded import GpuBackend, ShardedOperator, SimComm, SimWorld

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lib = _lib.lib()
dev = torch.device("cuda:0")
n = 1 << lg
nl = n // W
g = torch.Generator(device=dev)
g.manual_seed(5)
data = [[torch.empty(nl, device=dev).uniform_(lo, hi, generator=g) for lo, hi in ((-100, 100), (-100, 100), (-1, 1), (-1, 1))]
        for _ in range(W)]


def dump(tag):
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    lib.laplex_profile_dump(buf, len(buf))
    lib.laplex_profile_enable(0)
    d = json.loads(buf.value.decode())
    print(f"== {tag}: total {sum(v['ms'] for v in d.values()):.2f} ms")
    for k, v in sorted(d.items(), key=lambda kv: -kv[1]["ms"])[:14]:
        print("   %-24s %4d %8.3f" % (k, v["launches"], v["ms"]))


def sharded_step():
    w = SimWorld(W)
    be = GpuBackend()

    def run(r):
        a, b, x, gg = data[r]
        op = ShardedOperator(a, b, 1.0, SimComm(w, r), be)
        op.apply(x)
        op.backward(x, gg)
    ths = [threading.Thread(target=run, args=(r,)) for r in range(W)]
    [t.start() for t in ths]
    [t.join() for t in ths]


def plain_step():
    a, b, x, gg = data[0]
    op = L.DeviceOperator(a, b, 1.0)
    op.apply(x[None])
    op.backward(x[None], gg[None])


for f, tag in ((plain_step, f"unsharded n=k=2^{lg}/{W}"), (sharded_step, f"sharded W={W}, all shards")):
    f()
    f()
    torch.cuda.synchronize()
    lib.laplex_profile_enable(1)
    f()
    dump(tag)
