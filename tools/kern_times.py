"""Per-kernel CUDA-event times of one C5 fwd+bwd step at 2^LG (diagnostics, not a bench line).
LAPLEX_LIB selects a variant build."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2605_24584_b200 as L
from paper_2605_24584_b200 import _lib

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
N = 1 << lg
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(1)
a = torch.empty(N, device=dev).uniform_(-100, 100, generator=g)
b = torch.empty(N, device=dev).uniform_(-100, 100, generator=g)
x = torch.empty(1, N, device=dev).uniform_(-1, 1, generator=g)
gg = torch.empty(1, N, device=dev).uniform_(-1, 1, generator=g)
lib = _lib.lib()
for it in range(3):
    if it == 2:
        lib.laplex_profile_enable(1)
    op = L.DeviceOperator(a, b, 1.0)
    y = op.apply(x)
    op.backward(x, gg)
    del op, y
    torch.cuda.synchronize()
buf = __import__("ctypes").create_string_buffer(1 << 16)
lib.laplex_profile_dump(buf, len(buf))
d = json.loads(buf.value.decode())
tot = sum(v["ms"] for v in d.values())
print("total %.2f ms" % tot)
for k, v in sorted(d.items(), key=lambda kv: -kv[1]["ms"]):
    print("%-22s %3d %9.3f" % (k, v["launches"], v["ms"]))
