"""Per-kernel times of plan creation (2 sorts + plans) at 2^lg via the profile API."""
import ctypes as C
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
g.manual_seed(3)
a = torch.empty(N, device=dev).uniform_(-100, 100, generator=g)
b = torch.empty(N, device=dev).uniform_(-100, 100, generator=g)
lib = _lib.lib()
for _ in range(2):
    L.DeviceOperator(a, b, 1.0)
torch.cuda.synchronize()
lib.laplex_profile_enable(1)
reps = 3
for _ in range(reps):
    L.DeviceOperator(a, b, 1.0)
torch.cuda.synchronize()
buf = C.create_string_buffer(1 << 16)
lib.laplex_profile_dump(buf, len(buf))
prof = json.loads(buf.value.decode())
print(sys.argv[2] if len(sys.argv) > 2 else "", {k: round(v["ms"] / reps, 3) for k, v in prof.items()})
