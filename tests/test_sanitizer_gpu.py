"""GPU: compute-sanitizer gates on the library's kernels -- memcheck,
racecheck and synccheck over one plan build, forward, transpose, backward,
phased forward/backward, Gram-vector, sort and scan (tools/sanitize_driver,
torch-free).  lx_main is a persistent, warp-specialised mbarrier pipeline and
lx_sort_pass / lx_gather_agg use shared-memory staging: these tools are what
proves the barriers and shared-memory hand-offs are race-free.  Sizes cover a
multi-tile plan (merge tiles of 2048, sort tiles of 6144) and, for memcheck,
the two-pass permutation plans (sides > 2^22)."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "tools", "sanitize_driver")
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,n,rows", [
    ("memcheck", 20000, 3),
    ("memcheck", (1 << 22) + 1000, 1),
    ("racecheck", 9000, 2),
    ("synccheck", 9000, 2),
    ("initcheck", 9000, 2),
])
def test_compute_sanitizer(tool, n, rows):
    assert os.path.exists(DRIVER), "tools/sanitize_driver not built (build() builds it)"
    # the driver's own checks first (it compares every call with its expectations)
    r = subprocess.run([DRIVER, str(n), str(rows)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok n=" in r.stdout + r.stderr, (r.stdout + r.stderr)[-4000:]
    cmd = [SAN, "--tool", tool, "--error-exitcode", "97"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    r = subprocess.run(cmd + [DRIVER, str(n), str(rows)], capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    if r.returncode != 0 and "compute-sanitizer is closed" in out:
        # the GPU pool can withdraw the sanitizer (its wrapper refuses to run); the
        # round's sanitizer results are kept in profiles/r02_*check*.txt
        pytest.skip("compute-sanitizer unavailable on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert r.returncode == 0, out[-4000:]
    assert "ok n=" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-2000:]
