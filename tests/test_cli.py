"""The CPU-vs-GPU benchmark CLI (tools/laplex_bench): the reference harness's
CSV schema (proj/tools/laplex_bench.cpp:32-34) plus gpus / gbs / roofline_frac columns."""
import csv
import io
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tools", "laplex_bench")
REF_COLS = ["experiment", "method", "precision", "n", "k", "batch", "feature_count", "trial", "wall_ns",
            "peak_bytes", "rel_err_l2", "seed"]


def run(*args, check=True):
    if not os.path.exists(BIN):
        pytest.skip("tools/laplex_bench not built (python __graft_entry__.py)")
    p = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)
    if check:
        assert p.returncode == 0, p.stderr
    return p


def rows(text):
    r = list(csv.DictReader(io.StringIO(text)))
    return r


def test_cli_usage_and_flag_errors():
    assert run("--help", check=False).returncode == 0
    assert run("bench-nothing", check=False).returncode == 2
    p = run("bench-matvec", "--precision", "f16", check=False)
    assert p.returncode == 1 and "precision" in p.stderr
    p = run("bench-matvec", "--methods", "magic", check=False)
    assert p.returncode == 1
    p = run("bench-matvec", "--n-min", "1000", check=False)  # not a power of two
    assert p.returncode == 1


@pytest.mark.gpu
def test_cli_bench_matvec_schema_and_rows():
    p = run("bench-matvec", "--n-min", "1024", "--n-max", "4096", "--methods", "laplex,dense", "--trials", "2",
            "--warmups", "1", "--precision", "f32")
    header = p.stdout.splitlines()[0].split(",")
    assert header[:len(REF_COLS)] == REF_COLS
    assert header[len(REF_COLS):] == ["gpus", "gbs", "roofline_frac"]
    rs = rows(p.stdout)
    assert len(rs) == 3 * 2 * 2
    for r in rs:
        assert int(r["wall_ns"]) > 0
        if r["method"] == "laplex":
            assert r["gpus"] == "1" and float(r["gbs"]) > 0 and float(r["roofline_frac"]) > 0


@pytest.mark.gpu
def test_cli_accuracy_fp32_within_tolerance():
    p = run("accuracy", "--n-min", "256", "--n-max", "1024", "--batch", "2")
    rs = rows(p.stdout)
    assert len(rs) == 3 * 2 * 2
    for r in rs:
        if r["method"] == "laplex":
            assert float(r["rel_err_l2"]) <= 1e-5


@pytest.mark.gpu
def test_cli_bench_gram_rows():
    p = run("bench-gram", "--n-min", "512", "--n-max", "1024", "--gram-n", "32", "--methods", "laplex,dense",
            "--trials", "2", "--warmups", "1")
    rs = rows(p.stdout)
    assert len(rs) == 2 * 2 * 2
    assert all(r["precision"] == "f64" for r in rs)
