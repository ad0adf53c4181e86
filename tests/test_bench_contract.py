"""CPU check of bench.py's reference arm (--impl reference): it runs the
UNMODIFIED reference (oracle/_ref bytecode or /root/reference) on a small
plate here, so the JSON contract the driver parses is covered without a GPU
(the GPU arm is exercised by the round-end bench)."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    sys.path.insert(0, REPO)
    from oracle import build_ref
    if build_ref.load() is None:
        pytest.skip("reference bdem unavailable")
    out = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "3",
         "--warmup", "0", "--ref-plate", "24", "14", "--ref-k", "1", "--ref-workers", "both"],
        capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference"
    assert line["metric"].startswith("Newton iters/sec")
    assert line["unit"] == "Newton it/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["steps"] == 3 and line["warmup"] == 0
    assert line["config"]["workload"].startswith("C3 plate")
    runs = line["measurements"]
    assert {r["workers"] for r in runs} == {os.cpu_count() or 1, 1}
    assert all(r["newton_iterations"] == 1 for r in runs)
    assert line["value"] == runs[0]["newton_per_s"]
    assert line["ms_per_step"] * 3 == __import__("pytest").approx(1e3 * runs[0]["seconds"])
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
