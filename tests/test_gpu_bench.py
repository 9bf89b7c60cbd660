"""bench.py's contract on a small cloud (the round-end driver runs it at full size): one JSON
line with the required keys, a roofline block, per-kernel times and e2e through the C ABI."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_json_contract():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--n", "300000", "--steps", "3", "--warmup", "3",
           "--no-cpu"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "gpu_launches", "roofline", "e2e", "clocks"):
        assert key in line, key
    assert line["value"] > 0 and line["gpu_launches"] > 0 and line["warmup"] >= 3
    r = line["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1 and r["peak"] > 0 and r["kernels"]
    e = line["e2e"]
    assert e["value"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
