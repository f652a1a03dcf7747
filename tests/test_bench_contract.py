"""The bench.py line the driver parses: one JSON object with the contract keys, on the GPU
(short run: 4 steps incl. one dense, 3 warm-up steps, 3 kernel reps, no CPU baseline)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_line_contract(cuda):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "4",
                          "--warmup", "3", "--kernel-reps", "3", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    r = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "clocks"):
        assert k in r, k
    assert r["n_gpus"] == 1 and r["steps"] == 4 and r["warmup"] == 3
    assert r["higher_is_better"] is False and r["unit"] == "ms/step" and r["value"] > 0
    assert r["gpu_launches"] > 0
    assert r["e2e"]["h2d_bytes_per_step"] > 0 and r["e2e"]["d2h_bytes_per_step"] > 0
    assert r["e2e"]["value"] >= r["value"] * 0.9  # host copies can only add time
    rf = r["roofline"]
    assert rf["bound"] in ("hbm", "tensor") and 0 < rf["frac"] < 1 and rf["peak"] > 0
    assert r["config"]["workload"] and r["config"]["seq_len"] == 4608
    assert r["attention"]["speedup_vs_dense"] > 1
