"""bench.py on the GPU tier: the N>1 path launched by bench.py itself.

Two ranks share cuda:0 (SPD_BENCH_BACKEND=gloo): a functional check of the
self-launch, the slab decomposition, the peer-memory exchange and the JSON
line (timings on a shared GPU mean nothing).
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_bench_two_ranks_self_launched():
    env = dict(os.environ, SPD_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=900,
                         cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["parallelism"] == "slab2"
    assert line["impl_detail"]["exchange"] == "peer", out.stderr[-2000:]
    assert "W" in line["configs"] and line["configs"]["W"]["value"] > 0
    assert line["roofline"]["frac"] > 0 and line["gpu_launches"] > 0
    # e2e at N = 2: the whole job's grid through execute(..., DeviceConfig(devices=(0, 0)))
    assert line["e2e"]["value"] > 0 and "devices=(0, 0)" in line["e2e"]["api"]
    assert line["e2e"]["h2d_bytes_per_step"] == 2 * (2 * 10240 + 2) * (10240 + 2)


@pytest.mark.gpu
def test_bench_default_line_has_configs_block():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline", "--e2e-callers", "2"], capture_output=True, text=True, timeout=900,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["config"]["workload"] == "B9" and line["e2e"]["value"] > 0
    for name in ("B49", "B27", "W"):
        c = line["configs"][name]
        assert c["value"] > 0 and 0 < c["roofline"]["frac"] < 1.5 and c["clocks"]["samples"] >= 0
