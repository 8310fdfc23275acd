"""bench.py's JSON-line contract on the CPU tier: the reference arm (the
oracle's C port of naive_apply on the host cores) runs anywhere."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "S5",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["unit"] == "GStencil/s" and line["value"] > 0
    assert line["steps"] == 3 and line["warmup"] == 3 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["config"]["workload"] == "S5"


def test_warmup_floor():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--warmup", "1"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert out.returncode != 0 and "warmup" in out.stderr


def test_reference_arm_self_launch_two_ranks():
    """--gpus 2 without a launcher: bench.py starts both ranks itself; rank 0
    alone prints the reference line (the others exit 0 without work)."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "S5",
                          "--gpus", "2", "--steps", "3", "--warmup", "3"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["config"]["parallelism"] == "slab2"


def test_reference_config_matches_ours():
    """Both arms print the same workload description (`config`)."""
    sys.path.insert(0, str(ROOT))
    import bench

    c = bench.workload_config("B9", 1)
    assert c["workload"] == "B9" and c["timesteps_per_step"] == 100 and c["grid_per_gpu"] == [10240, 10240]
