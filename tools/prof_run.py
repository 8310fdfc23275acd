"""Run `launches` x spd_run_ex(steps, flags) of one config (ncu target; never a bench number).
usage: python tools/prof_run.py CONFIG STEPS FLAGS LAUNCHES"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan
name, steps, flags, launches = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
desc, shape, d, r, kind, T = bench.CONFIGS[name]
plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
g = DeviceGrid(plan, shape, r)
g.load_dense_f64(torch.rand(g.dense_shape, dtype=torch.float64, device="cuda") - 0.5)
for _ in range(launches):
    g.run(steps, flags=flags)
torch.cuda.synchronize()
print("done", name, steps, flags, launches)
