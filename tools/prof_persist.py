"""Target for ncu: one persistent launch of T steps (never a bench number)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan
name = sys.argv[1] if len(sys.argv) > 1 else "B9"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 16
desc, shape, d, r, kind, T = bench.CONFIGS[name]
plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
g = DeviceGrid(plan, shape, r)
g.load_dense_f64(torch.rand(g.dense_shape, dtype=torch.float64, device="cuda") - 0.5)
g.run(steps, persistent=True)
g.run(steps, persistent=True)
torch.cuda.synchronize()
print("done", name, steps)
