"""Device time per step of one bench config (development aid; SPD_LIB picks
the build): python tools/quick_one.py B25 [steps]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench, paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
_, shape, d, r, kind, T = bench.CONFIGS[name]
plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
dg = DeviceGrid(plan, shape, r)
dg.load_dense_f64(torch.rand(dg.dense_shape, dtype=torch.float64, device="cuda") - 0.5)
dg.run(5); torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dg.run(steps); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / steps)
pts = float(np.prod(shape))
print(f"{name}: {best*1e3:.1f} us/step {pts/best/1e6:.1f} GStencil/s", flush=True)
