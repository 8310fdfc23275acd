"""Time spd_run_ex for configs (per-step launches, T steps, best of reps) and
print a hash of the result so library variants can be compared bit for bit.
usage: [SPD_LIB=...] python tools/time_cfg.py [flags=N] CONFIG..."""
import hashlib
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan

flags = 0
names = []
for a in sys.argv[1:]:
    if a.startswith("flags="):
        flags = int(a.split("=")[1])
    else:
        names.append(a)
for name in names or ["B9"]:
    desc, shape, d, r, kind, T = bench.CONFIGS[name]
    plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
    g = DeviceGrid(plan, shape, r)
    gen = torch.Generator(device="cuda").manual_seed(7)
    dense = torch.rand(g.dense_shape, dtype=torch.float64, device="cuda", generator=gen) - 0.5
    g.load_dense_f64(dense)
    g.run(T, flags=flags)
    torch.cuda.synchronize()
    h = hashlib.sha1(g.bufs[g.cur].cpu().numpy().tobytes()).hexdigest()[:12]
    best = 1e9
    import time
    time.sleep(1.0)  # cool-down: sustained runs reach the board power cap within ~0.1 s
    for rep in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            g.run(T, flags=flags)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / (3 * T))
    pts = 1
    for v in shape:
        pts *= v
    print(f"{name:4s} {best:7.1f} us/step  {pts / best / 1e3:7.1f} GSt/s  {4 * pts / best / 1e3 / 6545.6:.3f} of HBM  hash {h}",
          flush=True)
    del g, plan, dense
    torch.cuda.empty_cache()
