"""Per-step device results vs the CPU oracle on grids with many tiles per CTA
(ring wrap-around), every geometry (development aid)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan
from oracle import cnaive

def case(d, r, shape, steps, persistent=False):
    rng = np.random.default_rng([d, 31 + r])
    c = rng.uniform(0.5, 1.5, (2 * r + 1,) * d)
    c /= c.sum()
    k = sp.make_kernel("box", d, r, c) if d < 3 else sp.make_kernel_3d("box", r, c)
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    torch.manual_seed(0)
    dense = (torch.rand(tuple(n + 2 * r for n in shape), dtype=torch.float64) - 0.5).half().double()
    g = DeviceGrid(plan, shape, r)
    g.load_dense_f64(dense.cuda())
    g.run(steps, persistent=persistent)
    got = g.to_dense_f64().cpu().numpy()
    want = cnaive.naive_apply(c, d, r, dense.numpy(), r, steps, threads=os.cpu_count())
    err = np.abs(got - want)
    bad = err > 2e-3 * np.abs(want).max() + 1e-3
    msg = f"d={d} r={r} {shape} steps={steps} pers={persistent}: max err {err.max():.3e}, bad {bad.sum()}"
    if bad.any():
        idx = np.argwhere(bad)
        msg += f" first {idx[:3].tolist()} rows {idx[:,0].min()}..{idx[:,0].max()}"
    print(msg, flush=True)

for pers in (False, True):
    case(2, 3, (600, 1024), 9, pers)
    case(2, 3, (600, 1024), 6, pers)
    case(2, 3, (608, 1024), 9, pers)
    case(2, 1, (600, 1024), 9, pers)
    case(2, 3, (100, 1024), 9, pers)
