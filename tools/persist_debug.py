"""Locate persistent-vs-per-step mismatches (development aid)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan

def case(d, r, shape, steps, sweep, lag, dbg=0):
    os.environ["SPD_SWEEP"], os.environ["SPD_LAG"], os.environ["SPD_DBG"] = str(sweep), str(lag), str(dbg)
    rng = np.random.default_rng([d, 31 + r])
    c = rng.uniform(-1, 1, (2 * r + 1,) * d)
    k = sp.make_kernel("box", d, r, c) if d < 3 else sp.make_kernel_3d("box", r, c)
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    torch.manual_seed(0)
    dense = torch.rand(tuple(n + 2 * r for n in shape), dtype=torch.float64, device="cuda") - 0.5
    outs = []
    for persistent in (False, True):
        g = DeviceGrid(plan, shape, r)
        g.load_dense_f64(dense)
        g.run(steps, persistent=persistent)
        outs.append(g.to_dense_f64())
    bad = (outs[0] != outs[1]).nonzero()
    msg = f"d={d} r={r} {shape} steps={steps} sweep={sweep} lag={lag} dbg={dbg}: {len(bad)} mismatches"
    if len(bad):
        b = bad.cpu().numpy()
        msg += f"; rows {b[:, 0].min()}..{b[:, 0].max()} cols {b[:, -1].min()}..{b[:, -1].max()}; first {b[:5].tolist()}"
        rows = np.unique(b[:, 0] // 16)
        msg += f"; bands(16) {rows[:20].tolist()}"
    print(msg, flush=True)

for st in (3, 4, 6, 9):
    case(2, 3, (600, 1024), st, st, 2)
for st in (6, 9, 12):
    case(2, 3, (600, 1024), st, 1, 2)
for lag in (3, 4, 8):
    case(2, 3, (600, 1024), 9, 4, lag)
case(2, 3, (600, 1024), 9, 4, 2, 512)
case(2, 3, (600, 1024), 9, 9, 2, 512)
case(2, 1, (600, 1024), 12, 12, 2)
case(2, 1, (600, 1024), 12, 1, 2)
case(2, 2, (300, 1536), 7, 3, 2)
case(2, 1, (600, 1024), 9, 4, 2)

# magnitude check against the CPU oracle (r=3)
from oracle import cnaive
for r, shape, steps in ((3, (128, 512), 3), (3, (128, 512), 2), (1, (128, 512), 3)):
    os.environ["SPD_SWEEP"], os.environ["SPD_LAG"], os.environ["SPD_DBG"] = "1", "2", "0"
    rng = np.random.default_rng([2, 31 + r])
    c = rng.uniform(-1, 1, (2 * r + 1,) * 2)
    c /= np.abs(c).sum()
    k = sp.make_kernel("box", 2, r, c)
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    dense = (torch.rand(tuple(n + 2 * r for n in shape), dtype=torch.float64) - 0.5).half().double()
    outs = []
    for persistent in (False, True):
        g = DeviceGrid(plan, shape, r)
        g.load_dense_f64(dense.cuda())
        g.run(steps, persistent=persistent)
        outs.append(g.to_dense_f64().cpu().numpy())
    want = cnaive.naive_apply(c, 2, r, dense.numpy(), r, steps)
    print(f"r={r} steps={steps}: |ps-pers| {np.abs(outs[0]-outs[1]).max():.3e} |ps-oracle| {np.abs(outs[0]-want).max():.3e} "
          f"|pers-oracle| {np.abs(outs[1]-want).max():.3e} max|want| {np.abs(want).max():.3e}", flush=True)
