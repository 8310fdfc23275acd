"""A/B of spd_run_ex launch modes (timing + bit-identity), one GPU.
usage: python tools/chain_ab.py [configs...]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200 import engine
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan

MODES = {"per-step": 0, "persist-sm": engine.SPD_RUN_PERSISTENT | engine.SPD_RUN_STEPMAJOR,
         "persist-wave": engine.SPD_RUN_PERSISTENT}
names = sys.argv[1:] or ["B9", "B27", "B49", "W"]
for name in names:
    desc, shape, d, r, kind, T = bench.CONFIGS[name]
    plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
    g = DeviceGrid(plan, shape, r)
    torch.manual_seed(0)
    dense = torch.rand(g.dense_shape, dtype=torch.float64, device="cuda") - 0.5
    res = {}
    outs = {}
    for mode, fl in MODES.items():
        g.cur = 0
        g.load_dense_f64(dense)
        g.run(T, flags=fl)
        outs[mode] = g.bufs[g.cur].clone()
    for rep in range(3):
        for mode, fl in MODES.items():
            for _ in range(2):
                g.run(T, flags=fl)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(5):
                g.run(T, flags=fl)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (5 * T)
            res.setdefault(mode, []).append(us)
    same = {m: bool(torch.equal(outs[m], outs["per-step"])) for m in MODES}
    pts = 1
    for v in shape:
        pts *= v
    line = "  ".join(f"{m} {min(v):.1f}us ({pts / min(v) / 1e3:.0f} GSt/s)" for m, v in res.items())
    print(f"{name}: {line}  bit-identical {same}", flush=True)
    del g, plan, dense
    torch.cuda.empty_cache()
