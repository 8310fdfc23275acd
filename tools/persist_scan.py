"""Scan the persistent (wavefront) schedule: SPD_SWEEP x SPD_LAG per config
(development aid, device-timed, not the bench)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench, paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["B9"]
sweeps = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "0,2,4,8,16,32".split(","))]
lags = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else "2,3,4".split(","))]
for name in names:
    desc, shape, d, r, kind, T = bench.CONFIGS[name]
    plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
    g = DeviceGrid(plan, shape, r)
    g.load_dense_f64(torch.rand(g.dense_shape, dtype=torch.float64, device="cuda") - 0.5)
    pts = int(np.prod(shape))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.run(T); torch.cuda.synchronize()
    e0.record(); g.run(T); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name} per-step launches: {ms / T * 1e3:.1f} us/step {pts * T / ms / 1e6:.1f} GStencil/s", flush=True)
    for lag, S, dbg in [(l, S, dbg) for l in lags for S in sweeps for dbg in os.environ.get("DBGS", "0").split(",")]:
        os.environ["SPD_DBG"] = dbg
        if True:
            if S:
                os.environ["SPD_SWEEP"] = str(S)
            else:
                os.environ.pop("SPD_SWEEP", None)
            os.environ["SPD_LAG"] = str(lag)
            g.run(T, persistent=True); torch.cuda.synchronize()
            best = 1e9
            for _ in range(3):
                e0.record(); g.run(T, persistent=True); e1.record(); torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            print(f"{name} persistent sweep={S or 'auto'} lag={lag} dbg={dbg}: {best / T * 1e3:.1f} us/step "
                  f"{pts * T / best / 1e6:.1f} GStencil/s", flush=True)
