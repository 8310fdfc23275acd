"""Which part of the chained-launch machinery costs time (DEVEL build with
SPD_DBG switches; results are garbage when a dependency is skipped).
usage: SPD_LIB=tools/libspider_devel.so python tools/chain_dbg.py [config]"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200 import engine
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan

name = sys.argv[1] if len(sys.argv) > 1 else "B9"
desc, shape, d, r, kind, T = bench.CONFIGS[name]
plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
g = DeviceGrid(plan, shape, r)
dense = torch.rand(g.dense_shape, dtype=torch.float64, device="cuda") - 0.5
g.load_dense_f64(dense)
CH = engine.SPD_RUN_CHAINED | engine.SPD_RUN_FORWARD
FW = engine.SPD_RUN_FORWARD
CHA = engine.SPD_RUN_CHAINED
cases = [("per-step", 0, "0"), ("per-step fwd", FW, "0"), ("chained alt nothing", CHA, "736"), ("chained+gridwait", CH, "1024"),
         ("chained+gridwait nothing", CH, "1760"), ("chained", CH, "0"), ("no proxy fence", CH, "32"), ("no publish fence", CH, "64"),
         ("no poll wait", CH, "128"), ("no poll fence", CH, "512"), ("no poll wait+fence", CH, "640"),
         ("no fences at all", CH, "608"), ("nothing", CH, "736")]
for rep in range(2):
    for label, fl, dbg in cases:
        os.environ["SPD_DBG"] = dbg
        g.run(T, flags=fl)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(4):
            g.run(T, flags=fl)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} {label:22s} dbg={dbg:4s} {e0.elapsed_time(e1) * 1e3 / (4 * T):7.1f} us/step", flush=True)
