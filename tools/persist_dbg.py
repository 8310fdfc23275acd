"""Which part of the persistent step-major launch costs time (DEVEL build,
SPD_DBG switches; results are garbage when a dependency is skipped).
usage: SPD_LIB=tools/libspider_devel.so python tools/persist_dbg.py [config]"""
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
PS = engine.SPD_RUN_PERSISTENT | engine.SPD_RUN_STEPMAJOR
cases = [("per-step", 0, "0"), ("persist-sm", PS, "0"),
         ("no publisher (no poll)", PS, "2688"), ("no poller", PS, "4096"), ("no publisher/poller/fence", PS, "6176"),
         ("bare + no stores", PS, "6177"), ("poller handoff, no fences", PS, "2720"),
         ("publisher, no fence", PS, "4160"), ("all, no fences/polls", PS, "736"), ("all, no proxy fence", PS, "32"), ("per-step no stores", 0, "1")]
only = os.environ.get("CASE")
for rep in range(1):
    for label, fl, dbg in cases:
        if only is not None and dbg != only:
            continue
        os.environ["SPD_DBG"] = dbg
        g.run(T, flags=fl)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            g.run(T, flags=fl)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} {label:28s} dbg={dbg:5s} {e0.elapsed_time(e1) * 1e3 / (3 * T):7.1f} us/step", flush=True)
