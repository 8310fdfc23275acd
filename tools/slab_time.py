"""Multi-slab step time on one GPU (slabs share cuda:0), device-timed over the
slab steps only: fused peer stores vs the copy-engine exchange
(SPD_SLAB_COPY=1), against one plain grid; dev aid.
usage: python tools/slab_time.py CONFIG n"""
import ctypes as C
import os
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200._lib import check, lib
from paper_2506_22035_b200.distributed import LocalSlabs
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan

name = sys.argv[1] if len(sys.argv) > 1 else "B9"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
desc, shape, d, r, kind, T = bench.CONFIGS[name]
k = bench.make_kernel(kind, d, r)
plan = get_plan(k, sp.Parity.EVEN, "fp16", 0)
data = np.random.default_rng(1).uniform(-1, 1, tuple(s + 2 * r for s in shape)).astype(np.float16)
g = DeviceGrid(plan, shape, r)
g.upload(torch.from_numpy(data))
time.sleep(1.0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.run(T); e1.record(); torch.cuda.synchronize()
print(f"{name} one grid: {e0.elapsed_time(e1) * 1e3 / T:.1f} us/step", flush=True)
for mode in ("fused", "copy", "fused", "copy"):
    os.environ["SPD_SLAB_COPY"] = "1" if mode == "copy" else "0"
    ls = LocalSlabs({0: plan}, (0,) * n, shape, r)
    for kk, (s, gg) in enumerate(zip(ls.slabs, ls.grids)):
        gg.upload(torch.from_numpy(np.ascontiguousarray(data[s.lo: s.hi + 2 * r])))
    torch.cuda.synchronize()
    ls._create_handles()
    time.sleep(1.0)
    start = torch.cuda.Event(enable_timing=True)
    start.record()
    for t in range(T):
        for kk in range(n):
            cs, xs = ls.streams[kk]
            cs.wait_event(start) if t == 0 else None
            check(lib.spd_slab_step(ls.handles[kk], t, C.c_void_p(cs.cuda_stream), C.c_void_p(xs.cuda_stream)))
    ends = []
    for kk in range(n):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(ls.streams[kk][0])
        ends.append(ev)
    torch.cuda.synchronize()
    ms = max(start.elapsed_time(ev) for ev in ends)
    for h in ls.handles:
        lib.spd_slab_destroy(h)
    print(f"{name} {n} slabs {mode}: {ms * 1e3 / T:.1f} us/step (all slabs, one GPU)", flush=True)
