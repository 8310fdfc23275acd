"""Single-caller end-to-end execute() time of a config against the streamed
window count (SPD_STREAM_WINDOWS; 0 = whole-grid path).
usage: python tools/e2e_scan.py CONFIG windows..."""
import os
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
import paper_2506_22035_b200 as sp

name = sys.argv[1]
desc, shape, d, r, kind, T = bench.CONFIGS[name]
k = bench.make_kernel(kind, d, r)
dense = tuple(s + 2 * r for s in shape)
hin = torch.empty(dense, dtype=torch.float16, pin_memory=True)
hin.copy_((torch.rand(dense) * 2 - 1).half())
hout = torch.empty_like(hin, pin_memory=True)
cls = sp.Grid3D if d == 3 else sp.Grid
gin, gout = cls(hin.numpy(), r), cls(hout.numpy(), r)
ref = None
for w in sys.argv[2:]:
    os.environ["SPD_STREAM_WINDOWS"] = w
    sp.execute(k, gin, T, out=gout)
    if ref is None:
        ref = hout.clone()
    same = torch.equal(hout, ref)
    best = 1e9
    for _ in range(4):
        t0 = time.perf_counter()
        sp.execute(k, gin, T, out=gout)
        best = min(best, time.perf_counter() - t0)
    pts = float(np.prod(shape)) * T
    print(f"{name} windows={w}: {best * 1e3:7.2f} ms/call  {pts / best / 1e9:7.1f} GStencil/s e2e  same={same}",
          flush=True)
