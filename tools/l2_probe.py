"""Per-step time of a stencil on grids small enough to stay in L2 (is the step
kernel faster when its working set is L2-resident?  Sizing for L2 slab
blocking).  usage: python tools/l2_probe.py CONFIG extent...   (extent = rows
for 2D / planes for 3D; the other dims are the config's)"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan

name = sys.argv[1]
desc, shape, d, r, kind, T = bench.CONFIGS[name]
plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
for ext in [int(v) for v in sys.argv[2:]]:
    shp = (ext,) + tuple(shape[1:])
    g = DeviceGrid(plan, shp, r)
    dense = torch.rand(g.dense_shape, dtype=torch.float64, device="cuda") - 0.5
    g.load_dense_f64(dense)
    del dense
    g.run(T)
    best = 1e9
    for rep in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            g.run(T)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / (3 * T))
    pts = 1
    for v in shp:
        pts *= v
    mb = 2 * g.desc.alloc_elems * 2 / 2**20
    print(f"{name} {shp} {mb:7.1f} MiB both bufs  {best:8.2f} us/step  {pts / best / 1e3:7.1f} GSt/s", flush=True)
    del g
    torch.cuda.empty_cache()
