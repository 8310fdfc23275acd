"""Persistent (L2 wavefront) vs per-step launches at full size, bit for bit,
repeated (race detector for the publish / poll ordering; dev aid)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench, paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan
for name in sys.argv[1:] or ["B9", "B27", "B49"]:
    desc, shape, d, r, kind, T = bench.CONFIGS[name]
    plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
    torch.manual_seed(1)
    dense = torch.rand(tuple(n + 2 * r for n in shape), dtype=torch.float64, device="cuda") - 0.5
    ref = DeviceGrid(plan, shape, r); ref.load_dense_f64(dense); ref.run(T)
    want = ref.bufs[ref.cur].clone()
    for rep, (sw, lag) in enumerate([(None, None), ("16", "6"), ("4", "2"), ("1", "2")]):
        if sw: os.environ["SPD_SWEEP"], os.environ["SPD_LAG"] = sw, lag
        g = DeviceGrid(plan, shape, r); g.load_dense_f64(dense); g.run(T, persistent=True)
        ok = torch.equal(g.bufs[g.cur], want)
        print(f"{name} T={T} sweep={sw or 'auto'} lag={lag or 'auto'}: {'bit-identical' if ok else 'MISMATCH'}", flush=True)
        del g
    del ref, dense
    torch.cuda.empty_cache()
