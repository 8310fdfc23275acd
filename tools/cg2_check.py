"""CTA-pair (cta_group::2) 3D path vs the default path, bit for bit (dev aid).
Run twice: SPD_3D_CG2=1 writes /tmp/cg2.pt, plain run compares."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan
rng = np.random.default_rng(3)
c = rng.uniform(0.5, 1.5, (3, 3, 3)); c /= c.sum()
k = sp.make_kernel_3d("box", 1, c)
plan = get_plan(k, sp.Parity.EVEN, "fp16")
print("cg2 =", plan.info().cg2, flush=True)
outs = {}
for shape in [(16, 16, 512), (40, 48, 256), (64, 64, 600)]:
    torch.manual_seed(0)
    dense = torch.rand(tuple(n + 2 for n in shape), dtype=torch.float64, device="cuda") - 0.5
    g = DeviceGrid(plan, shape, 1)
    g.load_dense_f64(dense)
    g.run(3)
    torch.cuda.synchronize()
    outs[shape] = g.to_dense_f64().cpu()
path = "/tmp/cg2.pt"
if plan.info().cg2:
    torch.save(outs, path)
    print("saved", flush=True)
else:
    ref = torch.load(path)
    for kk in outs:
        same = torch.equal(outs[kk], ref[kk])
        print(kk, "bit-identical" if same else f"DIFF max {(outs[kk]-ref[kk]).abs().max().item():.3e}", flush=True)
