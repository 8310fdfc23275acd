"""Quick device timing of the step kernel (development aid, not the bench)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan

PERSIST = "persistent" in sys.argv

def bench(name, kern, shape, steps=20):
    plan = get_plan(kern, sp.Parity.EVEN, "fp16")
    dg = DeviceGrid(plan, shape, kern.r)
    dense = torch.rand(dg.dense_shape, dtype=torch.float64, device="cuda") - 0.5
    dg.load_dense_f64(dense); del dense
    dg.run(3); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dg.run(steps); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    pts = np.prod(shape)
    g = pts / ms / 1e6
    if PERSIST:
        dg.run(4, persistent=True); torch.cuda.synchronize()
        e0.record(); dg.run(steps, persistent=True); e1.record(); torch.cuda.synchronize()
        pm = e0.elapsed_time(e1) / steps
        print(f"{name} [persistent]: {pm*1e3:.1f} us/step  {pts/pm/1e6:.1f} GStencil/s", flush=True)
    print(f"{name}: {ms*1e3:.1f} us/step  {g:.1f} GStencil/s  {4*pts/ms/1e6:.0f} GB/s alg ({4*pts/ms/1e6/6541.8*100:.1f}% HBM)", flush=True)

c = np.zeros((3,3)); c[1,1]=0.5; c[0,1]=c[2,1]=c[1,0]=c[1,2]=0.125
rng = np.random.default_rng(0)
w = rng.uniform(0.5,1.5,9); w/=w.sum()
bench("Box-2D9P 10240^2", sp.make_kernel("box",2,1,w), (10240,10240))
w = rng.uniform(0.5,1.5,49); w/=w.sum()
bench("Box-2D49P 10240^2", sp.make_kernel("box",2,3,w), (10240,10240))
w = rng.uniform(0.5,1.5,27); w/=w.sum()
bench("Box-3D27P 512^3", sp.make_kernel_3d("box",1,w), (512,512,512))
bench("Heat-2D 16384^2", sp.make_kernel("star",2,1,c), (16384,16384))
if "generic" in sys.argv:
    for r in (2, 4, 7):
        n = 2 * r + 1
        w = rng.uniform(0.5, 1.5, n * n); w /= w.sum()
        L = 2 * r + 2
        bench(f"Box-2D{n*n}P r={r} ~10240^2", sp.make_kernel("box", 2, r, w), (10240, (10240 // (64 * L)) * 64 * L))
