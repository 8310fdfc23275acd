"""One-launch slab step (edge bands first, published per band) vs the plain
step and the two-launch slab step, single GPU, no exchange (dev aid)."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench, paper_2506_22035_b200 as sp
from paper_2506_22035_b200._lib import lib, check
from paper_2506_22035_b200.engine import DeviceGrid, _stream_ptr
from paper_2506_22035_b200.pipeline import get_plan
for name in sys.argv[1:] or ["B9", "W", "B27"]:
    desc, shape, d, r, kind, T = bench.CONFIGS[name]
    plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
    inf = plan.info()
    g = DeviceGrid(plan, shape, r)
    g.load_dense_f64(torch.rand(g.dense_shape, dtype=torch.float64, device="cuda") - 0.5)
    band = inf.tile_z if d == 3 else inf.tile_y
    nb = -(-shape[0] // band)
    order = [0, nb - 1] + list(range(1, nb - 1)) + [nb - 1, 0] + list(range(nb - 2, 0, -1))
    ordt = torch.tensor([[0, b] for b in order], dtype=torch.int32, device="cuda")
    par = [0]
    cnt = torch.zeros(nb, dtype=torch.int32, device="cuda")
    last = ((shape[0] - 1) // band) * band
    def plain():
        g.run(1)
    def ordered():
        a, b = g.bufs[g.cur], g.bufs[1 - g.cur]
        check(lib.spd_step_ordered(plan.handle, C.byref(g.desc), C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                   C.c_void_p(ordt[par[0] * nb:].data_ptr()), nb, C.c_void_p(cnt.data_ptr()), 1, _stream_ptr()))
        par[0] ^= 1
        g.flip()
    def two():
        g.step_edges(); g.step_range(band, last); g.flip()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for fn, lab in ((plain, "plain"), (ordered, "one launch, edges first, published"), (two, "edges + interior launches")):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(50): fn()
        e1.record(); torch.cuda.synchronize()
        print(f"{name} {lab}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us/step", flush=True)
