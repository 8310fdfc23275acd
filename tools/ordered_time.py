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
    def ordered(publish=1, ot=ordt):
        a, b = g.bufs[g.cur], g.bufs[1 - g.cur]
        check(lib.spd_step_ordered(plan.handle, C.byref(g.desc), C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                   C.c_void_p(ot[par[0] * nb:].data_ptr()), nb, C.c_void_p(cnt.data_ptr()), publish,
                                   _stream_ptr()))
        par[0] ^= 1
        g.flip()
    # plain traversal order through the ordered launch (isolates the order array / publishing)
    plain_order = list(range(nb)) + list(range(nb - 1, -1, -1))
    plain_ordt = torch.tensor([[0, b] for b in plain_order], dtype=torch.int32, device="cuda")
    def edge_first(publish=1):
        a, b = g.bufs[g.cur], g.bufs[1 - g.cur]
        check(lib.spd_step_edge_first(plan.handle, C.byref(g.desc), C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                      par[0], C.c_void_p(cnt.data_ptr()), publish, _stream_ptr()))
        par[0] ^= 1
        g.flip()
    def two():
        g.step_edges(); g.step_range(band, last); g.flip()
    import time
    variants = ((plain, "plain"), (ordered, "one launch, order array, published"),
                (lambda: ordered(0), "one launch, order array, not published"),
                (lambda: ordered(0, plain_ordt), "one launch, plain band order array, not published"),
                (edge_first, "edge-first (arithmetic order), published"),
                (lambda: edge_first(0), "edge-first (arithmetic order), not published"),
                (two, "edges + interior launches"))
    res = {lab: [] for _, lab in variants}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rnd in range(3):  # interleaved rounds, each after a cool-down (sustained runs hit the power cap)
        for fn, lab in variants:
            time.sleep(1.0)
            for _ in range(4): fn()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(20): fn()
            e1.record(); torch.cuda.synchronize()
            res[lab].append(e0.elapsed_time(e1) / 20 * 1e3)
    for _, lab in variants:
        print(f"{name} {lab}: {min(res[lab]):.1f} us/step (best of 3 x 20 after cool-down)", flush=True)
