"""Plain step launches then ordered (use_order) launches of one config, for an
ncu comparison of the two launch forms (dev aid)."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench, paper_2506_22035_b200 as sp
from paper_2506_22035_b200._lib import lib, check
from paper_2506_22035_b200.engine import DeviceGrid, _stream_ptr
from paper_2506_22035_b200.pipeline import get_plan
name = sys.argv[1] if len(sys.argv) > 1 else "B27"
desc, shape, d, r, kind, T = bench.CONFIGS[name]
plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
inf = plan.info()
g = DeviceGrid(plan, shape, r)
g.load_dense_f64(torch.rand(g.dense_shape, dtype=torch.float64, device="cuda") - 0.5)
band = inf.tile_z if d == 3 else inf.tile_y
nb = -(-shape[0] // band)
order = list(range(nb)) + list(range(nb - 1, -1, -1))
ordt = torch.tensor([[0, b] for b in order], dtype=torch.int32, device="cuda")
cnt = torch.zeros(nb, dtype=torch.int32, device="cuda")
for _ in range(4):
    g.run(1)
for i in range(4):
    a, b = g.bufs[g.cur], g.bufs[1 - g.cur]
    check(lib.spd_step_ordered(plan.handle, C.byref(g.desc), C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                               C.c_void_p(ordt[(i & 1) * nb:].data_ptr()), nb, C.c_void_p(cnt.data_ptr()), 0, _stream_ptr()))
    g.flip()
torch.cuda.synchronize()
print("done")
