"""Small runs of every kernel family for compute-sanitizer (dev aid)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan
rng = np.random.default_rng(0)
for d, r, shape in [(2, 1, (70, 600)), (2, 3, (40, 520)), (2, 2, (30, 390)), (3, 1, (12, 10, 200)), (1, 1, (1, 4000))]:
    c = rng.uniform(0.5, 1.5, (2 * r + 1,) * d); c /= c.sum()
    k = sp.make_kernel_3d("box", r, c) if d == 3 else sp.make_kernel("box", d, r, c)
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    g = DeviceGrid(plan, shape, r)
    g.load_dense_f64(torch.rand(tuple(n + 2 * r for n in shape), dtype=torch.float64, device="cuda"))
    g.run(2)
    if d >= 2:
        g.run(3, persistent=True)
    torch.cuda.synchronize()
    print("ok", d, r, shape, flush=True)

# round-2 paths: embedded radius 2 with a partial last chunk (width % 8 != 0),
# multi-slab execute with the in-kernel peer copies (both launch forms), and
# the streamed execute with tapered windows
import os
from paper_2506_22035_b200.pipeline import DeviceConfig
for d, r, shape in [(2, 2, (64, 390)), (2, 1, (256, 1024)), (3, 1, (32, 16, 128)), (2, 4, (100, 1000))]:
    c = rng.uniform(0.5, 1.5, (2 * r + 1,) * d); c /= c.sum()
    k = sp.make_kernel_3d("box", r, c) if d == 3 else sp.make_kernel("box", d, r, c)
    data = rng.uniform(-1, 1, tuple(n + 2 * r for n in shape)).astype(np.float16)
    g = sp.Grid3D(data, r) if d == 3 else sp.Grid(data, r)
    for form in ("0", "1"):
        os.environ["SPD_SLAB_TWO_LAUNCH"] = form
        sp.execute(k, g, 3, DeviceConfig(devices=(0, 0)))
    os.environ["SPD_STREAM_WINDOWS"] = "3"
    sp.execute(k, g, 2)
    del os.environ["SPD_STREAM_WINDOWS"]
    torch.cuda.synchronize()
    print("ok slabs/streamed", d, r, shape, flush=True)
