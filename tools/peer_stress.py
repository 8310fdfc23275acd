"""Long-run stress of the slab exchange (fused peer copies): 2-3 slabs on one
GPU through execute(..., DeviceConfig(devices=...)), many steps, both slab
launch forms, against the one-grid run bit for bit (dev aid)."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.pipeline import DeviceConfig

cases = [(2, 1, (2048, 4096), 3, 300), (2, 3, (1024, 2048), 2, 200), (3, 1, (96, 64, 256), 3, 200),
         (2, 2, (1200, 3066), 3, 150), (2, 1, (4096, 16384), 2, 150)]
bad = 0
for d, r, shape, n, steps in cases:
    rng = np.random.default_rng([d, r, n])
    c = rng.uniform(0.5, 1.5, (2 * r + 1,) * d)
    c /= c.sum()
    k = sp.make_kernel_3d("box", r, c) if d == 3 else sp.make_kernel("box", d, r, c)
    data = rng.uniform(-1, 1, tuple(s + 2 * r for s in shape)).astype(np.float16)
    g = sp.Grid3D(data, r) if d == 3 else sp.Grid(data, r)
    os.environ["SPD_STREAM_WINDOWS"] = "0"
    want, _ = sp.execute(k, g, steps)
    for form in ("0", "1"):
        os.environ["SPD_SLAB_TWO_LAUNCH"] = form
        got, _ = sp.execute(k, g, steps, DeviceConfig(devices=(0,) * n))
        same = np.array_equal(got.data, want.data)
        bad += not same
        print(f"d={d} r={r} {shape} slabs={n} steps={steps} two_launch={form}: {'ok' if same else 'MISMATCH'}", flush=True)
print("all ok" if bad == 0 else f"{bad} mismatches")
