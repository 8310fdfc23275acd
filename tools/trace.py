"""Per-role timeline of CTA 0 for one step (needs SPD_TRACE=1)."""
import ctypes as C, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("SPD_TRACE", "1")
import numpy as np, torch
import bench, paper_2506_22035_b200 as sp
from paper_2506_22035_b200 import _lib
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan
name = sys.argv[1] if len(sys.argv) > 1 else "B9"
desc, shape, d, r, kind, T = bench.CONFIGS[name]
plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
g = DeviceGrid(plan, shape, r)
g.load_dense_f64(torch.rand(g.dense_shape, dtype=torch.float64, device="cuda") - 0.5)
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g.run(4, flags=flags); torch.cuda.synchronize()
buf = (C.c_ulonglong * (8 * 16 * 64))()
assert _lib.lib.spd_debug_trace(buf) == 0
a = np.array(buf, dtype=np.int64).reshape(8, 16, 64)[0]
names = ["ld_wait", "ld_issued", "pr_natfull", "pr_bempty", "pr0_done", "pr7_done", "mma_accfree", "mma_issue", "epi_start", "epi_done"]
t0 = a[13, 0]
print(f"entry->setup done {(a[14,0]-a[13,0])/1965:.2f} us, entry->exit {(a[15,0]-a[13,0])/1965:.2f} us, first load issued {(a[1,0]-a[13,0])/1965:.2f} us, first epi done {(a[9,0]-a[13,0])/1965:.2f} us")
print("tile " + " ".join(f"{n:>11s}" for n in names))
for it in list(range(4)) + list(range(38, 46)):
    if a[9, it] == 0: break
    print(f"{it:4d} " + " ".join(f"{(a[e, it]-t0)/1965:11.2f}" for e in range(10)))
n = 0
while n < 63 and a[9, n + 1] != 0: n += 1
per = (a[9, n] - a[9, 2]) / max(n - 2, 1) / 1965
print(f"avg tile period (epi_done) {per:.3f} us")
for e, nm in ((1, 'ld_issued'), (2, 'natfull'), (5, 'prod_done'), (7, 'mma'), (9, 'epi_done')):
    pass
lat = np.mean([(a[2, i] - a[1, i]) for i in range(3, n)]) / 1965
prod = np.mean([(a[5, i] - a[3, i]) for i in range(3, n)]) / 1965
epi = np.mean([(a[9, i] - a[8, i]) for i in range(3, n)]) / 1965
sub = [np.mean([(a[e1, i] - a[e0, i]) for i in range(3, n)]) / 1965 for e0, e1 in ((8, 10), (10, 11))]
gap = [np.mean([(a[e1, i + 1] - a[e0, i]) for i in range(3, n - 1)]) / 1965 for e0, e1 in ((9, 12), (12, 8))]
print(f"epilogue batch 0: tmem load {sub[0]:.3f} us, pack+transpose {sub[1]:.3f} us; between tiles: "
      f"loop {gap[0]:.3f} us, accumulator wait {gap[1]:.3f} us")
print(f"TMA issue->natfull {lat:.3f} us  producer (bempty->last warp done) {prod:.3f} us  epilogue {epi:.3f} us")
