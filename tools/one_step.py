"""Run one small step (debug aid for compute-sanitizer)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2506_22035_b200 as sp
d = int(sys.argv[1]) if len(sys.argv) > 1 else 2
r = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n = 2 * r + 1
if d == 3:
    k = sp.make_kernel_3d("box", r, np.full(n**3, 1.0 / n**3)); g = sp.random_grid_3d(8, 16, 128, r, seed=0)
else:
    k = sp.make_kernel("box", d, r, np.full(n**d, 1.0 / n**d)); g = sp.random_grid(1 if d == 1 else 64, 512, r, seed=0)
out, st = sp.execute(k, g, 1)
print("ok", out.interior.shape, float(np.abs(out.interior).max()))
