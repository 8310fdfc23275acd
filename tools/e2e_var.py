"""Run-to-run variation of bench.py's e2e measurement (3 concurrent callers and
one caller), with the streamed path on and off (SPD_STREAM_WINDOWS=0)."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import bench
import paper_2506_22035_b200 as sp

name = sys.argv[1] if len(sys.argv) > 1 else "B9"
desc, shape, d, r, kind, T = bench.CONFIGS[name]
dense = tuple(s + 2 * r for s in shape)
k = bench.make_kernel(kind, d, r)
for mode in ("", "0"):
    os.environ["SPD_STREAM_WINDOWS"] = mode
    for rep in range(3):
        e = bench.e2e_rate(sp, k, d, r, dense, T, int(np.prod(shape)), 3, 4)
        print(f"{name} streaming={'off' if mode == '0' else 'auto'} rep {rep}: 3 callers {e['value']:7.1f}  "
              f"1 caller {e['single_caller']['value']:7.1f} GStencil/s", flush=True)
