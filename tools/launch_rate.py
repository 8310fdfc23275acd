"""Per-launch device and host time of run(n) on a tiny (S5) and a large (B9) grid (dev aid)."""
import sys; sys.path.insert(0, '/root/repo')
import torch, bench, paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan
for name, steps in (("S5", 2000), ("B9", 100)):
    desc, shape, d, r, kind, T = bench.CONFIGS[name]
    plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
    g = DeviceGrid(plan, shape, r); g.load_dense_f64(torch.rand(g.dense_shape, dtype=torch.float64, device="cuda"))
    g.run(steps); torch.cuda.synchronize()
    import time
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(); g.run(steps); e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"{name}: device {e0.elapsed_time(e1)*1e3/steps:.2f} us/step, host wall {(t1-t0)*1e6/steps:.2f} us/step", flush=True)
