"""B27 with the default two-M-tile 3D geometry against SPD_PLAN_3D_MT3 (three
M-tiles per tile): result hashes (must match) plus short-run and sustained
time / energy per step, interleaved.  usage: python tools/mt3_ab.py [seconds] [CONFIG]
Needs the experiment build of profiles/r02_mt3.txt (the flag was reverted)."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import pynvml
import torch
import bench
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid, Plan, SPD_PLAN_3D_MT3

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
name = sys.argv[2] if len(sys.argv) > 2 else "B27"
pynvml.nvmlInit()
nv = pynvml.nvmlDeviceGetHandleByIndex(0)
desc, shape, d, r, kind, T = bench.CONFIGS[name]
kern = bench.make_kernel(kind, d, r)
pts = 1
for v in shape:
    pts *= v
arms = {}
for tag, flags in (("MT2", 0), ("MT3", SPD_PLAN_3D_MT3)):
    plan = Plan(kern, sp.Parity.EVEN, "fp16", flags=flags)
    g = DeviceGrid(plan, shape, r)
    gen = torch.Generator(device="cuda").manual_seed(7)
    g.load_dense_f64(torch.rand(g.dense_shape, dtype=torch.float64, device="cuda", generator=gen) - 0.5)
    g.run(T)
    torch.cuda.synchronize()
    arms[tag] = (plan, g)
# compare interiors (the two layouts pad planes differently)
a = arms["MT2"][1].to_dense_f64()
b = arms["MT3"][1].to_dense_f64()
print(f"{name}: MT2 vs MT3 bit-identical: {bool(torch.equal(a, b))}  (max |diff| {float((a - b).abs().max()):.3e})", flush=True)
del a, b
for rep in range(2):
    for tag in ("MT2", "MT3"):
        g = arms[tag][1]
        time.sleep(1.5)
        best = 1e9
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            g.run(T)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / T)
        time.sleep(1.5)
        e_start = pynvml.nvmlDeviceGetTotalEnergyConsumption(nv)
        t0 = time.perf_counter()
        n = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        while time.perf_counter() - t0 < secs:
            g.run(T)
            n += T
            torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        mj = (pynvml.nvmlDeviceGetTotalEnergyConsumption(nv) - e_start) / n
        sus = e0.elapsed_time(e1) * 1e3 / n
        clk = pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM)
        print(f"{name} {tag} rep {rep}: short {best:7.2f} us/step ({pts / best / 1e3:7.1f} GStencil/s) | sustained "
              f"{sus:7.2f} us/step ({pts / sus / 1e3:7.1f}) {mj:6.1f} mJ/step at {clk} MHz", flush=True)
