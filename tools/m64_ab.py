"""One arm of an A/B between library builds (SPD_LIB=...; e.g. the all-M = 128
build of tools/build_variant.sh nom64 -DSPD_NO_M64): result hash, short-run
step time at full clock (after a cool-down) and sustained energy / time per
step under the board power cap.
usage: [SPD_LIB=...] python tools/m64_ab.py [seconds] CONFIG..."""
import os
import hashlib
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import pynvml
import torch
import bench
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid, Plan

args = sys.argv[1:]
secs = float(args.pop(0)) if args and args[0].replace(".", "").isdigit() else 3.0
pynvml.nvmlInit()
nv = pynvml.nvmlDeviceGetHandleByIndex(0)


def short(g, T):
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
    return best


def sustained(g, T):
    time.sleep(1.5)
    g.run(T)
    torch.cuda.synchronize()
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
    mj = (pynvml.nvmlDeviceGetTotalEnergyConsumption(nv) - e_start)  # mJ
    return e0.elapsed_time(e1) * 1e3 / n, mj / n, pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM)


tag = os.path.basename(os.environ.get("SPD_LIB", "libspider.so"))
for name in args or ["B9", "B27"]:
    desc, shape, d, r, kind, T = bench.CONFIGS[name]
    plan = Plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
    g = DeviceGrid(plan, shape, r)
    gen = torch.Generator(device="cuda").manual_seed(7)
    g.load_dense_f64(torch.rand(g.dense_shape, dtype=torch.float64, device="cuda", generator=gen) - 0.5)
    g.run(T)
    torch.cuda.synchronize()
    h = hashlib.sha1(g.bufs[g.cur].cpu().numpy().tobytes()).hexdigest()[:12]
    try:
        halves = "".join(str(int(v)) for v in plan.mma_halves())
    except Exception:  # a library from before spd_plan_mma_halves
        halves = "-"
    us = short(g, T)
    sus, mj, clk = sustained(g, T)
    pts = 1
    for v in shape:
        pts *= v
    print(f"{name} {tag:22s} halves {halves:16s} hash {h}: short {us:7.2f} us/step ({pts / us / 1e3:7.1f} GStencil/s)"
          f" | sustained {sus:7.2f} us/step ({pts / sus / 1e3:7.1f}) {mj:6.1f} mJ/step at {clk} MHz", flush=True)
