"""Step time against SM clock and board power over a long run of one config
(is the sustained bench power-limited?).  Chunks of 100 steps, each timed with
CUDA events; NVML sampled every 5 ms.  usage: python tools/power_probe.py CONFIG [seconds]"""
import sys
import threading
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import pynvml
import torch
import bench
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan

name = sys.argv[1] if len(sys.argv) > 1 else "B9"
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
persistent = len(sys.argv) > 3 and sys.argv[3] == "persistent"
desc, shape, d, r, kind, T = bench.CONFIGS[name]
plan = get_plan(bench.make_kernel(kind, d, r), sp.Parity.EVEN, "fp16")
g = DeviceGrid(plan, shape, r)
g.load_dense_f64(torch.rand(g.dense_shape, dtype=torch.float64, device="cuda") - 0.5)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
                        pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)))
        time.sleep(0.005)


th = threading.Thread(target=sampler, daemon=True)
th.start()
print(f"{name}{' persistent' if persistent else ''}: power limit {pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1000:.0f} W",
      flush=True)
e_start = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
chunks = []
t_start = time.perf_counter()
while time.perf_counter() - t_start < secs:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.run(T, persistent=persistent)
    e1.record()
    e1.synchronize()
    chunks.append((time.perf_counter(), e0.elapsed_time(e1) * 1e3 / T))
stop.set()
th.join()
e_total = pynvml.nvmlDeviceGetTotalEnergyConsumption(h) - e_start  # mJ
print(f"energy {e_total / (len(chunks) * T):.2f} mJ per step over {len(chunks) * T} steps, "
      f"mean {sum(c[1] for c in chunks[len(chunks) // 2:]) / (len(chunks) - len(chunks) // 2):.1f} us/step (second half)",
      flush=True)
for i in range(0, len(chunks), max(1, len(chunks) // 25)):
    t, us = chunks[i]
    near = [s for s in samples if abs(s[0] - t) < 0.02]
    if near:
        clk = sorted(s[1] for s in near)[len(near) // 2]
        pw = sorted(s[2] for s in near)[len(near) // 2]
        bits = 0
        for s in near:
            bits |= s[3]
        print(f"t={t - t_start:6.3f}s  {us:6.1f} us/step  sm {clk} MHz  {pw:6.0f} W  reasons {bits:#x}  temp {near[-1][4]} C",
              flush=True)
