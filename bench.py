"""Benchmark of the SPIDER hot path on B200 (contract: see DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config B9|B49|B27|B25|W|S5]
                    [--impl ours|reference] [--no-cpu-baseline]

One bench "step" = one pass of the configuration over its grid: T Jacobi
timesteps of the stencil (T = 100 for B9/B27/B49/W).  Per GPU the grid is the
configuration's grid (weak scaling: N ranks own N slabs of that size, stacked
along y / z, with one NCCL halo exchange per timestep).  Metric: GStencil/s =
points x timesteps / device time, whole job (all ranks), max over ranks.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle's C port of naive_apply, all host threads) on the same config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (description, shape, d, r, kind, timesteps)
    "S5": ("Star-2D5P (Heat-2D) fp16 512x512, 4 timesteps", (512, 512), 2, 1, "heat2d", 4),
    "B9": ("Box-2D9P fp16 10240x10240, 100 timesteps", (10240, 10240), 2, 1, "box", 100),
    "B49": ("Box-2D49P (7x7) fp16 10240x10240, 100 timesteps", (10240, 10240), 2, 3, "box", 100),
    "B27": ("Box-3D27P fp16 512^3, 100 timesteps", (512, 512, 512), 3, 1, "box", 100),
    # the paper's Box-2D2R ablation stencil; width a multiple of L = 6
    "B25": ("Box-2D25P (5x5) fp16 10240x10242, 100 timesteps", (10240, 10242), 2, 2, "box", 100),
    "W": ("Box-2D9P fp16 16384x16384 per GPU, 100 timesteps", (16384, 16384), 2, 1, "box", 100),
}


def coefficients(kind: str, d: int, r: int, seed: int = 1):
    """Contractive weights so fp16 survives 100 steps."""
    n = 2 * r + 1
    if kind == "heat2d":
        c = np.zeros((3, 3))
        a = 0.125
        c[1, 1] = 1 - 4 * a
        c[0, 1] = c[2, 1] = c[1, 0] = c[1, 2] = a
        return c
    u = np.random.default_rng([seed, d, r, 100]).uniform(0.5, 1.5, (n,) * d)
    return u / u.sum()


def make_kernel(kind, d, r):
    import paper_2506_22035_b200 as sp

    c = coefficients(kind, d, r)
    shape = "star" if kind.startswith("heat") else "box"
    return sp.make_kernel_3d(shape, r, c) if d == 3 else sp.make_kernel(shape, d, r, c)


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)

class ClockSampler:
    """Samples SM clock and throttle reasons through NVML (every 10 ms) while
    the timed region runs (the bench's clocks line)."""

    REASONS = {  # nvml clocks-event-reason bits
        "hw_slowdown": 0x8,
        "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40,
        "sw_power_cap": 0x4,
    }

    def __init__(self, device: int, period: float = 0.01):
        self.device = device
        self.period = period
        self.sm, self.maxsm, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._thread = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        except Exception:
            self._thread = None
        return self

    def _run(self):
        nv, h = self._nvml, self._h
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                self.maxsm.append(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, bit in self.REASONS.items():
                    if bits & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "nvml"}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.maxsm), "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml"}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config: str):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        v = d.get(config)
        if isinstance(v, dict):
            return v.get("dram_bytes_per_launch"), v.get("source")
    return None, None


# ---------------------------------------------------------------------------
# CPU baseline (reference algorithm, oracle C port, all host threads)

def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_reference_rate(cfg_name: str, budget_s: float = 10.0):
    """GStencil/s of the oracle C port on a bounded sample of the workload:
    the full grid, as many timesteps as fit in ~budget_s (>= 1)."""
    from oracle import cnaive

    desc, shape, d, r, kind, T = CONFIGS[cfg_name]
    coeffs = coefficients(kind, d, r)
    rng = np.random.default_rng(0)
    dense = rng.uniform(-1, 1, tuple(s + 2 * r for s in shape))
    threads = cpu_threads()
    points = int(np.prod(shape))
    t0 = time.perf_counter()
    cnaive.naive_apply(coeffs, d, r, dense, r, 1, threads=threads)
    t1 = time.perf_counter() - t0
    steps = max(1, min(T, int(budget_s / max(t1, 1e-6))))
    if steps > 1:
        t0 = time.perf_counter()
        cnaive.naive_apply(coeffs, d, r, dense, r, steps, threads=threads)
        t1 = time.perf_counter() - t0
    else:
        steps = 1
    return points * steps / t1 / 1e9, threads, f"{shape} grid x {steps} timestep(s), {t1:.2f} s wall, fp64"


def cpu_model():
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------

def run_reference(args, cfg_name):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    desc, shape, d, r, kind, T = CONFIGS[cfg_name]
    from oracle import cnaive

    coeffs = coefficients(kind, d, r)
    rng = np.random.default_rng(0)
    dense = rng.uniform(-1, 1, tuple(s + 2 * r for s in shape))
    threads = cpu_threads()
    points = int(np.prod(shape))
    # one bench step = `ts` timesteps over the full grid in one call (a
    # bounded sample of the T-timestep workload, ~5e8 point updates, so the
    # per-call grid copies of the C port are amortised like the workload's)
    ts = max(1, min(T, int(round(5e8 / points))))
    for _ in range(args.warmup):
        cnaive.naive_apply(coeffs, d, r, dense, r, ts, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cnaive.naive_apply(coeffs, d, r, dense, r, ts, threads=threads)
    el = time.perf_counter() - t0
    value = points * ts * args.steps / el / 1e9
    sample = f"{shape} grid x {ts} timestep(s) per step ({args.steps} steps), fp64, {cpu_model()}"
    line = {
        "impl": "reference",
        "metric": f"GStencil/s ({desc})",
        "value": round(value, 5),
        "unit": "GStencil/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic U(-1,1) grid, contractive normalised weights",
        "config": {"workload": cfg_name, "description": desc, "grid": list(shape), "timesteps": T},
        "cpu_baseline": {"value": round(value, 5), "unit": "GStencil/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 5), "unit": "GStencil/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, cfg_name):
    import torch
    import torch.distributed as dist

    import paper_2506_22035_b200 as sp
    from paper_2506_22035_b200.engine import DeviceGrid
    from paper_2506_22035_b200.pipeline import get_plan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # SPD_BENCH_BACKEND=gloo lets several ranks share one GPU (functional
    # checks of the multi-rank path on a 1-GPU box; timings then mean nothing)
    backend = os.environ.get("SPD_BENCH_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    desc, shape, d, r, kind, T = CONFIGS[cfg_name]
    kern = make_kernel(kind, d, r)
    plan = get_plan(kern, sp.Parity.EVEN, "fp16", local)
    info = plan.info()
    points_local = int(np.prod(shape))
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    dense_shape = tuple(s + 2 * r for s in shape)
    peer = None
    if world == 1 and not args.force_slab:
        grid = DeviceGrid(plan, shape, r)
        dense = torch.rand(dense_shape, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
        grid.load_dense_f64(dense)
        del dense
        launches_per_step = T
        if args.graph:
            graph = torch.cuda.CUDAGraph()
            # capture T steps (an even T keeps the buffer parity fixed per replay)
            s = torch.cuda.Stream()
            s.wait_stream(stream)
            with torch.cuda.stream(s):
                grid.run(T)  # warm the kernel attributes outside capture
            stream.wait_stream(s)
            torch.cuda.synchronize()
            with torch.cuda.graph(graph):
                grid.run(T)

            def one_step():
                graph.replay()
        else:
            # T step kernels straight into the stream: consecutive launches
            # overlap through programmatic dependent launch (measured faster
            # than a CUDA-graph replay of the same T launches)
            def one_step():
                grid.run(T)
    else:
        from paper_2506_22035_b200.distributed import DeviceSlabOps, Slab, SlabDriver

        ops = DeviceSlabOps(plan, shape, r)
        dense = torch.rand(dense_shape, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
        ops.grid.load_dense_f64(dense)
        del dense
        extent = shape[0]
        slab = Slab(rank, world, rank * extent, (rank + 1) * extent)
        comm = torch.cuda.Stream()
        drv = SlabDriver(slab, ops, comm_stream=comm, compute_stream=stream)
        boundary, interior = drv._bands()
        launches_per_step = T * (len(boundary) + len(interior))
        if args.exchange == "peer":
            # halos through peer memory (CUDA IPC + stream memory operations):
            # one host call per timestep, no NCCL on the data path
            from paper_2506_22035_b200.distributed import PeerSlab

            try:
                peer = PeerSlab(plan, slab, ops.grid, compute_stream=stream, comm_stream=comm)
            except Exception as exc:  # IPC unavailable: NCCL send/recv driver
                print(f"peer exchange unavailable ({exc}); using NCCL send/recv", file=sys.stderr)
                args.exchange = "nccl"

        def one_step():
            if peer is not None:
                for _ in range(T):
                    peer.step()
            else:
                for _ in range(T):
                    drv.step()

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            one_step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda" if backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = world * points_local * T * args.steps / (ms / 1e3) / 1e9

    # roofline of the dominant kernel (the step kernel): algorithmic 4 B per
    # point per timestep (fp16 read + write), SURVEY.md §8(d)
    hbm, peak_kind = measured_peaks()
    n_launch = args.steps * T
    slab_mode = world > 1 or args.force_slab
    launch_s = (ms / 1e3) / n_launch if not slab_mode else None
    if not slab_mode:
        achieved = 4.0 * points_local / launch_s / 1e9
    else:
        achieved = 4.0 * points_local * T * args.steps / (ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(cfg_name)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": 4 * points_local,
                "avg_launch_us": round(launch_s * 1e6, 2) if launch_s else None,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})", "traffic_source": traffic_src}

    # end to end through the public API: pinned host fp16 grid in, result out.
    # Every call is a full execute() (H2D of its grid, T steps, D2H of the
    # result); `callers` host threads issue calls concurrently, each on its own
    # CUDA stream with its own pinned buffers, so one call's copies overlap
    # another's steps (PCIe is full duplex) -- the way a server drives the
    # engine.  Wall-clock over all calls; the one-caller figure is kept too.
    e2e = None
    if rank == 0 and world == 1 and not args.no_e2e and not args.force_slab:
        e2e = e2e_rate(sp, kern, d, r, dense_shape, T, points_local, args.e2e_callers,
                       max(2, min(args.steps, 4)))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample = cpu_reference_rate(cfg_name)
        cpu = {"value": round(v, 5), "unit": "GStencil/s", "cores": cores, "kind": "port",
               "sample": sample + f", {cpu_model()}"}

    if rank == 0:
        slab = "x".join(str(s) for s in shape)
        line = {
            "metric": f"GStencil/s ({desc})",
            "value": round(value, 2),
            "unit": "GStencil/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "fp16",
            "data": "synthetic U(-1,1) grid, contractive normalised weights (random init)",
            "config": {"workload": cfg_name, "description": desc, "grid_per_gpu": list(shape),
                       "timesteps_per_step": T, "parallelism": f"slab{world}" if slab_mode else "single",
                       "launch": "cuda-graph" if args.graph else "stream, programmatic dependent launch",
                       "exchange": (args.exchange if slab_mode else None),
                       "l2": f"inputs larger than L2 ({2 * np.prod(dense_shape) / 2**20:.0f} MiB per buffer)",
                       "tile": {"L": info.L, "n_tile": info.n_tile, "mmas_per_tile": info.mmas_per_tile},
                       "slab": slab},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": n_launch if not slab_mode else args.steps * launches_per_step,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if peer is not None:
        barrier()
        peer.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_rate(sp, kern, d, r, dense_shape, T, points, callers, calls_per_caller):
    """End-to-end GStencil/s through `sp.execute` with host buffers (see main)."""
    import numpy as np
    import torch

    cls = sp.Grid3D if d == 3 else sp.Grid
    bufs = []
    for i in range(max(1, callers)):
        host_in = torch.empty(dense_shape, dtype=torch.float16, pin_memory=True)
        host_in.copy_((torch.rand(dense_shape, dtype=torch.float32) * 2 - 1).half())
        host_out = torch.empty_like(host_in, pin_memory=True)
        bufs.append((cls(host_in.numpy(), r), cls(host_out.numpy(), r)))
    nbytes = int(np.prod(dense_shape)) * 2

    def timed(n_callers, n_calls):
        streams = [torch.cuda.Stream() for _ in range(n_callers)]
        start = threading.Barrier(n_callers + 1)
        errors = []

        def worker(i):
            try:
                with torch.cuda.stream(streams[i]):
                    g_in, g_out = bufs[i]
                    sp.execute(kern, g_in, T, out=g_out)  # warm (allocator, stream)
                    start.wait()
                    for _ in range(n_calls):
                        sp.execute(kern, g_in, T, out=g_out)
            except BaseException as exc:  # surface worker failures
                errors.append(exc)
                start.abort()

        threads = [threading.Thread(target=worker, args=(i,)) for i in range(n_callers)]
        for t in threads:
            t.start()
        try:
            start.wait()
        except threading.BrokenBarrierError:
            pass  # a worker failed; its exception is re-raised below
        t0 = time.perf_counter()
        for t in threads:
            t.join()
        wall = time.perf_counter() - t0
        if errors:
            raise errors[0]
        return n_callers * n_calls, wall

    n1, w1 = timed(1, calls_per_caller)
    single = points * T * n1 / w1 / 1e9
    nc, wc = timed(callers, calls_per_caller) if callers > 1 else (n1, w1)
    value = points * T * nc / wc / 1e9
    return {"value": round(value, 3), "unit": "GStencil/s", "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes, "ms_per_step": round(wc / nc * 1e3, 3),
            "callers": callers, "calls": nc, "timing": "host wall clock over all calls",
            "single_caller": {"value": round(single, 3), "ms_per_step": round(w1 / n1 * 1e3, 3)},
            "api": "paper_2506_22035_b200.execute(kernel, Grid(pinned fp16), T, out=Grid(pinned fp16))"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="B9", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-callers", type=int, default=3,
                    help="host threads issuing concurrent execute() calls in the e2e measurement")
    ap.add_argument("--force-slab", action="store_true", help="use the multi-GPU slab driver even at N=1")
    ap.add_argument("--graph", action="store_true", help="replay the T step launches as one CUDA graph")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="N>1 halo exchange: peer memory (CUDA IPC, default) or NCCL send/recv")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args, args.config)
    return run_ours(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
