"""Benchmark of the SPIDER hot path on B200 (contract: DESIGN.md §6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config B9|B49|B27|B25|W|S5]
                    [--impl ours|reference] [--no-cpu-baseline] [--no-e2e] [--no-configs]

One bench "step" = one pass of the configuration over its grid: T Jacobi
timesteps of the stencil (T = 100 for B9/B27/B49/W).  Per GPU the grid is the
configuration's grid (weak scaling: N ranks own N slabs of that size, stacked
along y / z, with one halo exchange per timestep).  Metric: GStencil/s =
points x timesteps / device time, whole job (all ranks), max over ranks.

`--gpus N` with no launcher environment (WORLD_SIZE unset) starts the N ranks
itself (one process per GPU, 127.0.0.1 rendezvous); under torchrun it uses the
launcher's ranks.  The default line (B9) carries a `configs` block with the
other BASELINE configurations (B49, B27, W; at N > 1 the W weak-scaling
configuration) measured in the same run.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle's C port of naive_apply, all host threads) on the same config.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
# measured alongside the headline configuration in the default run
SIDE_CONFIGS = {1: ("B49", "B27", "W"), "multi": ("W",)}


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


def workload_config(cfg_name: str, world: int) -> dict:
    """The workload description both arms print (`config`)."""
    desc, shape, d, r, kind, T = CONFIGS[cfg_name]
    dense = tuple(s + 2 * r for s in shape)
    return {"workload": cfg_name, "description": desc, "grid_per_gpu": list(shape), "timesteps_per_step": T,
            "parallelism": f"slab{world}" if world > 1 else "single",
            "l2": f"inputs larger than L2 ({2 * np.prod(dense) / 2**20:.0f} MiB per fp16 buffer)"}


# ---------------------------------------------------------------------------
# clocks sampling (NVML during the timed region)

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
        self.power, self.limit, self.bits = [], None, 0
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
                self.bits |= bits
                for name, bit in self.REASONS.items():
                    if bits & bit:
                        self.reasons.add(name)
                self.power.append(nv.nvmlDeviceGetPowerUsage(h) / 1000.0)
                if self.limit is None:
                    self.limit = nv.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
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
                "samples": len(self.sm), "source": "nvml",
                "power_w": round(statistics.median(self.power), 1) if self.power else None,
                "power_limit_w": self.limit, "reason_bits": hex(self.bits),
                "power_note": "NVML board power, averaged over ~1 s: lags timed regions shorter than that "
                              "(sustained stepping sits at the limit, profiles/r02_power.txt)"}


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
# CPU reference algorithm (oracle C port of naive_apply, all host threads)

def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_runner(cfg_name: str):
    """Resident two-buffer fp64 grid of the workload for the C port."""
    from oracle import cnaive

    desc, shape, d, r, kind, T = CONFIGS[cfg_name]
    rng = np.random.default_rng(0)
    dense = rng.uniform(-1, 1, tuple(s + 2 * r for s in shape))
    threads = cpu_threads()
    return cnaive.NaiveRunner(coefficients(kind, d, r), d, r, dense, r, threads=threads), threads


def cpu_reference_rate(cfg_name: str, budget_s: float = 10.0):
    """GStencil/s of the oracle C port on a bounded sample of the workload:
    the full grid, as many timesteps as fit in ~budget_s (>= 1), buffers
    allocated and warmed before timing."""
    desc, shape, d, r, kind, T = CONFIGS[cfg_name]
    runner, threads = cpu_runner(cfg_name)
    points = int(np.prod(shape))
    t0 = time.perf_counter()
    runner.run(1)  # warm: page-faults both buffers, spins up the threads
    t1 = time.perf_counter() - t0
    steps = max(1, min(T, int(budget_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    runner.run(steps)
    el = time.perf_counter() - t0
    return points * steps / el / 1e9, threads, f"{shape} grid x {steps} timestep(s), {el:.2f} s wall, fp64"


def run_reference(args, cfg_name):
    """Reference arm: one bench step = the workload's T timesteps over the
    full grid (same work per step as our arm), on two resident fp64 buffers.
    Warm-up steps run one timestep each (buffer page-in, thread spin-up)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    desc, shape, d, r, kind, T = CONFIGS[cfg_name]
    runner, threads = cpu_runner(cfg_name)
    points = int(np.prod(shape))
    for _ in range(args.warmup):
        runner.run(1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        runner.run(T)
    el = time.perf_counter() - t0
    world = int(os.environ.get("WORLD_SIZE", "1"))
    # whole-job work of the configuration at N GPUs (weak scaling: N grids),
    # done by the host cores on rank 0
    value = points * T * args.steps / el / 1e9
    sample = (f"{shape} grid x {T} timesteps per step ({args.steps} steps, resident buffers), fp64, "
              f"{cpu_model()}")
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
        "config": workload_config(cfg_name, world),
        "cpu_baseline": {"value": round(value, 5), "unit": "GStencil/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 5), "unit": "GStencil/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm

class Ctx:
    """Per-process distributed context."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={self.world}")
        # SPD_BENCH_BACKEND=gloo lets several ranks share one GPU (functional
        # checks of the multi-rank path on a 1-GPU box; timings then mean nothing)
        self.backend = os.environ.get("SPD_BENCH_BACKEND", "nccl")
        self.local = local % torch.cuda.device_count()
        torch.cuda.set_device(self.local)
        if self.world > 1:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(self.backend)
        self.dist = dist

    def barrier(self):
        if self.world > 1:
            if self.backend == "nccl":
                self.dist.barrier(device_ids=[self.local])
            else:
                self.dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        import torch

        if self.world == 1:
            return v
        t = torch.tensor([v], device="cuda" if self.backend == "nccl" else "cpu", dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


def measure(ctx: Ctx, args, cfg_name: str, exchange: str) -> dict:
    """Device-timed throughput of one configuration (all ranks)."""
    import torch

    import paper_2506_22035_b200 as sp
    from paper_2506_22035_b200.engine import DeviceGrid
    from paper_2506_22035_b200.pipeline import get_plan

    world, rank = ctx.world, ctx.rank
    desc, shape, d, r, kind, T = CONFIGS[cfg_name]
    kern = make_kernel(kind, d, r)
    plan = get_plan(kern, sp.Parity.EVEN, "fp16", ctx.local)
    info = plan.info()
    points_local = int(np.prod(shape))
    stream = torch.cuda.current_stream()
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    dense_shape = tuple(s + 2 * r for s in shape)
    peer = None
    slab_mode = world > 1 or args.force_slab
    if not slab_mode:
        grid = DeviceGrid(plan, shape, r)
        dense = torch.rand(dense_shape, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
        grid.load_dense_f64(dense)
        del dense
        launches_per_step = T
        if args.graph:
            graph = torch.cuda.CUDAGraph()
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
            # overlap through programmatic dependent launch
            def one_step():
                grid.run(T)
    else:
        from paper_2506_22035_b200.distributed import DeviceSlabOps, PeerSlab, Slab, SlabDriver

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
        if exchange == "peer":
            # halos through peer memory (CUDA IPC + stream memory operations):
            # one host call and one launch per timestep, no NCCL on the data path
            try:
                peer = PeerSlab(plan, slab, ops.grid, compute_stream=stream, comm_stream=comm)
                # spd_slab_step: one edge-first launch per timestep for small 2D slabs,
                # an edge launch + an interior launch for 3D and large slabs (csrc/peer.cu)
                tiles = -(-shape[-1] // (info.n_tile * info.L)) * -(-shape[-2 if d >= 2 else -1] // info.tile_y)
                if d == 3:
                    tiles *= -(-shape[0] // info.tile_z)
                env = os.environ.get("SPD_SLAB_TWO_LAUNCH")
                two = bool(int(env)) if env else (d == 3 or tiles >= 10000)
                launches_per_step = T * (2 if two else 1)
            except Exception as exc:  # IPC / peer access unavailable: NCCL send/recv driver (all ranks)
                print(f"peer exchange unavailable ({exc}); using NCCL send/recv", file=sys.stderr)
                exchange = "nccl"

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
    ctx.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(ctx.local) as clk:
        torch.cuda.synchronize()
        ctx.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            one_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ctx.barrier()
    ms = ctx.max_over_ranks(e0.elapsed_time(e1))
    value = world * points_local * T * args.steps / (ms / 1e3) / 1e9

    # roofline of the dominant kernel (the step kernel): algorithmic 4 B per
    # point per timestep (fp16 read + write); in one-grid mode
    # the timed region is nothing but the T x K step launches on this stream
    hbm, peak_kind = measured_peaks()
    n_launch = args.steps * T
    launch_s = (ms / 1e3) / n_launch
    achieved = 4.0 * points_local / launch_s / 1e9
    traffic, traffic_src = ncu_traffic(cfg_name)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": 4 * points_local,
                "avg_launch_us": round(launch_s * 1e6, 2),
                "timing": ("step kernel launches only" if not slab_mode else
                           "slab steps (step kernel + halo exchange) per timestep"),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})", "traffic_source": traffic_src}
    if peer is not None:
        ctx.barrier()
        peer.close()
    res = {"value": round(value, 2), "ms_per_step": round(ms / args.steps, 4), "roofline": roofline,
           "clocks": clk.summary(), "gpu_launches": args.steps * launches_per_step,
           "impl_detail": {"launch": "cuda-graph" if args.graph else "stream, programmatic dependent launch",
                           "exchange": exchange if slab_mode else None,
                           "tile": {"L": info.L, "n_tile": info.n_tile, "mmas_per_tile": info.mmas_per_tile,
                                    "m_tiles": info.m_tiles}}}
    del plan
    torch.cuda.empty_cache()
    return res


def run_ours(args, cfg_name):
    import torch

    import paper_2506_22035_b200 as sp

    ctx = Ctx(args)
    world, rank = ctx.world, ctx.rank
    desc, shape, d, r, kind, T = CONFIGS[cfg_name]
    head = measure(ctx, args, cfg_name, args.exchange)

    side = {}
    if not args.no_configs and cfg_name == "B9":
        for name in SIDE_CONFIGS[1 if world == 1 else "multi"]:
            side[name] = measure(ctx, args, name, args.exchange)
            side[name]["config"] = workload_config(name, world)

    # end to end through the public API: pinned host fp16 grid in, result out.
    # At N > 1 the whole job's grid (N slabs of the per-GPU grid) goes through
    # one execute(..., DeviceConfig(devices=...)) call on rank 0, after the
    # other ranks have left (they hold no GPU work while it runs).
    e2e = None
    if world > 1:
        ctx.barrier()
        ctx.dist.destroy_process_group()
        if rank != 0:
            return 0
    if rank == 0 and not args.no_e2e and not args.force_slab:
        points_local = int(np.prod(shape))
        glob = (shape[0] * world,) + tuple(shape[1:])
        dense_shape = tuple(s + 2 * r for s in glob)
        devices = None if world == 1 else tuple(k % torch.cuda.device_count() for k in range(world))
        try:
            e2e = e2e_rate(sp, make_kernel(kind, d, r), d, r, dense_shape, T, points_local * world,
                           args.e2e_callers if world == 1 else 1, max(2, min(args.steps, 4)), devices)
        except Exception as exc:  # keep the device-timed line; say why e2e is missing
            if world == 1:
                raise
            e2e = {"value": None, "unit": "GStencil/s", "error": f"{type(exc).__name__}: {exc}"[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample = cpu_reference_rate(cfg_name)
        cpu = {"value": round(v, 5), "unit": "GStencil/s", "cores": cores, "kind": "port",
               "sample": sample + f", {cpu_model()}"}

    if rank == 0:
        line = {
            "metric": f"GStencil/s ({desc})",
            "value": head["value"],
            "unit": "GStencil/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": head["ms_per_step"],
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "fp16",
            "data": "synthetic U(-1,1) grid, contractive normalised weights (random init)",
            "config": workload_config(cfg_name, world),
            "impl_detail": head["impl_detail"],
            "roofline": head["roofline"],
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": head["gpu_launches"],
            "clocks": head["clocks"],
        }
        if side:
            line["configs"] = side
        print(json.dumps(line), flush=True)
    return 0


def e2e_rate(sp, kern, d, r, dense_shape, T, points, callers, calls_per_caller, devices=None):
    """End-to-end GStencil/s through `sp.execute` with host buffers.  Every
    call is a full execute() (H2D of its grid, T steps, D2H of the result);
    `callers` host threads issue calls concurrently, each on its own CUDA
    stream with its own pinned buffers, so one call's copies overlap another's
    steps (PCIe is full duplex) -- the way a server drives the engine.  Wall
    clock over all calls; the one-caller figure is kept too.  `devices`: the
    multi-GPU form, execute(..., DeviceConfig(devices=devices)) (one caller).
    """
    import torch

    cfg = sp.DeviceConfig(devices=devices) if devices is not None else sp.DeviceConfig()

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
                    sp.execute(kern, g_in, T, cfg, out=g_out)  # warm (allocator, stream, grid cache)
                    start.wait()
                    for _ in range(n_calls):
                        sp.execute(kern, g_in, T, cfg, out=g_out)
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
    # concurrent callers: twice the calls per caller, so the ramp-up and the
    # last call running alone weigh less in the wall-clock window
    nc, wc = timed(callers, 2 * calls_per_caller) if callers > 1 else (n1, w1)
    value = points * T * nc / wc / 1e9
    return {"value": round(value, 3), "unit": "GStencil/s", "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes, "ms_per_step": round(wc / nc * 1e3, 3),
            "callers": callers, "calls": nc, "timing": "host wall clock over all calls",
            "single_caller": {"value": round(single, 3), "ms_per_step": round(w1 / n1 * 1e3, 3)},
            "api": ("paper_2506_22035_b200.execute(kernel, Grid(pinned fp16), T, "
                    + (f"DeviceConfig(devices={tuple(devices)}), " if devices is not None else "")
                    + "out=Grid(pinned fp16))")}


# ---------------------------------------------------------------------------
# self-launch of N ranks (no torchrun in the environment)

def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """Re-run this command as n rank processes (RANK/LOCAL_RANK/WORLD_SIZE,
    127.0.0.1 rendezvous); rank 0's stdout carries the JSON line."""
    port = str(_free_port())
    procs = []
    for rank in range(n):
        env = dict(os.environ, RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve()), *sys.argv[1:]], env=env))
    rcs = [p.wait() for p in procs]
    bad = [rc for rc in rcs if rc != 0]
    return bad[0] if bad else 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="B9", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the side configurations block")
    ap.add_argument("--e2e-callers", type=int, default=3,
                    help="host threads issuing concurrent execute() calls in the e2e measurement")
    ap.add_argument("--force-slab", action="store_true", help="use the multi-GPU slab driver even at N=1")
    ap.add_argument("--graph", action="store_true", help="replay the T step launches as one CUDA graph")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="N>1 halo exchange: peer memory (CUDA IPC, default) or NCCL send/recv")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference(args, args.config)
    return run_ours(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
