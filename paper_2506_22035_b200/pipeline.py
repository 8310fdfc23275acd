"""Drop-in execution API: transform_stencil / execute / naive_apply / verify.

Mirrors the reference engine surface (reference pipeline.py:42-333) with the
hot path moved to the B200:

* `transform_stencil` — the AOT transform per kernel row (C++ twin of
  transform.py, exact), same `TransformedStencil` result.
* `execute` — same signature and return type; the T-step loop runs on the
  sparse tensor cores (libspider.so, tcgen05.mma.sp).  Storage is fp16 (or
  bf16 via `DeviceConfig`) with fp32 accumulation.  `ExecConfig` keeps the
  reference's fields and its fp16 rejection; device precision is chosen by
  `DeviceConfig`.
* `naive_apply` — the brute-force executor, on the device in fp64 with the
  reference's tap order and separate multiply/add roundings: bit-identical to
  the reference's numpy oracle.
* `verify` — device `execute` against device `naive_apply` over seeded grids,
  same report keys.
"""
from __future__ import annotations

import json
import os
import threading
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from .accounting import MMA_M16N8K16, fetch_runs, tile_counts
from .core import Grid, Grid3D, StencilKernel, random_grid
from .engine import DeviceGrid, Plan, TORCH_DTYPES, naive_apply_device, require_cuda
from .transform import CompressedKernel, Parity, RowPermutation, band_rows, input_row_permutation, transform_row

_HOST_PRECISIONS = {"fp64": np.float64, "fp32": np.float32}

# fp16/bf16 storage tolerances on max|got-want|/max|want| for T <= 4 steps
# against the fp64 oracle on identically quantised inputs.
DEFAULT_TOLERANCE = {"fp16": 1e-2, "bf16": 5e-2}


@dataclass(frozen=True)
class ExecConfig:
    """Reference execution knobs (reference pipeline.py:42-63).

    Kept field-for-field so reference callers construct it unchanged; the
    device path reads `parity` from it and computes in fp16.
    """

    parity: Parity = Parity.EVEN
    a_block: int | None = None
    b_block: int | None = None
    a_warp: int = 16
    b_warp: int = 8
    mma: object = MMA_M16N8K16
    precision: str = "fp64"
    compute_mode: str = "ceil"
    packing: bool = True

    def __post_init__(self) -> None:
        if self.precision not in _HOST_PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(_HOST_PRECISIONS)}")
        object.__setattr__(self, "parity", Parity(self.parity))

    @property
    def dtype(self):
        return _HOST_PRECISIONS[self.precision]


@dataclass(frozen=True)
class DeviceConfig:
    """Device-path knobs: storage dtype of the grid on the B200 and parity.

    `devices`: run on several GPUs from this process -- the grid is cut into
    slabs along y (2D) / z (3D), one per listed device, with the halo rows
    exchanged through peer memory every step (distributed.LocalSlabs).  A
    device may be listed more than once (several slabs on one GPU).  Results
    are bit-identical to the one-device run."""

    parity: Parity = Parity.EVEN
    dtype: str = "fp16"
    device: int | None = None
    devices: tuple | None = None

    def __post_init__(self) -> None:
        if self.dtype not in TORCH_DTYPES:
            raise ValueError(f"device dtype must be one of {sorted(TORCH_DTYPES)}")
        object.__setattr__(self, "parity", Parity(self.parity))
        if self.devices is not None:
            devs = tuple(int(v) for v in self.devices)
            if not devs or any(v < 0 for v in devs):
                raise ValueError(f"bad device list {self.devices!r}")
            if self.device is not None and self.device != devs[0]:
                raise ValueError("give either device or devices")
            object.__setattr__(self, "devices", devs)


@dataclass
class ExecStats:
    """Execution counters.  The reference keys (pipeline.py:66-108) keep their
    algorithmic meaning (per kernel row and step, L x L compressed MACs per
    x-chunk); `device` adds what the B200 actually issued."""

    grid_a: int
    grid_b: int
    steps: int
    radius: int
    kernel_rows: int
    L: int
    parity: str
    packing: bool
    total_macs: int = 0
    dense_macs: int = 0
    input_elements: int = 0
    param_elements: int = 0
    mma_invocations: int = 0
    sparse_mma_calls: int = 0
    fetch_runs_packed: int = 0
    fetch_runs_unpacked: int = 0
    fetch_runs_active: int = 0
    tile_counts: dict = field(default_factory=dict)
    # B200 engine: tcgen05 instruction, tile geometry and issued work
    device: dict = field(default_factory=dict)

    def as_dict(self) -> dict:
        return {
            "grid": [self.grid_a, self.grid_b],
            "steps": self.steps,
            "radius": self.radius,
            "kernel_rows": self.kernel_rows,
            "L": self.L,
            "parity": self.parity,
            "packing": self.packing,
            "total_macs": self.total_macs,
            "dense_macs": self.dense_macs,
            "input_elements": self.input_elements,
            "param_elements": self.param_elements,
            "mma_invocations": self.mma_invocations,
            "sparse_mma_calls": self.sparse_mma_calls,
            "fetch_runs_packed": self.fetch_runs_packed,
            "fetch_runs_unpacked": self.fetch_runs_unpacked,
            "fetch_runs_active": self.fetch_runs_active,
            "tile_counts": dict(self.tile_counts),
            "device": dict(self.device),
        }


@dataclass
class TransformedStencil:
    r: int
    L: int
    parity: Parity
    rows: list
    permutation: RowPermutation


def _parity_of(cfg) -> Parity:
    if isinstance(cfg, (ExecConfig, DeviceConfig)):
        return cfg.parity
    return Parity(cfg)


def transform_stencil(kernel: StencilKernel, cfg=ExecConfig()) -> TransformedStencil:
    """One compressed kernel per kernel row (reference pipeline.py:128-144).

    3D kernels (extension) give one record per (rho_z, rho_y), row-major."""
    if kernel.d not in (1, 2, 3) or np.asarray(kernel.coeffs).ndim != kernel.d:
        raise ValueError(f"unsupported dimensionality {kernel.d}")
    parity = _parity_of(cfg)
    L = band_rows(kernel.r)
    rows = [(rho, transform_row(kernel.row(rho), kernel.r, parity)) for rho in kernel.row_offsets()]
    return TransformedStencil(r=kernel.r, L=L, parity=parity, rows=rows, permutation=input_row_permutation(L, parity))


# ---------------------------------------------------------------------------
# plan cache (one per kernel/parity/dtype/device)

_PLANS: dict = {}
_PLANS_LOCK = threading.Lock()


def get_plan(kernel: StencilKernel, parity: Parity, dtype: str, device: int | None = None) -> Plan:
    """Cached plan.  Plans are read-only once built, so `execute` may be
    called from several host threads at once (each on its own current CUDA
    stream), as the reference's pure functions may."""
    dev = require_cuda(device).index if device is None else int(device)
    key = (kernel.d, kernel.r, np.asarray(kernel.coeffs, dtype=np.float64).tobytes(), Parity(parity), dtype, dev,
           bool(os.environ.get("SPD_NO_EMBED")))  # the plan's geometry depends on it
    with _PLANS_LOCK:
        plan = _PLANS.get(key)
        if plan is None:
            plan = Plan(kernel, parity, dtype, dev)
            _PLANS[key] = plan
    return plan


def _device_cfg(cfg) -> DeviceConfig:
    if isinstance(cfg, DeviceConfig):
        return cfg
    if isinstance(cfg, ExecConfig):
        return DeviceConfig(parity=cfg.parity)
    return DeviceConfig(parity=Parity(cfg))


def _check_inputs(kernel: StencilKernel, grid, steps: int) -> None:
    if steps < 1:
        raise ValueError(f"step count must be >= 1, got {steps}")
    if grid.halo < kernel.r:
        raise ValueError(f"grid halo {grid.halo} too small for stencil radius {kernel.r}")
    if (kernel.d == 3) != isinstance(grid, Grid3D):
        raise ValueError("unsupported dimensionality: 3D kernels need a Grid3D and vice versa")
    L = band_rows(kernel.r)
    if grid.B % L != 0:
        raise ValueError(f"grid width {grid.B} must be a multiple of the x-chunk size L={L}")


def _exec_cfg(cfg) -> ExecConfig:
    """The reference-side config (tiling / instruction shape for the counters)."""
    if isinstance(cfg, ExecConfig):
        return cfg
    return ExecConfig(parity=_parity_of(cfg))


def _stats(kernel: StencilKernel, grid, steps: int, cfg, plan: Plan) -> ExecStats:
    """ExecStats with the reference's counter semantics (pipeline.py:200-259):
    per step and kernel row, L x L compressed MACs per x-chunk, the reference
    tile plan and fetch-run metric; `device` holds what the B200 issued."""
    ecfg = _exec_cfg(cfg)
    parity = _parity_of(cfg)
    L = band_rows(kernel.r)
    n_rows = len(list(kernel.row_offsets()))
    planes = grid.Z if isinstance(grid, Grid3D) else 1
    cols = planes * grid.A * (grid.B // L)
    mma = ecfg.mma
    n_groups = -(-cols // mma.n)
    inv_k = -(-2 * L // mma.k)
    m_groups = -(-L // mma.m)
    per = steps * n_rows
    st = ExecStats(
        grid_a=grid.A,
        grid_b=grid.B,
        steps=steps,
        radius=kernel.r,
        kernel_rows=n_rows,
        L=L,
        parity=parity.value,
        packing=ecfg.packing,
        tile_counts=tile_counts(min(kernel.d, 2), kernel.r, grid.A, grid.B, ecfg),
    )
    if isinstance(mma, type(MMA_M16N8K16)) and (mma.m, mma.n, mma.k) == (16, 8, 16):
        st.fetch_runs_packed, st.fetch_runs_unpacked, st.fetch_runs_active = fetch_runs(L, ecfg.packing, mma)
    st.total_macs = per * L * cols * L
    st.dense_macs = 2 * st.total_macs
    st.input_elements = per * 2 * L * cols
    st.param_elements = per * L * L * n_groups
    st.mma_invocations = per * m_groups * n_groups * inv_k
    st.sparse_mma_calls = per
    if plan is not None:
        info = plan.info()
        tiles_x = -(-grid.B // (info.n_tile * L)) if kernel.d != 1 else -(-grid.B // (info.n_tile * L * info.r_out))
        tiles = tiles_x * (-(-grid.A // info.tile_y) if kernel.d >= 2 else 1) * (-(-planes // info.tile_z))
        halves = plan.mma_halves()
        n64 = int(np.count_nonzero(halves))  # M = 64 half-lane MMAs per M-tile
        st.device = {
            "arch": "sm_100a",
            "instruction": "tcgen05.mma.sp.cta_group::1.kind::f16 M128|M64 N%d K32" % info.n_tile,
            "dtype": plan.dtype,
            "launches": steps,
            "tiles_per_step": tiles,
            "tile": {"n_tile": info.n_tile, "tile_rows": info.r_out * info.m_tiles, "tile_z": info.tile_z,
                     "input_rows": info.r_in, "mmas_per_tile": info.mmas_per_tile * info.m_tiles},
            "mma_instructions": steps * tiles * info.mmas_per_tile * info.m_tiles,
            "m64_instructions": steps * tiles * n64 * info.m_tiles,
            "issued_sparse_macs": steps * tiles * (info.mmas_per_tile * 128 - n64 * 64) * info.m_tiles * info.n_tile * 16,
        }
    return st


def exec_stats(kernel: StencilKernel, grid, steps: int, cfg=ExecConfig()) -> ExecStats:
    """The reference counters of `execute(kernel, grid, steps, cfg)` without
    running it (host only; `device` is empty)."""
    _check_inputs(kernel, grid, steps)
    return _stats(kernel, grid, steps, cfg, None)


class _GridPool:
    """Device grids kept between `execute` calls, per (plan, shape, halo).

    A call takes a free grid (or allocates one) and returns it when its
    result is on the host, so concurrent callers never share buffers and a
    repeated call skips the two zeroed allocations.  Nothing outside the dense
    region is ever written, so the zero padding the kernels rely on survives
    reuse.  `release_device_grids()` frees the cache."""

    def __init__(self, keep: int = 8):
        self.keep = keep
        self._free: dict = {}
        self._lock = threading.Lock()

    def acquire(self, plan: Plan, shape, halo: int) -> DeviceGrid:
        key = (id(plan), tuple(shape), int(halo))
        with self._lock:
            lst = self._free.get(key)
            if lst:
                return lst.pop()
        return DeviceGrid(plan, shape, halo)

    def release(self, dg: DeviceGrid) -> None:
        key = (id(dg.plan), tuple(dg.desc_shape), int(dg.halo))
        with self._lock:
            lst = self._free.setdefault(key, [])
            if len(lst) < self.keep:
                dg.cur, dg.step = 0, 0
                lst.append(dg)

    def clear(self) -> None:
        with self._lock:
            self._free.clear()


_GRIDS = _GridPool()


def release_device_grids() -> None:
    """Free the device grids cached between `execute` calls."""
    _GRIDS.clear()


# Streamed-execute cost model (per point): PCIe copy of an fp16 point one way
# (~55 GB/s pinned), one step of a point on the device (B9, full clock) and the
# fill / drain / tail of one step launch (profiles/r02_l2_probe.txt).  It
# reproduces the measured B9 window scan (profiles/r02_streamed_e2e.txt).
_COPY_PS_PER_POINT = 36.0
_STEP_PS_PER_POINT = 0.75
_LAUNCH_OVERHEAD_PS = 4.7e6


def _window_weights(windows: int) -> list:
    """Relative slab sizes: the first and the last window half the size of
    the others (their upload / download is the part no step hides), while a
    full window's upload still fits under the previous window's steps (a
    copied point costs ~48x a point-step, a window ~100 steps)."""
    if windows <= 2:
        return [1] * windows
    return [1] + [2] * (windows - 2) + [1]


def _stream_gain(extent: int, row_points: int, margin: int, steps: int, windows: int) -> float:
    """Modelled time saved (ps) by `windows` streamed windows over the
    whole-grid path: the copies of all but the first upload and the last
    download overlap the steps; every window recomputes its margin rows and
    pays its own launch fill and drain."""
    copies = 2 * extent * row_points * _COPY_PS_PER_POINT
    w = _window_weights(windows)
    saved = copies - copies / 2 * (w[0] + w[-1]) / sum(w)
    margins = steps * 2 * margin * (windows - 1) * row_points * _STEP_PS_PER_POINT
    launches = steps * (windows - 1) * _LAUNCH_OVERHEAD_PS
    return saved - margins - launches


def stream_windows(extent: int, band: int, steps: int, r: int, windows: int | None = None,
                   row_points: int = 10240) -> list:
    """Windows of a streamed execute (see `_execute_streamed`): a list of
    (slab_lo, slab_hi, win_lo, win_hi) in interior rows (2D) / planes (3D), or
    [] when streaming does not pay.

    The extent is cut into `windows` band-aligned slabs (the first and the
    last half the size of the others, `_window_weights`); window k is slab k
    widened by the margin M = T*r rounded up to whole tile bands (clipped to
    the grid).  After T steps the rows the window's frozen outer halo has
    contaminated lie within T*r of the window edge, outside the slab, and the
    band-aligned window keeps every tile where the whole-grid run has it, so
    the slab comes out bit-identical.  The default count maximises the
    modelled gain (`_stream_gain`, 2..8 windows, each at least two margins
    tall) and streams only when that gain is over 5 % of the whole-grid
    time; SPD_STREAM_WINDOWS overrides (B9, T = 100: 4 windows; 1000 steps:
    none)."""
    margin = -(-steps * r // band) * band
    units = -(-extent // band)
    if windows is None:
        env = os.environ.get("SPD_STREAM_WINDOWS")
        if env:
            windows = int(env)
        else:
            whole = 2 * extent * row_points * _COPY_PS_PER_POINT + steps * extent * row_points * _STEP_PS_PER_POINT
            best, windows = 0.05 * whole, 0
            for n in range(2, 9):
                if extent // n < 2 * margin:
                    break
                g = _stream_gain(extent, row_points, margin, steps, n)
                if g > best:
                    best, windows = g, n
    windows = min(int(windows), units)
    if windows < 2:
        return []
    w = _window_weights(windows)
    edges, acc = [0], 0
    for x in w:
        acc += x
        edges.append(units * acc // sum(w))
    out = []
    for k in range(windows):
        lo = edges[k] * band
        hi = min(extent, edges[k + 1] * band)
        if hi > lo:
            out.append((lo, hi, max(0, lo - margin), min(extent, hi + margin)))
    return out if len(out) >= 2 else []


_STREAMS = threading.local()


def _side_streams(device: int, n: int) -> list:
    """n CUDA streams of `device` owned by this host thread (reused across
    calls, so concurrent callers never share them)."""
    cache = getattr(_STREAMS, "by_dev", None)
    if cache is None:
        cache = _STREAMS.by_dev = {}
    lst = cache.setdefault(device, [])
    while len(lst) < n:
        lst.append(torch.cuda.Stream(device))
    return lst[:n]


def _execute_streamed(plan: Plan, kernel: StencilKernel, data: np.ndarray, halo: int, steps: int, windows: list,
                      target: torch.Tensor) -> None:
    """One-device execute with the host transfers overlapped with the steps.

    Each window (`stream_windows`) is an independent grid: its upload (copy
    stream), its T steps (compute stream) and the download of its slab rows
    (second copy stream) are chained by events, so window k+1's upload and
    window k-1's download run under window k's steps -- PCIe is full duplex
    and the copy engines are separate from the SMs.  The price is the margin
    rows every window recomputes; the result is bit-identical to the
    whole-grid run.  `target`: the dense host result (pinned for overlap)."""
    dense_shape = tuple(int(v) for v in data.shape)
    row_elems = int(np.prod(dense_shape[1:]))
    rest = tuple(v - 2 * halo for v in dense_shape[1:])
    host_in = torch.from_numpy(data)
    s_in, s_out, s_c = _side_streams(plan.device, 3)
    caller = torch.cuda.current_stream()
    for st in (s_in, s_out, s_c):
        st.wait_stream(caller)
    grids = []
    try:
        for k, (lo, hi, wl, wh) in enumerate(windows):
            g = _GRIDS.acquire(plan, (wh - wl,) + rest, halo)
            grids.append(g)
            g.upload(host_in[wl : wh + 2 * halo], stream=s_in)
            up = torch.cuda.Event()
            up.record(s_in)
            s_c.wait_event(up)
            g.run(steps, stream=s_c)
            done = torch.cuda.Event()
            done.record(s_c)
            s_out.wait_event(done)
            a = 0 if k == 0 else lo - wl + halo
            b = wh - wl + 2 * halo if k == len(windows) - 1 else hi - wl + halo
            g.download_rows(target.data_ptr() + wl * row_elems * 2, a, b, stream=s_out)
        caller.wait_stream(s_out)
        s_out.synchronize()
    finally:
        for g in grids:
            _GRIDS.release(g)


def execute(kernel: StencilKernel, grid, steps: int, cfg=ExecConfig(), *, out=None):
    """Run `steps` steps on the B200 sparse-tensor-core path; returns
    (Grid, ExecStats) like reference pipeline.py:189-262.  The input grid is
    never modified.

    float16 host grids are transferred as-is by DMA (pinned host memory gives
    asynchronous copies) and the result comes back as float16, into
    `out.data` when an `out` grid of the same shape is given (otherwise into a
    pinned buffer from torch's caching host allocator).  Other dtypes are
    quantised on the device and the result is returned as float64 (float32
    inputs give float32).  The work runs on the plan's device (DeviceConfig
    .device, default the current one), on that device's current stream.
    With `DeviceConfig(devices=(d0, d1, ...))` the grid is split into slabs
    across those devices (one host thread per slab, peer-memory halo
    exchange; distributed.LocalSlabs), same result bit for bit.
    """
    _check_inputs(kernel, grid, steps)
    dcfg = _device_cfg(cfg)
    devices = dcfg.devices if dcfg.devices is not None and len(dcfg.devices) > 1 else None
    first = dcfg.devices[0] if dcfg.devices is not None else dcfg.device
    plan = get_plan(kernel, dcfg.parity, dcfg.dtype, first)
    stats = _stats(kernel, grid, steps, cfg, plan)  # raises the reference's tile-plan errors first
    shape = (grid.Z, grid.A, grid.B) if kernel.d == 3 else (grid.A, grid.B)
    data = grid.data
    native16 = dcfg.dtype == "fp16" and data.dtype == np.float16
    if native16 and out is not None:
        if out.data.shape != data.shape or out.data.dtype != np.float16 or not out.data.flags.c_contiguous:
            raise ValueError("out grid must be a contiguous float16 array of the input's shape")
    if devices is not None:
        from .distributed import execute_slabs

        plans = {dev: get_plan(kernel, dcfg.parity, dcfg.dtype, dev) for dev in set(devices)}
        target = out.data if (native16 and out is not None) else None
        res = execute_slabs(plans, devices, shape, grid.halo, data, steps, native16, target)
        if not native16:
            if data.dtype == np.float32:
                res = res.astype(np.float32)
            if out is not None:
                out.data[...] = res
                res = out.data
        stats.device["devices"] = list(devices)
        stats.device["exchange"] = "peer memory (spd_slab_run), one slab per listed device"
        cls = Grid3D if kernel.d == 3 else Grid
        return cls(res, grid.halo, grid.step + steps), stats
    with _InFlight(plan.device) as concurrent:
        # Streamed windows pay off for a lone caller; with other calls in
        # flight on the device (now or within the last second) their copies
        # already overlap this call's steps, and the margin rows would only
        # add work.
        if native16 and kernel.d >= 2 and concurrent == 0:
            band = plan.info().tile_z if kernel.d == 3 else plan.info().tile_y
            windows = stream_windows(shape[0], band, steps, kernel.r, row_points=int(np.prod(shape[1:])))
            if windows:
                with torch.cuda.device(plan.device):
                    target = torch.from_numpy(out.data) if out is not None else torch.empty(
                        data.shape, dtype=torch.float16, pin_memory=True)
                    _execute_streamed(plan, kernel, np.ascontiguousarray(data), grid.halo, steps, windows, target)
                stats.device["streamed_windows"] = len(windows)
                cls = Grid3D if kernel.d == 3 else Grid
                return cls(target.numpy(), grid.halo, grid.step + steps), stats
        return _execute_whole(plan, kernel, grid, steps, shape, native16, out, stats)


class _InFlight:
    """Counts execute() calls in flight per device.  Entering returns how many
    other calls were running on it, or -1 when none is running now but calls
    overlapped within the last QUIET seconds: a caller among several
    concurrent ones (bench: three host threads, B9 whole-grid 1236-1255
    GStencil/s aggregate) loses throughput when one of its calls streams
    (1114-1217 with streaming allowed whenever a call found the device idle;
    tools/e2e_var.py)."""

    QUIET = 1.0
    _lock = threading.Lock()
    _count: dict = {}
    _last_overlap: dict = {}

    def __init__(self, device: int):
        self.device = device

    def __enter__(self) -> int:
        import time

        now = time.monotonic()
        with self._lock:
            n = self._count.get(self.device, 0)
            self._count[self.device] = n + 1
            if n > 0:
                self._last_overlap[self.device] = now
            elif now - self._last_overlap.get(self.device, -1e9) < self.QUIET:
                n = -1
        return n

    def __exit__(self, *exc) -> None:
        import time

        with self._lock:
            self._count[self.device] -= 1
            if self._count[self.device] > 0:
                self._last_overlap[self.device] = time.monotonic()


def _execute_whole(plan: Plan, kernel: StencilKernel, grid, steps: int, shape, native16: bool, out, stats):
    """Whole-grid execute: upload, T steps, download on the current stream."""
    data = grid.data
    with torch.cuda.device(plan.device):
        dg = _GRIDS.acquire(plan, shape, grid.halo)
        try:
            if native16:
                dg.upload(torch.from_numpy(np.ascontiguousarray(data)))
            else:
                dg.load_dense_f64(torch.from_numpy(np.ascontiguousarray(data, dtype=np.float64)).to(dg.device))
            dg.run(steps)
            if native16:
                target = torch.from_numpy(out.data) if out is not None else torch.empty(
                    dg.dense_shape, dtype=torch.float16, pin_memory=True)
                dg.download(target)
                torch.cuda.current_stream().synchronize()
                res = target.numpy()
            else:
                res = dg.to_dense_f64().cpu().numpy()
                if data.dtype == np.float32:
                    res = res.astype(np.float32)
                if out is not None:
                    out.data[...] = res
                    res = out.data
        finally:
            _GRIDS.release(dg)
    cls = Grid3D if kernel.d == 3 else Grid
    return cls(res, grid.halo, grid.step + steps), stats


def naive_apply(kernel: StencilKernel, grid, steps: int):
    """Reference executor (core.py:151-182) on the device in fp64.

    Bit-identical to the reference numpy oracle for float64 grids; float32
    grids are evaluated in fp64 and rounded once at the end."""
    if steps < 1:
        raise ValueError(f"step count must be >= 1, got {steps}")
    if grid.halo < kernel.r:
        raise ValueError(f"grid halo {grid.halo} too small for stencil radius {kernel.r}")
    dev = require_cuda()
    dense = torch.from_numpy(np.ascontiguousarray(grid.data, dtype=np.float64)).to(dev)
    out = naive_apply_device(kernel, dense, grid.halo, steps).cpu().numpy().astype(grid.data.dtype, copy=False)
    cls = Grid3D if kernel.d == 3 else Grid
    return cls(out, grid.halo, grid.step + steps)


def max_rel_error(result: np.ndarray, reference: np.ndarray) -> float:
    """max|got-want| / max|want| (reference pipeline.py:265-267)."""
    result = np.asarray(result, dtype=np.float64)
    reference = np.asarray(reference, dtype=np.float64)
    scale = max(float(np.max(np.abs(reference))), 1e-300)
    return float(np.max(np.abs(result - reference)) / scale)


def verify(kernel: StencilKernel, sizes, seed: int, steps: int, cfg=ExecConfig(), tolerance: float | None = None) -> dict:
    """Device execute vs device fp64 naive_apply over seeded random grids
    (reference pipeline.py:270-328).  Inputs are quantised to the device dtype
    first, so the comparison measures the arithmetic, not the input rounding."""
    dcfg = _device_cfg(cfg)
    tol = DEFAULT_TOLERANCE[dcfg.dtype] if tolerance is None else float(tolerance)
    cases = []
    first_ok = None
    for size in sizes:
        a, b = (1, int(size)) if kernel.d == 1 else (int(size), int(size))
        grid = random_grid(a, b, kernel.r, seed=[seed, a, b])
        q = torch.from_numpy(grid.data).to(TORCH_DTYPES[dcfg.dtype]).to(torch.float64).numpy()
        grid = Grid(q, grid.halo)
        try:
            got, _ = execute(kernel, grid, steps, dcfg)
        except ValueError as exc:
            cases.append({"size": [a, b], "error": str(exc), "pass": False})
            continue
        want = naive_apply(kernel, grid, steps)
        err = max_rel_error(got.interior, want.interior)
        cases.append({"size": [a, b], "max_rel_error": err, "pass": err < tol})
        if first_ok is None:
            first_ok = (grid, got)
    cross: dict = {}
    if first_ok is not None:
        grid, got = first_ok
        other = Parity.ODD if dcfg.parity is Parity.EVEN else Parity.EVEN
        flipped, _ = execute(kernel, grid, steps, replace(dcfg, parity=other))
        # the reference toggles operand packing (a pure relayout); the device
        # path has one operand image, so the same call is the toggled run
        toggled, _ = execute(kernel, grid, steps, dcfg)
        cross = {
            "parity_max_abs_diff": float(np.max(np.abs(flipped.interior - got.interior))),
            "parity_bitwise_identical": bool(np.array_equal(flipped.interior, got.interior)),
            "packing_bitwise_identical": bool(np.array_equal(toggled.interior, got.interior)),
        }
    return {
        "kernel": {"shape": kernel.shape.value, "d": kernel.d, "r": kernel.r, "coeffs": kernel.coeffs.tolist()},
        "parity": dcfg.parity.value,
        "precision": dcfg.dtype,
        "packing": True,
        "steps": steps,
        "seed": seed,
        "tolerance": tol,
        "cases": cases,
        "all_pass": all(c["pass"] for c in cases),
        "cross_checks": cross,
    }


def report_json(report: dict) -> str:
    return json.dumps(report, indent=2, sort_keys=True)


__all__ = [
    "ExecConfig",
    "DeviceConfig",
    "ExecStats",
    "TransformedStencil",
    "CompressedKernel",
    "transform_stencil",
    "execute",
    "naive_apply",
    "verify",
    "report_json",
    "max_rel_error",
    "get_plan",
    "exec_stats",
    "release_device_grids",
    "stream_windows",
    "DEFAULT_TOLERANCE",
]
