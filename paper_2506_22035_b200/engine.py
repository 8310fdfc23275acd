"""Device engine: plans, device-resident grids and the step loop.

A `Plan` owns the packed tcgen05.mma.sp operands for one stencil (the AOT
transform of every kernel row, laid out for TMEM).  A `DeviceGrid` owns the two
ping-pong buffers of a halo-padded grid in the engine's HBM layout
(include/spider.h, spd_grid_desc).  All compute goes through libspider.so; no
path here falls back to the host.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import DTYPE_CODES, check, dptr, i32ptr, lib, spd_grid_desc, u16ptr, u32ptr
from .core import StencilKernel
from .transform import Parity

TORCH_DTYPES = {"fp16": torch.float16, "bf16": torch.bfloat16}
SPD_PLAN_CTA_PAIR = 1  # include/spider.h
SPD_PLAN_NO_EMBED = 2
SPD_RUN_PERSISTENT, SPD_RUN_CHAINED, SPD_RUN_FORWARD, SPD_RUN_STEPMAJOR = 1, 2, 4, 8  # include/spider.h
# default spd_run_ex flags of DeviceGrid.run (one launch per step)
RUN_FLAGS = 0
NP_DTYPES = {"fp16": np.float16}


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "the SPIDER device engine needs a CUDA device (sm_100a); there is no CPU fallback"
        )
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
    return dev


def _stream_ptr(stream=None, device=None):
    """Raw cudaStream_t: `stream`, else torch's current stream of `device`."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return C.c_void_p(s.cuda_stream)


@dataclass(frozen=True)
class PlanInfo:
    L: int
    r_in: int
    r_out: int
    mmas_per_tile: int
    n_tile: int
    tile_z: int
    tile_y: int
    kchunks: int
    m_tiles: int = 1  # M = 128 tiles per tile (3D: 2, sharing one input block)
    mt_rows: int = 0  # input-row shift of M-tile t's MMA schedule: t * mt_rows
    cg2: int = 0      # CTA-pair mode (3D): rank t owns M-tile t and its own A/E images
    r_dev: int = 0    # device radius (3 for a radius-2 stencil embedded in a zero ring)


class Plan:
    """Packed device operands for one stencil kernel (spd_plan_create).

    device=-1 builds a host-only plan (operand images without an upload),
    which the CPU test tier uses to check the packer.
    """

    def __init__(self, kernel: StencilKernel, parity=Parity.EVEN, dtype: str = "fp16", device: int | None = None,
                 cta_pair: bool = False):
        if dtype not in DTYPE_CODES:
            raise ValueError(f"dtype must be one of {sorted(DTYPE_CODES)}, got {dtype!r}")
        self.kernel = kernel
        self.parity = Parity(parity)
        self.dtype = dtype
        if device is None:
            device = require_cuda().index
        self.device = int(device)
        coeffs = np.ascontiguousarray(kernel.coeffs, dtype=np.float64).ravel()
        self._coeffs = coeffs
        self.cta_pair = bool(cta_pair)
        h = C.c_void_p()
        flags = SPD_PLAN_CTA_PAIR if cta_pair else 0
        if os.environ.get("SPD_NO_EMBED"):  # development override: radius 2 on the generic L = 6 path
            flags |= SPD_PLAN_NO_EMBED
        check(lib.spd_plan_create_ex(kernel.d, kernel.r, self.parity.code, dptr(coeffs), DTYPE_CODES[dtype],
                                     self.device, flags, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.spd_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> PlanInfo:
        buf = np.zeros(12, dtype=np.int32)
        check(lib.spd_plan_info(self._h, i32ptr(buf)))
        return PlanInfo(*[int(v) for v in buf])

    def operands(self):
        """(a_img [R*S,128,16] uint16, e_words [R*S,128] uint32, start_rows [S]);
        R = 2 in CTA-pair mode (rank-major), else 1."""
        inf = self.info()
        ranks = 2 if inf.cg2 else 1
        a = np.zeros((ranks * inf.mmas_per_tile, 128, 16), dtype=np.uint16)
        e = np.zeros((ranks * inf.mmas_per_tile, 128), dtype=np.uint32)
        s = np.zeros(inf.mmas_per_tile, dtype=np.int32)
        check(lib.spd_plan_operands(self._h, u16ptr(a), u32ptr(e), i32ptr(s)))
        return a, e, s

    def geometry(self):
        """(in_off [R_in,3], out_off [R_out*m_tiles,3]) tile row offsets (dz, dy, dx)."""
        inf = self.info()
        a = np.zeros((inf.r_in, 3), dtype=np.int32)
        b = np.zeros((inf.r_out * (2 if inf.cg2 else inf.m_tiles), 3), dtype=np.int32)
        check(lib.spd_plan_geometry(self._h, i32ptr(a), i32ptr(b)))
        return a, b

    def lane_map(self) -> np.ndarray:
        """MMA row (accumulator TMEM lane) of logical kernel-matrix row
        m = L*a + i (output row a, chunk position i), length r_out*L."""
        inf = self.info()
        lanes = np.zeros(inf.r_out * inf.L, dtype=np.int32)
        check(lib.spd_plan_lane_map(self._h, i32ptr(lanes)))
        return lanes

    def mma_halves(self) -> np.ndarray:
        """Per MMA of the tile schedule: 0 = M = 128 over all accumulator
        lanes, 1 / 2 = M = 64 over lanes 0-15 / 16-31 of each quadrant."""
        out = np.zeros(self.info().mmas_per_tile, dtype=np.int32)
        check(lib.spd_plan_mma_halves(self._h, i32ptr(out)))
        return out

    def layout(self, nz: int, ny: int, nx: int, halo: int) -> spd_grid_desc:
        desc = spd_grid_desc()
        check(lib.spd_grid_layout(self._h, int(nz), int(ny), int(nx), int(halo), C.byref(desc)))
        return desc


def _on_device(fn):
    """Run a DeviceGrid method with its grid's device current: libspider
    launches on the current device, and the default stream is that device's
    current torch stream (execute may target a device that is not current)."""
    import functools

    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        if torch.cuda.current_device() == self.device.index:
            return fn(self, *args, **kwargs)
        with torch.cuda.device(self.device):
            return fn(self, *args, **kwargs)

    return wrapper


class DeviceGrid:
    """Ping-pong buffers of one grid in the engine layout, resident in HBM."""

    def __init__(self, plan: Plan, shape, halo: int):
        require_cuda()
        self.plan = plan
        nz, ny, nx = _shape3(plan.kernel.d, shape)
        self.desc_shape = tuple(int(v) for v in shape)
        self.desc = plan.layout(nz, ny, nx, halo)
        dev = torch.device("cuda", plan.device)
        self.device = dev
        tdt = TORCH_DTYPES[plan.dtype]
        self.bufs = [torch.zeros(self.desc.alloc_elems, dtype=tdt, device=dev) for _ in range(2)]
        self.cur = 0  # index of the buffer holding the current state
        self.step = 0

    @property
    def halo(self) -> int:
        return int(self.desc.halo)

    @property
    def dense_shape(self):
        h = self.desc.halo
        if self.plan.kernel.d == 3:
            return (self.desc.nz + 2 * h, self.desc.ny + 2 * h, self.desc.nx + 2 * h)
        return (self.desc.ny + 2 * h, self.desc.nx + 2 * h)

    def _sp(self, stream):
        return _stream_ptr(stream, self.device)

    @_on_device
    def _sync_halo(self, stream=None) -> None:
        """Replicate the Dirichlet ring of the current buffer into the other
        one (stream-ordered after the upload that wrote it)."""
        check(lib.spd_copy_halo(C.byref(self.desc), C.c_void_p(self.bufs[self.cur].data_ptr()),
                                C.c_void_p(self.bufs[1 - self.cur].data_ptr()), self._sp(stream)))

    @_on_device
    def load_dense_f64(self, dense: torch.Tensor, stream=None) -> None:
        """Quantise a dense fp64 device tensor (halo included) into the grid."""
        if dense.dtype != torch.float64 or not dense.is_cuda:
            raise ValueError("expected a CUDA float64 tensor")
        dense = dense.contiguous()
        if tuple(dense.shape) != tuple(self.dense_shape):
            raise ValueError(f"dense grid shape {tuple(dense.shape)} != {self.dense_shape}")
        check(lib.spd_pack_grid(C.byref(self.desc), DTYPE_CODES[self.plan.dtype], C.c_void_p(dense.data_ptr()),
                                C.c_void_p(self.bufs[self.cur].data_ptr()), self._sp(stream)))
        self._sync_halo(stream)

    @_on_device
    def to_dense_f64(self, stream=None) -> torch.Tensor:
        out = torch.empty(self.dense_shape, dtype=torch.float64, device=self.bufs[0].device)
        check(lib.spd_unpack_grid(C.byref(self.desc), DTYPE_CODES[self.plan.dtype],
                                  C.c_void_p(self.bufs[self.cur].data_ptr()), C.c_void_p(out.data_ptr()),
                                  self._sp(stream)))
        return out

    def _staged(self, staged) -> bool:
        """Host transfers through a device staging buffer (one linear DMA +
        a repack kernel) instead of a strided DMA: the default for short rows
        (3D grids), where the strided copy engine path is slow."""
        if staged is None:
            env = os.environ.get("SPD_STAGED")
            staged = bool(int(env)) if env else (self.desc.dims == 3 or self.dense_shape[-1] * 2 < 16384)
        return staged

    def _staging(self, stream):
        buf = torch.empty(self.dense_shape, dtype=TORCH_DTYPES[self.plan.dtype], device=self.bufs[0].device)
        if stream is not None:
            buf.record_stream(stream)
        return buf

    @_on_device
    def upload(self, host: torch.Tensor, stream=None, staged=None) -> None:
        """DMA of a host 16-bit dense grid (pinned for async)."""
        if host.dtype != TORCH_DTYPES[self.plan.dtype] or host.is_cuda:
            raise ValueError(f"expected a host {TORCH_DTYPES[self.plan.dtype]} tensor")
        if tuple(host.shape) != tuple(self.dense_shape) or not host.is_contiguous():
            raise ValueError(f"host grid must be contiguous with shape {self.dense_shape}")
        if self._staged(staged):
            st = self._staging(stream)
            check(lib.spd_upload_staged(C.byref(self.desc), C.c_void_p(host.data_ptr()),
                                        C.c_void_p(self.bufs[self.cur].data_ptr()), C.c_void_p(st.data_ptr()),
                                        self._sp(stream)))
        else:
            check(lib.spd_upload(C.byref(self.desc), C.c_void_p(host.data_ptr()),
                                 C.c_void_p(self.bufs[self.cur].data_ptr()), self._sp(stream)))
        self._sync_halo(stream)

    @_on_device
    def download(self, host: torch.Tensor, stream=None, staged=None) -> None:
        if host.dtype != TORCH_DTYPES[self.plan.dtype] or host.is_cuda:
            raise ValueError(f"expected a host {TORCH_DTYPES[self.plan.dtype]} tensor")
        if tuple(host.shape) != tuple(self.dense_shape) or not host.is_contiguous():
            raise ValueError(f"host grid must be contiguous with shape {self.dense_shape}")
        if self._staged(staged):
            st = self._staging(stream)
            check(lib.spd_download_staged(C.byref(self.desc), C.c_void_p(self.bufs[self.cur].data_ptr()),
                                          C.c_void_p(host.data_ptr()), C.c_void_p(st.data_ptr()),
                                          self._sp(stream)))
        else:
            check(lib.spd_download(C.byref(self.desc), C.c_void_p(self.bufs[self.cur].data_ptr()),
                                   C.c_void_p(host.data_ptr()), self._sp(stream)))

    @_on_device
    def download_rows(self, host_ptr: int, lo: int, hi: int, stream=None) -> None:
        """Dense rows (2D) / planes (3D) [lo, hi) of the current buffer into
        the same rows of a host dense array starting at `host_ptr` (the
        array's first halo row; only those rows are written)."""
        check(lib.spd_download_rows(C.byref(self.desc), C.c_void_p(self.bufs[self.cur].data_ptr()),
                                    C.c_void_p(int(host_ptr)), int(lo), int(hi), self._sp(stream)))

    @_on_device
    def run(self, steps: int, stream=None, persistent: bool = False, flags: int | None = None) -> None:
        """`steps` Jacobi steps on the device, ping-ponging the buffers
        (one launch per step, or one persistent launch).  `flags` overrides
        the spd_run_ex flags (SPD_RUN_*); default RUN_FLAGS."""
        if steps < 1:
            raise ValueError(f"step count must be >= 1, got {steps}")
        if flags is None:
            flags = SPD_RUN_PERSISTENT if persistent else RUN_FLAGS
        a, b = self.bufs[self.cur], self.bufs[1 - self.cur]
        check(lib.spd_run_ex(self.plan.handle, C.byref(self.desc), C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                             int(steps), int(flags), self._sp(stream)))
        self.cur = (self.cur + steps) % 2
        self.step += steps

    @_on_device
    def step_range(self, lo: int, hi: int, stream=None) -> None:
        """One step over output rows (2D) / planes (3D) [lo, hi) only; does
        not flip the buffers (call `flip()` once the whole domain is done)."""
        a, b = self.bufs[self.cur], self.bufs[1 - self.cur]
        check(lib.spd_step_range(self.plan.handle, C.byref(self.desc), C.c_void_p(a.data_ptr()),
                                 C.c_void_p(b.data_ptr()), int(lo), int(hi), self._sp(stream)))

    @_on_device
    def step_edges(self, stream=None) -> None:
        """One step over the first and last tile bands only (one launch); with
        step_range over the bands between them this is a full step."""
        a, b = self.bufs[self.cur], self.bufs[1 - self.cur]
        check(lib.spd_step_edges(self.plan.handle, C.byref(self.desc), C.c_void_p(a.data_ptr()),
                                 C.c_void_p(b.data_ptr()), self._sp(stream)))

    def flip(self) -> None:
        self.cur = 1 - self.cur
        self.step += 1

    def view_rows(self, which: int | None = None) -> torch.Tensor:
        """2D/1D: the stored buffer as [rows, pitch]; 3D: [planes, rows, pitch]."""
        buf = self.bufs[self.cur if which is None else which]
        d = self.desc
        if self.plan.kernel.d == 3:
            return buf.view(-1, d.plane // d.pitch, d.pitch)
        return buf.view(-1, d.pitch)


def _shape3(d: int, shape):
    shape = tuple(int(s) for s in shape)
    if d == 3:
        if len(shape) != 3:
            raise ValueError("3D grids need an interior shape (Z, A, B)")
        return shape
    if len(shape) != 2:
        raise ValueError("2D/1D grids need an interior shape (A, B)")
    return (1,) + shape


def naive_apply_device(kernel: StencilKernel, dense: torch.Tensor, halo: int, steps: int) -> torch.Tensor:
    """fp64 brute-force executor on the device (reference core.py:151-182).

    `dense` is the halo-padded fp64 CUDA tensor; returns a new tensor.  Same
    row-major tap order and separate multiply/add roundings as the numpy
    oracle, so results are bit-identical to it.
    """
    require_cuda()
    if steps < 1:
        raise ValueError(f"step count must be >= 1, got {steps}")
    if halo < kernel.r:
        raise ValueError(f"grid halo {halo} too small for stencil radius {kernel.r}")
    dense = dense.contiguous()
    if kernel.d == 3:
        nz, ny, nx = (s - 2 * halo for s in dense.shape)
    else:
        nz = 1
        ny, nx = (s - 2 * halo for s in dense.shape)
    out = torch.empty_like(dense)
    scratch = torch.empty_like(dense)
    coeffs = np.ascontiguousarray(kernel.coeffs, dtype=np.float64).ravel()
    check(lib.spd_naive_apply_f64(kernel.d, kernel.r, dptr(coeffs), nz, ny, nx, halo, C.c_void_p(dense.data_ptr()),
                                  C.c_void_p(out.data_ptr()), C.c_void_p(scratch.data_ptr()), int(steps),
                                  _stream_ptr()))
    return out


def mma_selftest(a: np.ndarray, e: np.ndarray, b: np.ndarray) -> np.ndarray:
    """One tcgen05.mma.sp on the device: decode(a, e) @ b (M=128, K=32)."""
    require_cuda()
    n = b.shape[1]
    ta = torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint16).view(np.int16)).cuda()
    te = torch.from_numpy(np.ascontiguousarray(e, dtype=np.uint8)).cuda()
    tb = torch.from_numpy(np.ascontiguousarray(b, dtype=np.uint16).view(np.int16)).cuda()
    td = torch.empty((128, n), dtype=torch.float32, device="cuda")
    check(lib.spd_mma_selftest(C.c_void_p(ta.data_ptr()), C.c_void_p(te.data_ptr()), C.c_void_p(tb.data_ptr()), n,
                               C.c_void_p(td.data_ptr()), _stream_ptr()))
    return td.cpu().numpy()


_ = _lib
