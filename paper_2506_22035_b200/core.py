"""Stencil definitions and halo-padded grids (host data model).

Mirrors the reference problem-definition layer (reference core.py:22-148):
same names, validation rules and error-message substrings, so reference-style
callers and tests work unchanged.  Adds the 3D extension the BASELINE configs
need (Box-3D27P / Heat-3D): `make_kernel(..., d=3, ...)` is rejected exactly
like the reference does, and 3D kernels come from `make_kernel_3d`.

There is no arithmetic here: executing a stencil always goes to the device
(`pipeline.execute` / `pipeline.naive_apply`).
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np


class Shape(str, Enum):
    """Footprint of a stencil: full (2r+1)^d box or axis-aligned star."""

    BOX = "box"
    STAR = "star"


@dataclass(frozen=True)
class StencilKernel:
    """Validated stencil coefficients, indexed by offset + r along each axis.

    d = 1: shape (2r+1,); d = 2: (2r+1, 2r+1) as (rho, delta);
    d = 3: (2r+1, 2r+1, 2r+1) as (rho_z, rho_y, delta).
    """

    shape: Shape
    d: int
    r: int
    coeffs: np.ndarray

    @property
    def points(self) -> int:
        return int(self.coeffs.size)

    def row_offsets(self):
        """Offsets of the kernel rows (reference core.py:46-50).

        1D: the single row 0.  2D: rho in [-r, r].  3D: (rho_z, rho_y) pairs in
        row-major order — the order the device transform emits its rows in.
        """
        if self.d == 1:
            return range(0, 1)
        span = range(-self.r, self.r + 1)
        if self.d == 2:
            return span
        return [(rz, ry) for rz in span for ry in span]

    def row(self, rho) -> np.ndarray:
        """The 2r+1 coefficients of one kernel row (reference core.py:52-60)."""
        if self.d == 1:
            if rho != 0:
                raise ValueError("1D kernel has a single row at offset 0")
            return self.coeffs
        if self.d == 2:
            if not -self.r <= rho <= self.r:
                raise ValueError(f"row offset {rho} outside [-{self.r}, {self.r}]")
            return self.coeffs[rho + self.r]
        rz, ry = rho
        if not (-self.r <= rz <= self.r and -self.r <= ry <= self.r):
            raise ValueError(f"row offset {rho} outside [-{self.r}, {self.r}]^2")
        return self.coeffs[rz + self.r, ry + self.r]

    def rows_array(self) -> np.ndarray:
        """All kernel rows stacked in transform order: (n_rows, 2r+1)."""
        return np.ascontiguousarray(self.coeffs.reshape(-1, 2 * self.r + 1), dtype=np.float64)


def _validate(shape, d: int, r, coeffs, allowed_d) -> StencilKernel:
    shape = Shape(shape)
    if d not in allowed_d:
        raise ValueError(f"dimensionality must be {' or '.join(map(str, allowed_d))}, got {d}")
    if not isinstance(r, (int, np.integer)) or isinstance(r, bool) or r < 1:
        raise ValueError(f"radius must be an integer >= 1, got {r}")
    r = int(r)
    values = np.asarray(coeffs, dtype=np.float64)
    n = 2 * r + 1
    if values.size != n**d:
        raise ValueError(f"kernel needs {n**d} coefficients for d={d}, r={r}; got {values.size}")
    values = values.reshape((n,) * d).copy()
    if shape is Shape.STAR and d >= 2:
        mask = np.zeros(values.shape, dtype=bool)
        for axis in range(d):
            index = [r] * d
            index[axis] = slice(None)
            mask[tuple(index)] = True
        if np.any(values[~mask] != 0.0):
            raise ValueError("star kernel has nonzero coefficients off both axes")
    values.setflags(write=False)
    return StencilKernel(shape=shape, d=d, r=r, coeffs=values)


def make_kernel(shape, d: int, r: int, coeffs) -> StencilKernel:
    """Validate a 1D/2D kernel (reference core.py:63-89; d=3 is rejected there
    too — use make_kernel_3d for the 3D extension)."""
    return _validate(shape, d, r, coeffs, (1, 2))


def make_kernel_3d(shape, r: int, coeffs) -> StencilKernel:
    """3D extension (Box-3D27P, Heat-3D 7-point): coeffs[(rz, ry, dx)]."""
    return _validate(shape, 3, r, coeffs, (3,))


@dataclass
class Grid:
    """Interior A x B plus a Dirichlet halo of width `halo` on every side
    (reference core.py:92-127).  1D problems use A = 1."""

    data: np.ndarray
    halo: int
    step: int = 0

    def __post_init__(self) -> None:
        if self.data.ndim != 2:
            raise ValueError("grid storage must be 2D (1D problems use A = 1)")
        if self.halo < 0 or min(self.data.shape) <= 2 * self.halo:
            raise ValueError("grid extent too small for its halo")

    @property
    def A(self) -> int:
        return self.data.shape[0] - 2 * self.halo

    @property
    def B(self) -> int:
        return self.data.shape[1] - 2 * self.halo

    @property
    def interior(self) -> np.ndarray:
        h = self.halo
        return self.data[h : h + self.A, h : h + self.B]

    def copy(self) -> "Grid":
        return Grid(self.data.copy(), self.halo, self.step)

    def astype(self, dtype) -> "Grid":
        return Grid(self.data.astype(dtype), self.halo, self.step)


@dataclass
class Grid3D:
    """3D extension of Grid: interior Z x A x B, halo on all six faces."""

    data: np.ndarray
    halo: int
    step: int = 0

    def __post_init__(self) -> None:
        if self.data.ndim != 3:
            raise ValueError("3D grid storage must have 3 axes")
        if self.halo < 0 or min(self.data.shape) <= 2 * self.halo:
            raise ValueError("grid extent too small for its halo")

    @property
    def Z(self) -> int:
        return self.data.shape[0] - 2 * self.halo

    @property
    def A(self) -> int:
        return self.data.shape[1] - 2 * self.halo

    @property
    def B(self) -> int:
        return self.data.shape[2] - 2 * self.halo

    @property
    def interior(self) -> np.ndarray:
        h = self.halo
        return self.data[h : h + self.Z, h : h + self.A, h : h + self.B]

    def copy(self) -> "Grid3D":
        return Grid3D(self.data.copy(), self.halo, self.step)

    def astype(self, dtype) -> "Grid3D":
        return Grid3D(self.data.astype(dtype), self.halo, self.step)


def grid_from_interior(interior, halo: int, fill: float = 0.0):
    """Embed an interior array in a constant halo (reference core.py:130-141).
    3D interiors give a Grid3D."""
    inner = np.asarray(interior, dtype=np.float64)
    if inner.ndim == 1:
        inner = inner[None, :]
    full = np.full(tuple(n + 2 * halo for n in inner.shape), fill, dtype=inner.dtype)
    full[tuple(slice(halo, halo + n) for n in inner.shape)] = inner
    return Grid3D(full, halo) if inner.ndim == 3 else Grid(full, halo)


def random_grid(A: int, B: int, halo: int, seed, dtype=np.float64) -> Grid:
    """Seeded U(-1, 1) grid, halo included (reference core.py:144-148)."""
    rng = np.random.default_rng(seed)
    return Grid(rng.uniform(-1.0, 1.0, size=(A + 2 * halo, B + 2 * halo)).astype(dtype), halo)


def random_grid_3d(Z: int, A: int, B: int, halo: int, seed, dtype=np.float64) -> Grid3D:
    rng = np.random.default_rng(seed)
    shape = (Z + 2 * halo, A + 2 * halo, B + 2 * halo)
    return Grid3D(rng.uniform(-1.0, 1.0, size=shape).astype(dtype), halo)


# The reference keeps its file I/O and the brute-force executor in core
# (core.py:151-254); here they live in io.py and pipeline.py (the executor runs
# on the device).  Re-export them lazily (PEP 562) so `from <pkg>.core import
# save_grid, naive_apply` works as with the reference without an import cycle.
_IO_NAMES = {"GRID_MAGIC", "save_grid", "load_grid", "grid_to_dict", "grid_from_dict", "save_grid_json",
             "load_grid_json", "kernel_to_dict", "kernel_from_dict", "save_kernel", "load_kernel"}


def __getattr__(name):
    import importlib

    if name in _IO_NAMES:
        return getattr(importlib.import_module(".io", __package__), name)
    if name == "naive_apply":
        return importlib.import_module(".pipeline", __package__).naive_apply
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
