"""ctypes wrapper of oracle/liboracle.so (TEST ONLY; see oracle/naive.c)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .build import LIB, build

_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(str(LIB))
        D = C.POINTER(C.c_double)
        _lib.oracle_naive_f64.restype = C.c_int
        _lib.oracle_naive_f64.argtypes = [C.c_int, C.c_int, D, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                          D, D, D, C.c_int, C.c_int]
        _lib.oracle_naive_steps.restype = C.c_int
        _lib.oracle_naive_steps.argtypes = [C.c_int, C.c_int, D, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                            D, D, C.c_int, C.c_int]
    return _lib


def naive_apply(coeffs, d: int, r: int, data: np.ndarray, halo: int, steps: int, threads: int | None = None):
    lib = _load()
    data = np.ascontiguousarray(data, dtype=np.float64)
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
    if d == 3:
        nz, ny, nx = (n - 2 * halo for n in data.shape)
    else:
        nz = 1
        ny, nx = (n - 2 * halo for n in data.shape)
    out = np.empty_like(data)
    scratch = np.empty_like(data)
    threads = threads or os.cpu_count() or 1
    D = C.POINTER(C.c_double)
    rc = lib.oracle_naive_f64(d, r, coeffs.ctypes.data_as(D), nz, ny, nx, halo, data.ctypes.data_as(D),
                              out.ctypes.data_as(D), scratch.ctypes.data_as(D), steps, threads)
    if rc != 0:
        raise ValueError("oracle_naive_f64: bad arguments")
    return out


class NaiveRunner:
    """Two resident fp64 buffers advanced in place by `run(steps)` (no per-call
    allocation or grid copies): the bench's CPU reference arm.  `state` is the
    current dense grid (halo included)."""

    def __init__(self, coeffs, d: int, r: int, data: np.ndarray, halo: int, threads: int | None = None):
        self.lib = _load()
        self.d, self.r, self.halo = d, r, halo
        self.coeffs = np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
        self.bufs = [np.ascontiguousarray(data, dtype=np.float64).copy(), np.ascontiguousarray(data, dtype=np.float64).copy()]
        if d == 3:
            self.nz, self.ny, self.nx = (n - 2 * halo for n in data.shape)
        else:
            self.nz = 1
            self.ny, self.nx = (n - 2 * halo for n in data.shape)
        self.threads = threads or os.cpu_count() or 1
        self.cur = 0

    def run(self, steps: int) -> None:
        D = C.POINTER(C.c_double)
        a, b = self.bufs[self.cur], self.bufs[1 - self.cur]
        rc = self.lib.oracle_naive_steps(self.d, self.r, self.coeffs.ctypes.data_as(D), self.nz, self.ny, self.nx,
                                         self.halo, a.ctypes.data_as(D), b.ctypes.data_as(D), int(steps),
                                         self.threads)
        if rc < 0:
            raise ValueError("oracle_naive_steps: bad arguments")
        self.cur = (self.cur + rc) % 2

    @property
    def state(self) -> np.ndarray:
        return self.bufs[self.cur]
