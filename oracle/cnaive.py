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
