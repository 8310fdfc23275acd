"""AOT kernel-matrix transform: banded matrix, strided column swap, 2:4 encode.

Same public surface as the reference transform layer (reference
transform.py:37-267).  The arithmetic runs in the C++ AOT builder of
libspider.so (csrc/aot.cpp) — one implementation shared with the device plan,
so the operands the tensor cores see are exactly the ones these functions
return.  Parity with the reference is exact (tests/test_transform_parity.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from fractions import Fraction

import numpy as np

from . import _lib
from ._lib import check, dptr, i32ptr, i64ptr, lib, u8ptr

PAD_COLUMNS = 2


class Parity(str, Enum):
    """Column class moved by the strided swap (reference transform.py:280-288)."""

    EVEN = "even"
    ODD = "odd"

    @property
    def start(self) -> int:
        return 0 if self is Parity.EVEN else 1

    @property
    def code(self) -> int:
        return self.start


def band_rows(r: int) -> int:
    """L = 2r+2 (reference transform.py:37-41)."""
    return check(lib.spd_band_rows(int(r)))


def sparsity_ratio(r: int, L: int) -> Fraction:
    """Nonzero fraction (2r+1)/(2r+L) of the unpadded band (transform.py:44-51)."""
    if r < 1:
        raise ValueError(f"radius must be >= 1, got {r}")
    if L < 1:
        raise ValueError(f"L must be >= 1, got {L}")
    return Fraction(2 * r + 1, 2 * r + L)


def sptc_compatible(r: int, L: int) -> bool:
    return sparsity_ratio(r, L) <= Fraction(1, 2)


@dataclass
class KernelMatrix:
    values: np.ndarray
    r: int
    swapped: bool = False
    parity: Parity | None = None

    @property
    def L(self) -> int:
        return self.values.shape[0]

    @property
    def width(self) -> int:
        return self.values.shape[1]


@dataclass
class CompressedKernel:
    """L x L kept values plus L x (L/2) x 2 ascending position pairs."""

    values: np.ndarray
    metadata: np.ndarray
    r: int
    parity: Parity

    @property
    def L(self) -> int:
        return self.values.shape[0]

    @property
    def segments_per_row(self) -> int:
        return self.metadata.shape[1]


@dataclass(frozen=True)
class RowPermutation:
    mapping: np.ndarray
    parity: Parity

    @property
    def size(self) -> int:
        return self.mapping.shape[0]

    def apply(self, x: np.ndarray) -> np.ndarray:
        return np.asarray(x)[self.mapping]

    def __call__(self, j: int) -> int:
        return int(self.mapping[j])


@dataclass
class Check24Report:
    valid: bool
    violations: list


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def build_kernel_matrix(kernel_row, r: int) -> KernelMatrix:
    L = band_rows(r)
    row = _f64(kernel_row).ravel()
    if row.size != 2 * r + 1:
        raise ValueError(f"kernel row needs 2r+1 = {2 * r + 1} entries, got {row.size}")
    out = np.empty((L, 2 * L), dtype=np.float64)
    check(lib.spd_build_kernel_matrix(int(r), dptr(row), dptr(out)))
    return KernelMatrix(values=out, r=r)


def input_row_permutation(L: int, parity: Parity = Parity.EVEN) -> RowPermutation:
    parity = Parity(parity)
    mapping = np.empty(2 * L if L > 0 else 0, dtype=np.int64)
    check(lib.spd_row_permutation(int(L), parity.code, i64ptr(mapping)))
    mapping.setflags(write=False)
    return RowPermutation(mapping=mapping, parity=parity)


def swap_columns(values: np.ndarray, parity: Parity) -> np.ndarray:
    values = _f64(values)
    out = np.empty_like(values)
    check(lib.spd_swap_columns(dptr(values), values.shape[0], values.shape[1], Parity(parity).code, dptr(out)))
    return out


def strided_swap(matrix: KernelMatrix, parity: Parity = Parity.EVEN) -> KernelMatrix:
    if matrix.swapped:
        raise ValueError("kernel matrix already swapped; the swap is one-shot")
    parity = Parity(parity)
    return KernelMatrix(values=swap_columns(matrix.values, parity), r=matrix.r, swapped=True, parity=parity)


def check_2to4(matrix) -> Check24Report:
    values = matrix.values if isinstance(matrix, KernelMatrix) else np.asarray(matrix)
    if values.ndim != 2:
        raise ValueError("expected a 2D matrix")
    values = _f64(values)
    rows, width = values.shape
    cap = max(1, rows * max(width // 4, 1))
    viol = np.zeros(2 * cap, dtype=np.int32)
    n = check(lib.spd_check_2to4(dptr(values), rows, width, i32ptr(viol), cap))
    pairs = [(int(viol[2 * k]), int(viol[2 * k + 1])) for k in range(n)]
    return Check24Report(valid=n == 0, violations=pairs)


def encode_segment(segment) -> tuple[float, float, int, int]:
    seg = _f64(segment)
    if seg.shape != (4,):
        raise ValueError("segment must have exactly 4 entries")
    vals = np.zeros(2, dtype=np.float64)
    pos = np.zeros(2, dtype=np.uint8)
    check(lib.spd_encode_segment(dptr(seg), dptr(vals), u8ptr(pos)))
    return float(vals[0]), float(vals[1]), int(pos[0]), int(pos[1])


def encode(matrix: KernelMatrix) -> CompressedKernel:
    if not matrix.swapped or matrix.parity is None:
        raise ValueError("encode expects a swapped kernel matrix")
    values = _f64(matrix.values)
    rows, width = values.shape
    out_v = np.zeros((rows, width // 2), dtype=np.float64)
    out_m = np.zeros((rows, width // 4, 2), dtype=np.uint8)
    check(lib.spd_encode(dptr(values), rows, width, dptr(out_v), u8ptr(out_m)))
    return CompressedKernel(values=out_v, metadata=out_m, r=matrix.r, parity=matrix.parity)


def validate_metadata(metadata: np.ndarray) -> None:
    meta = np.asarray(metadata)
    if meta.ndim != 3 or meta.shape[2] != 2:
        raise ValueError("metadata must have shape (rows, segments, 2)")
    if meta.min(initial=0) < 0 or meta.max(initial=0) > 3:
        raise ValueError("metadata positions must lie in {0,1,2,3}")
    if np.any(meta[..., 0] >= meta[..., 1]):
        raise ValueError("metadata position pairs must be strictly ascending")


def decode(compressed: CompressedKernel) -> KernelMatrix:
    meta = np.asarray(compressed.metadata)
    validate_metadata(meta)
    rows, segs = meta.shape[0], meta.shape[1]
    vals = _f64(compressed.values)
    meta = np.ascontiguousarray(meta, dtype=np.uint8)
    out = np.zeros((rows, 4 * segs), dtype=np.float64)
    check(lib.spd_decode(dptr(vals), u8ptr(meta), rows, segs, dptr(out)))
    return KernelMatrix(values=out, r=compressed.r, swapped=True, parity=compressed.parity)


def metadata_to_bytes(metadata: np.ndarray) -> bytes:
    meta = np.ascontiguousarray(metadata, dtype=np.uint8)
    n = meta.size // 2
    out = np.zeros(n, dtype=np.uint8)
    check(lib.spd_metadata_to_bytes(u8ptr(meta), n, u8ptr(out)))
    return out.tobytes()


def metadata_from_bytes(raw: bytes, L: int, segments: int) -> np.ndarray:
    packed = np.frombuffer(raw, dtype=np.uint8)
    if packed.size != L * segments:
        raise ValueError(f"expected {L * segments} metadata bytes, got {packed.size}")
    packed = packed.reshape(L, segments)
    meta = np.stack([packed & 0b11, (packed >> 2) & 0b11], axis=2).astype(np.uint8)
    validate_metadata(meta)
    return meta


def transform_row(row, r: int, parity: Parity = Parity.EVEN) -> CompressedKernel:
    """encode(strided_swap(build_kernel_matrix(row, r), parity)) in one C call."""
    L = band_rows(r)
    row = _f64(row).ravel()
    if row.size != 2 * r + 1:
        raise ValueError(f"kernel row needs 2r+1 = {2 * r + 1} entries, got {row.size}")
    vals = np.zeros((L, L), dtype=np.float64)
    meta = np.zeros((L, L // 2, 2), dtype=np.uint8)
    parity = Parity(parity)
    check(lib.spd_transform_row(int(r), parity.code, dptr(row), dptr(vals), u8ptr(meta)))
    return CompressedKernel(values=vals, metadata=meta, r=r, parity=parity)


__all__ = [
    "PAD_COLUMNS",
    "Parity",
    "band_rows",
    "sparsity_ratio",
    "sptc_compatible",
    "KernelMatrix",
    "CompressedKernel",
    "RowPermutation",
    "Check24Report",
    "build_kernel_matrix",
    "input_row_permutation",
    "swap_columns",
    "strided_swap",
    "check_2to4",
    "encode_segment",
    "encode",
    "validate_metadata",
    "decode",
    "metadata_to_bytes",
    "metadata_from_bytes",
    "transform_row",
]
_ = _lib


# SPCK record I/O lives in io.py; the reference keeps it in transform
# (transform.py:270-352).  Lazy re-exports (PEP 562) keep
# `from <pkg>.transform import save_compressed_set, compressed_from_dict` working.
_IO_NAMES = {"COMPRESSED_MAGIC", "compressed_record_bytes", "save_compressed_set", "load_compressed_set",
             "compressed_to_dict", "compressed_from_dict", "save_compressed_json"}


def __getattr__(name):
    import importlib

    if name in _IO_NAMES:
        return getattr(importlib.import_module(".io", __package__), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
