"""File formats of the reference front end, byte-compatible.

* SPGR flat binary grids: 16-byte header ``<4sIII`` (magic, A, B, halo) then
  row-major little-endian float64 including the halo (reference
  core.py:185-207).  The 3D extension uses magic ``SPG3`` and a 20-byte header
  ``<4sIIII`` (magic, Z, A, B, halo); the reference has no 3D grids.
* JSON grids and JSON kernels (reference core.py:210-254); kernels with
  ``"d": 3`` load through `make_kernel_3d`.
* SPCK compressed-kernel records: ``<4sHHB`` (magic, r, L, parity code) +
  L*L float64 values + L*(L/2) metadata bytes, records back to back
  (reference transform.py:270-352), plus the JSON mirror.

Host-side only (no device code); the CLI (`cli.py`) reads and writes these
around the device engine.
"""
from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np

from .core import Grid, Grid3D, StencilKernel, make_kernel, make_kernel_3d
from .transform import CompressedKernel, Parity, metadata_from_bytes, metadata_to_bytes, validate_metadata

GRID_MAGIC = b"SPGR"
GRID3_MAGIC = b"SPG3"
COMPRESSED_MAGIC = b"SPCK"
_GRID_HEADER = struct.Struct("<4sIII")
_GRID3_HEADER = struct.Struct("<4sIIII")
_COMPRESSED_HEADER = struct.Struct("<4sHHB")


# ---------------------------------------------------------------------------
# grids

def save_grid(grid, path) -> None:
    """Write SPGR (2D) or SPG3 (3D extension); values as float64."""
    if isinstance(grid, Grid3D):
        header = _GRID3_HEADER.pack(GRID3_MAGIC, grid.Z, grid.A, grid.B, grid.halo)
    else:
        header = _GRID_HEADER.pack(GRID_MAGIC, grid.A, grid.B, grid.halo)
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(np.ascontiguousarray(grid.data, dtype="<f8").tobytes())


def load_grid(path):
    """Read SPGR / SPG3 (reference core.py:197-207: same messages)."""
    raw = Path(path).read_bytes()
    if len(raw) >= 4 and raw[:4] == GRID3_MAGIC:
        if len(raw) < _GRID3_HEADER.size:
            raise ValueError(f"{path}: truncated grid file")
        _, z, a, b, halo = _GRID3_HEADER.unpack_from(raw)
        shape = (z + 2 * halo, a + 2 * halo, b + 2 * halo)
        body = np.frombuffer(raw, dtype="<f8", offset=_GRID3_HEADER.size)
        if body.size != int(np.prod(shape)):
            raise ValueError(f"{path}: expected {int(np.prod(shape))} values, found {body.size}")
        return Grid3D(body.reshape(shape).astype(np.float64), halo)
    if len(raw) < _GRID_HEADER.size:
        raise ValueError(f"{path}: truncated grid file")
    magic, a, b, halo = _GRID_HEADER.unpack_from(raw)
    if magic != GRID_MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}, expected {GRID_MAGIC!r}")
    rows, cols = a + 2 * halo, b + 2 * halo
    body = np.frombuffer(raw, dtype="<f8", offset=_GRID_HEADER.size)
    if body.size != rows * cols:
        raise ValueError(f"{path}: expected {rows * cols} values, found {body.size}")
    return Grid(body.reshape(rows, cols).astype(np.float64), halo)


def grid_to_dict(grid) -> dict:
    out = {"A": grid.A, "B": grid.B, "halo": grid.halo, "data": grid.data.tolist()}
    if isinstance(grid, Grid3D):
        out["Z"] = grid.Z
    return out


def grid_from_dict(obj: dict):
    data = np.asarray(obj["data"], dtype=np.float64)
    grid = Grid3D(data, int(obj["halo"])) if data.ndim == 3 else Grid(data, int(obj["halo"]))
    if grid.A != obj["A"] or grid.B != obj["B"] or (data.ndim == 3 and grid.Z != obj.get("Z")):
        raise ValueError("grid JSON dims inconsistent with data payload")
    return grid


def save_grid_json(grid, path) -> None:
    Path(path).write_text(json.dumps(grid_to_dict(grid)))


def load_grid_json(path):
    return grid_from_dict(json.loads(Path(path).read_text()))


# ---------------------------------------------------------------------------
# kernels

def kernel_to_dict(kernel: StencilKernel) -> dict:
    return {"shape": kernel.shape.value, "d": kernel.d, "r": kernel.r, "coeffs": kernel.coeffs.tolist()}


def kernel_from_dict(obj: dict) -> StencilKernel:
    d = int(obj["d"])
    if d == 3:
        return make_kernel_3d(obj["shape"], int(obj["r"]), obj["coeffs"])
    return make_kernel(obj["shape"], d, int(obj["r"]), obj["coeffs"])


def save_kernel(kernel: StencilKernel, path) -> None:
    Path(path).write_text(json.dumps(kernel_to_dict(kernel), indent=2))


def load_kernel(path) -> StencilKernel:
    return kernel_from_dict(json.loads(Path(path).read_text()))


# ---------------------------------------------------------------------------
# compressed kernels (SPCK)

def _parity_code(parity: Parity) -> int:
    return 0 if Parity(parity) is Parity.EVEN else 1


def _parity_from_code(code: int) -> Parity:
    if code not in (0, 1):
        raise ValueError(f"bad parity code {code}")
    return Parity.EVEN if code == 0 else Parity.ODD


def compressed_record_bytes(ck: CompressedKernel) -> bytes:
    header = _COMPRESSED_HEADER.pack(COMPRESSED_MAGIC, ck.r, ck.L, _parity_code(ck.parity))
    body = np.ascontiguousarray(ck.values, dtype="<f8").tobytes()
    return header + body + bytes(metadata_to_bytes(ck.metadata))


def _record_from_buffer(raw: bytes, offset: int):
    if len(raw) - offset < _COMPRESSED_HEADER.size:
        raise ValueError("truncated compressed-kernel record")
    magic, r, L, code = _COMPRESSED_HEADER.unpack_from(raw, offset)
    if magic != COMPRESSED_MAGIC:
        raise ValueError(f"bad magic {magic!r}, expected {COMPRESSED_MAGIC!r}")
    pos = offset + _COMPRESSED_HEADER.size
    need = L * L * 8 + L * (L // 2)
    if len(raw) - pos < need:
        raise ValueError("truncated compressed-kernel record")
    values = np.frombuffer(raw, dtype="<f8", count=L * L, offset=pos).reshape(L, L)
    pos += L * L * 8
    meta = metadata_from_bytes(raw[pos : pos + L * (L // 2)], L, L // 2)
    pos += L * (L // 2)
    ck = CompressedKernel(values=values.astype(np.float64), metadata=meta, r=r, parity=_parity_from_code(code))
    return ck, pos


def save_compressed_set(kernels, path) -> None:
    with open(path, "wb") as fh:
        for ck in kernels:
            fh.write(compressed_record_bytes(ck))


def load_compressed_set(path) -> list:
    raw = Path(path).read_bytes()
    out, offset = [], 0
    while offset < len(raw):
        ck, offset = _record_from_buffer(raw, offset)
        out.append(ck)
    if not out:
        raise ValueError(f"{path}: no compressed-kernel records found")
    return out


def compressed_to_dict(ck: CompressedKernel) -> dict:
    return {"r": ck.r, "L": ck.L, "parity": Parity(ck.parity).value, "values": ck.values.tolist(),
            "metadata": np.asarray(ck.metadata).tolist()}


def compressed_from_dict(obj: dict) -> CompressedKernel:
    """Inverse of compressed_to_dict (reference transform.py:338-346): the
    metadata is validated (ascending pairs, in range) before use."""
    meta = np.asarray(obj["metadata"], dtype=np.uint8)
    validate_metadata(meta)
    return CompressedKernel(values=np.asarray(obj["values"], dtype=np.float64), metadata=meta, r=int(obj["r"]),
                            parity=Parity(obj["parity"]))


def save_compressed_json(kernels, path) -> None:
    Path(path).write_text(json.dumps([compressed_to_dict(ck) for ck in kernels], indent=2))


__all__ = [
    "save_grid", "load_grid", "grid_to_dict", "grid_from_dict", "save_grid_json", "load_grid_json",
    "kernel_to_dict", "kernel_from_dict", "save_kernel", "load_kernel",
    "compressed_record_bytes", "save_compressed_set", "load_compressed_set", "compressed_to_dict",
    "compressed_from_dict", "save_compressed_json",
]
