"""ctypes binding of libspider.so (C ABI declared in include/spider.h).

The library is mandatory: there is no Python or CPU fallback for any entry
point.  Importing this module on a box without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
# SPD_LIB: development override (A/B timing of two builds); default in-tree
LIB_PATH = Path(os.environ["SPD_LIB"]) if os.environ.get("SPD_LIB") else _HERE / "libspider.so"

SPD_OK = 0
SPD_EINVAL = -1
SPD_ECUDA = -2
SPD_EUNSUPPORTED = -3

DTYPE_CODES = {"fp16": 0, "bf16": 1}


class SpiderError(RuntimeError):
    """A CUDA failure inside libspider (SPD_ECUDA)."""


class spd_grid_desc(C.Structure):
    _fields_ = [
        ("nz", C.c_int64),
        ("ny", C.c_int64),
        ("nx", C.c_int64),
        ("halo", C.c_int32),
        ("dims", C.c_int32),
        ("pitch", C.c_int64),
        ("plane", C.c_int64),
        ("origin", C.c_int64),
        ("alloc_elems", C.c_int64),
    ]


_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_D = C.POINTER(C.c_double)
_U8 = C.POINTER(C.c_uint8)
_U16 = C.POINTER(C.c_uint16)
_U32 = C.POINTER(C.c_uint32)
_I32 = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_DESC = C.POINTER(spd_grid_desc)

# name -> (restype, argtypes); the list is the exported C ABI of spider.h.
SIGNATURES = {
    "spd_last_error": (C.c_char_p, []),
    "spd_abi_version": (_I, []),
    "spd_band_rows": (_I, [_I]),
    "spd_row_permutation": (_I, [_I, _I, _I64P]),
    "spd_build_kernel_matrix": (_I, [_I, _D, _D]),
    "spd_swap_columns": (_I, [_D, _I, _I, _I, _D]),
    "spd_check_2to4": (_I, [_D, _I, _I, _I32, _I]),
    "spd_encode_segment": (_I, [_D, _D, _U8]),
    "spd_encode": (_I, [_D, _I, _I, _D, _U8]),
    "spd_decode": (_I, [_D, _U8, _I, _I, _D]),
    "spd_metadata_to_bytes": (_I, [_U8, _I, _U8]),
    "spd_transform_row": (_I, [_I, _I, _D, _D, _U8]),
    "spd_plan_create": (_I, [_I, _I, _I, _D, _I, _I, C.POINTER(_P)]),
    "spd_plan_create_ex": (_I, [_I, _I, _I, _D, _I, _I, _I, C.POINTER(_P)]),
    "spd_plan_destroy": (_I, [_P]),
    "spd_plan_info": (_I, [_P, _I32]),
    "spd_plan_operands": (_I, [_P, _U16, _U32, _I32]),
    "spd_plan_geometry": (_I, [_P, _I32, _I32]),
    "spd_plan_lane_map": (_I, [_P, _I32]),
    "spd_plan_mma_halves": (_I, [_P, _I32]),
    "spd_grid_layout": (_I, [_P, _I64, _I64, _I64, _I, _DESC]),
    "spd_run": (_I, [_P, _DESC, _P, _P, _I, _P]),
    "spd_run_ex": (_I, [_P, _DESC, _P, _P, _I, _I, _P]),
    "spd_step_range": (_I, [_P, _DESC, _P, _P, _I64, _I64, _P]),
    "spd_step_edges": (_I, [_P, _DESC, _P, _P, _P]),
    "spd_step_ordered": (_I, [_P, _DESC, _P, _P, _P, _I, _P, _I, _P]),
    "spd_step_edge_first": (_I, [_P, _DESC, _P, _P, _I, _P, _I, _P]),
    "spd_pack_grid": (_I, [_DESC, _I, _P, _P, _P]),
    "spd_unpack_grid": (_I, [_DESC, _I, _P, _P, _P]),
    "spd_upload": (_I, [_DESC, _P, _P, _P]),
    "spd_download": (_I, [_DESC, _P, _P, _P]),
    "spd_download_rows": (_I, [_DESC, _P, _P, _I64, _I64, _P]),
    "spd_upload_staged": (_I, [_DESC, _P, _P, _P, _P]),
    "spd_download_staged": (_I, [_DESC, _P, _P, _P, _P]),
    "spd_copy_halo": (_I, [_DESC, _P, _P, _P]),
    "spd_naive_apply_f64": (_I, [_I, _I, _D, _I64, _I64, _I64, _I, _P, _P, _P, _I, _P]),
    "spd_mma_selftest": (_I, [_P, _P, _P, _I, _P, _P]),
    "spd_halo_pack": (_I, [_DESC, _P, _I, _I, _P, _P]),
    "spd_halo_unpack": (_I, [_DESC, _P, _I, _I, _P, _P]),
    "spd_ipc_export": (_I, [_P, _P, _I64P]),
    "spd_ipc_open": (_I, [_P, C.c_int64, C.POINTER(_P), C.POINTER(_P)]),
    "spd_ipc_close": (_I, [_P]),
    "spd_slab_create": (_I, [_P, _DESC, _P, _P, _P, _P, _P, _DESC, _P, _P, _P, _DESC, _P, C.POINTER(_P)]),
    "spd_slab_step": (_I, [_P, _I, _P, _P]),
    "spd_slab_destroy": (_I, [_P]),
    "spd_slab_run": (_I, [_P, _I, _I, _P, _P]),
    "spd_peer_enable": (_I, [_I, _I]),
}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2506_22035_b200/build.py` "
            "(or __graft_entry__.build()); there is no fallback path"
        )
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("SPD_LIB") and not hasattr(lib, name):
            continue  # development override: an older build may lack newer entry points
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> int:
    """Map a C status code to the reference's exception types."""
    if rc >= 0:
        return rc
    msg = (lib.spd_last_error() or b"").decode(errors="replace")
    if rc in (SPD_EINVAL, SPD_EUNSUPPORTED):
        raise ValueError(msg)
    raise SpiderError(msg)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_D)


def u8ptr(a: np.ndarray):
    return a.ctypes.data_as(_U8)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_I64P)


def i32ptr(a: np.ndarray):
    return a.ctypes.data_as(_I32)


def u16ptr(a: np.ndarray):
    return a.ctypes.data_as(_U16)


def u32ptr(a: np.ndarray):
    return a.ctypes.data_as(_U32)
