"""The C-ABI library loads on a CPU-only box and exports every entry point
include/spider.h declares (no compute calls here)."""
import ctypes
import re
from pathlib import Path

import paper_2506_22035_b200._lib as L

HEADER = Path(__file__).resolve().parents[1] / "include" / "spider.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spd_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_surface():
    names = declared_functions()
    assert len(names) >= 25
    for must in ("spd_plan_create", "spd_run", "spd_transform_row", "spd_naive_apply_f64", "spd_mma_selftest"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(L.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_covers_header():
    assert set(declared_functions()) == set(L.SIGNATURES)


def test_abi_version():
    assert L.lib.spd_abi_version() == 1
