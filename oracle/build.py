"""Builds oracle/liboracle.so from oracle/naive.c with gcc (TEST ONLY)."""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "naive.c"
LIB = HERE / "liboracle.so"


def build(force: bool = False) -> Path:
    if not force and LIB.exists() and LIB.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run(
        ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread",
         "-o", str(tmp), str(SRC)],
        check=True,
    )
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
