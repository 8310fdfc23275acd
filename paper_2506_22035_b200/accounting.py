"""Reference execution counters that do not depend on the device.

`execute` returns an `ExecStats` whose reference keys must carry the
reference's values: the block/warp tile plan of the
Ampere-era model (reference tiling.py:36-149, pipeline.py:146-173) and the
coalescing metric of the kernel-operand fetch stream (tiling.py:348-383,
pipeline.py:215-219).  These are integer formulas of the reference's cost
model, restated here; the B200 engine's own tiling is reported separately
under `ExecStats.device`.
"""
from __future__ import annotations

from dataclasses import dataclass

from .transform import band_rows

WARP_LANES = 32
FRAGMENT_ELEMENTS = 4


@dataclass(frozen=True)
class MmaShape:
    """Instruction tile of the reference's model (sptc.py:23-38); the default
    m16n8k16 is the sm_80 `mma.sp` shape the reference counts in."""

    m: int = 16
    n: int = 8
    k: int = 16

    def __post_init__(self) -> None:
        if self.k % 4 != 0:
            raise ValueError(f"K dimension must be divisible by 4, got {self.k}")
        if self.m < 1 or self.n < 1:
            raise ValueError("MMA dimensions must be positive")


MMA_M16N8K16 = MmaShape(16, 8, 16)


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def tile_plan(A: int, B: int, r: int, a_block: int, b_block: int, a_warp: int, b_warp: int, mma: MmaShape) -> dict:
    """Validated three-level tile plan quantities (reference tiling.py:113-149)."""
    if r < 1:
        raise ValueError(f"radius must be >= 1, got {r}")
    if a_warp % mma.m != 0:
        raise ValueError(f"warp tile rows {a_warp} not a multiple of M_mma {mma.m}")
    if b_warp % mma.n != 0:
        raise ValueError(f"warp tile cols {b_warp} not a multiple of N_mma {mma.n}")
    if a_block % a_warp != 0:
        raise ValueError(f"block tile rows {a_block} not a multiple of warp rows {a_warp}")
    if b_block % b_warp != 0:
        raise ValueError(f"block tile cols {b_block} not a multiple of warp cols {b_warp}")
    if a_block > A or b_block > B:
        raise ValueError(f"block tile {a_block}x{b_block} exceeds problem size {A}x{B}")
    if A % a_block != 0 or B % b_block != 0:
        raise ValueError("problem size must split into whole block tiles")
    L = band_rows(r)
    inv_k = _ceil_div(2 * L, mma.k)
    return {
        "block_tiles": (A // a_block) * (B // b_block),
        "warps_per_block": (a_block // a_warp) * (b_block // b_warp),
        "invocations_per_warp_pass": (a_warp // mma.m) * (b_warp // mma.n) * inv_k,
        "shared_input_elements": (a_block + 2 * r) * b_block,
    }


def _auto_tile(n: int, unit: int, cap: int = 64):
    """Largest multiple of `unit` up to `cap` dividing n (pipeline.py:146-151)."""
    best = None
    for d in range(unit, min(n, cap) + 1, unit):
        if n % d == 0:
            best = d
    return best


def tile_counts(d: int, r: int, A: int, B: int, cfg) -> dict:
    """`ExecStats.tile_counts` (reference pipeline.py:154-173).  Raises
    ValueError for explicit block tiles that do not fit the grid, like the
    reference's execute."""
    if d == 1:
        return {"block_tiles": 1}
    a_block = cfg.a_block or _auto_tile(A, cfg.a_warp)
    b_block = cfg.b_block or _auto_tile(B, cfg.b_warp)
    explicit = cfg.a_block is not None or cfg.b_block is not None
    if a_block is None or b_block is None:
        if explicit:
            raise ValueError("explicit block tiles incompatible with grid size")
        return {}
    return tile_plan(A, B, r, a_block, b_block, cfg.a_warp, cfg.b_warp, cfg.mma)


def run_count(addresses) -> int:
    """Maximal consecutive-ascending runs in an address stream (tiling.py:348-357)."""
    addrs = list(addresses)
    if not addrs:
        return 0
    return 1 + sum(1 for prev, cur in zip(addrs, addrs[1:]) if cur != prev + 1)


def kernel_fetch_addresses(L: int, packed: bool, mma: MmaShape = MMA_M16N8K16) -> list:
    """Warp fetch addresses of the whole kernel operand in issue order
    (tiling.py:360-383): packed indexes the fragment-ordered buffer, unpacked
    the row-major L x L values (instruction padding issues no fetch)."""
    if (mma.m, mma.n, mma.k) != (16, 8, 16):
        raise ValueError("packed layouts are defined for the 16x8x16 instruction")
    invocations = _ceil_div(2 * L, mma.k)
    k_half = mma.k // 2
    addrs = []
    for k in range(invocations):
        for lane in range(WARP_LANES):
            for e in range(FRAGMENT_ELEMENTS):
                if packed:
                    addrs.append(k * WARP_LANES * FRAGMENT_ELEMENTS + lane * FRAGMENT_ELEMENTS + e)
                    continue
                # kernel_fragment_slot (tiling.py:188-194)
                row, local = lane // 4 + 8 * (e // 2), 2 * (lane % 4) + (e % 2)
                col = k * k_half + local
                if row < L and col < L:
                    addrs.append(row * L + col)
    return addrs


def fetch_runs(L: int, packing: bool, mma: MmaShape = MMA_M16N8K16) -> tuple:
    """(fetch_runs_packed, fetch_runs_unpacked, fetch_runs_active) (pipeline.py:215-219)."""
    packed = run_count(kernel_fetch_addresses(L, True, mma))
    unpacked = run_count(kernel_fetch_addresses(L, False, mma))
    return packed, unpacked, packed if packing else unpacked


__all__ = ["MmaShape", "MMA_M16N8K16", "tile_plan", "tile_counts", "run_count", "kernel_fetch_addresses",
           "fetch_runs"]
