"""numpy restatement of the reference brute-force executor (TEST ONLY).

Follows reference core.py:151-182 step for step: taps in row-major kernel order
(rho outer, delta inner; for the 3D extension rho_z, rho_y, delta), an fp64
accumulator initialised to zero, `acc += w * shifted_slice` per tap, interior
write-back into a double buffer whose halo is never written.
"""
from __future__ import annotations

import numpy as np


def taps(coeffs: np.ndarray, d: int, r: int):
    """(offsets..., weight) in the reference's accumulation order (core.py:165-172)."""
    c = np.asarray(coeffs, dtype=np.float64).reshape((2 * r + 1,) * d)
    span = range(-r, r + 1)
    out = []
    if d == 1:
        for t, dx in enumerate(span):
            out.append(((dx,), float(c[t])))
    elif d == 2:
        for i, ry in enumerate(span):
            for j, dx in enumerate(span):
                out.append(((ry, dx), float(c[i, j])))
    else:
        for i, rz in enumerate(span):
            for j, ry in enumerate(span):
                for k, dx in enumerate(span):
                    out.append(((rz, ry, dx), float(c[i, j, k])))
    return out


def naive_apply(coeffs, d: int, r: int, data: np.ndarray, halo: int, steps: int) -> np.ndarray:
    """T Jacobi steps on a halo-padded array; returns the new padded array.

    d = 1 and 2 use the reference's 2D storage ((A+2h) x (B+2h), A = 1 for 1D);
    d = 3 uses (Z+2h) x (A+2h) x (B+2h).
    """
    if steps < 1:
        raise ValueError(f"step count must be >= 1, got {steps}")
    if halo < r:
        raise ValueError(f"grid halo {halo} too small for stencil radius {r}")
    h = halo
    cur = np.array(data, copy=True)
    nxt = cur.copy()
    dtype = cur.dtype
    tl = taps(coeffs, d, r)
    if d == 3:
        Z, A, B = (n - 2 * h for n in cur.shape)
    else:
        A, B = (n - 2 * h for n in cur.shape)
    for _ in range(steps):
        if d == 3:
            acc = np.zeros((Z, A, B), dtype=dtype)
            for (rz, ry, dx), w in tl:
                acc += w * cur[h + rz : h + rz + Z, h + ry : h + ry + A, h + dx : h + dx + B]
            nxt[h : h + Z, h : h + A, h : h + B] = acc
        else:
            acc = np.zeros((A, B), dtype=dtype)
            for off, w in tl:
                ry, dx = (0, off[0]) if d == 1 else off
                acc += w * cur[h + ry : h + ry + A, h + dx : h + dx + B]
            nxt[h : h + A, h : h + B] = acc
        cur, nxt = nxt, cur
    return cur


def max_rel_error(got, want) -> float:
    """Reference parity metric (pipeline.py:265-267)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(float(np.max(np.abs(want))), 1e-300)
    return float(np.max(np.abs(got - want)) / scale)
