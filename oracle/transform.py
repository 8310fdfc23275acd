"""numpy restatement of the reference AOT transform (TEST ONLY).

reference transform.py:37-267 and pipeline.py:128-144.
"""
from __future__ import annotations

import numpy as np


def band_rows(r: int) -> int:  # transform.py:37-41
    if r < 1:
        raise ValueError(f"radius must be >= 1, got {r}")
    return 2 * r + 2


def permutation(L: int, parity: int) -> np.ndarray:  # transform.py:130-139
    if L % 2:
        raise ValueError(f"L must be even, got {L}")
    m = np.arange(2 * L, dtype=np.int64)
    for j in range(parity, L, 2):
        m[j], m[j + L] = j + L, j
    return m


def kernel_matrix(row, r: int) -> np.ndarray:  # transform.py:118-127
    L = band_rows(r)
    row = np.asarray(row, dtype=np.float64).ravel()
    K = np.zeros((L, 2 * L))
    for i in range(L):
        K[i, i : i + 2 * r + 1] = row
    return K


def swap(K: np.ndarray, parity: int) -> np.ndarray:  # transform.py:142-160
    return K[:, permutation(K.shape[1] // 2, parity)]


def check_2to4(K: np.ndarray):  # transform.py:163-180
    rows, width = K.shape
    cnt = (K.reshape(rows, width // 4, 4) != 0.0).sum(axis=2)
    return [(int(i), int(s)) for i, s in np.argwhere(cnt > 2)]


def encode_segment(seg):  # transform.py:183-205
    seg = np.asarray(seg, dtype=np.float64)
    nz = [t for t in range(4) if seg[t] != 0.0]
    if len(nz) > 2:
        raise ValueError("2:4 violated")
    if len(nz) == 2:
        return float(seg[nz[0]]), float(seg[nz[1]]), nz[0], nz[1]
    if len(nz) == 1:
        p = nz[0]
        return (float(seg[p]), 0.0, p, p + 1) if p < 3 else (0.0, float(seg[3]), 2, 3)
    return 0.0, 0.0, 0, 1


def encode(Ksw: np.ndarray):  # transform.py:208-223
    rows, width = Ksw.shape
    segs = width // 4
    vals = np.zeros((rows, 2 * segs))
    meta = np.zeros((rows, segs, 2), dtype=np.uint8)
    for i in range(rows):
        for s in range(segs):
            v0, v1, p0, p1 = encode_segment(Ksw[i, 4 * s : 4 * s + 4])
            vals[i, 2 * s : 2 * s + 2] = (v0, v1)
            meta[i, s] = (p0, p1)
    return vals, meta


def decode(vals: np.ndarray, meta: np.ndarray) -> np.ndarray:  # transform.py:236-246
    rows, segs = meta.shape[:2]
    out = np.zeros((rows, 4 * segs))
    for i in range(rows):
        for s in range(segs):
            for t in range(2):
                out[i, 4 * s + meta[i, s, t]] = vals[i, 2 * s + t]
    return out


def metadata_bytes(meta: np.ndarray) -> bytes:  # transform.py:253-257
    m = np.asarray(meta, dtype=np.uint8)
    return (m[..., 0] | (m[..., 1] << 2)).astype(np.uint8).tobytes()


def transform_row(row, r: int, parity: int):  # pipeline.py:135-137
    return encode(swap(kernel_matrix(row, r), parity))
