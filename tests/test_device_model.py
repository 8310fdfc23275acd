"""CPU model of one device tile, built from the plan's real packed operands.

The host-only plan (device=-1) exposes exactly what libspider uploads: the
compressed A values [S,128,16] (fp16 bits), the E metadata words [S,128] in the
TMEM lane/bit layout, the MMA start rows and the tile geometry.  This test
decodes them with the hardware semantics pinned by tools/umma_sp_probe.cu
(metadata lane = m0 + 8*k1 + 16*m2, bits 16*m1 + 4*c, nibble idx0|idx1<<2),
rebuilds the B operand the producer warps stage (2L windows, involution from
transform.py:130-139), runs D = sum_s A_s @ B_s in fp64 and compares with the
oracle.  It checks geometry, packing and the permutation logic without a GPU.
"""
import numpy as np
import pytest

import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import Plan
from oracle import naive


def decode_A(a_img, e_words):
    S = a_img.shape[0]
    vals = a_img.view(np.float16).astype(np.float64)
    nib = np.zeros((S, 128, 8), dtype=np.int64)
    for lane in range(128):
        m0, k1, m2 = lane % 8, (lane // 8) % 2, lane // 16
        for m1 in (0, 1):
            for c4 in range(4):
                m = m0 + 8 * m1 + 16 * m2
                nib[:, m, 4 * k1 + c4] = (e_words[:, lane].astype(np.int64) >> (16 * m1 + 4 * c4)) & 0xF
    A = np.zeros((S, 128, 32))
    p0, p1 = nib & 3, nib >> 2
    assert np.all(p0 < p1), "metadata must be ascending pairs"
    for s in range(S):
        for m in range(128):
            for seg in range(8):
                A[s, m, 4 * seg + p0[s, m, seg]] += vals[s, m, 2 * seg]
                A[s, m, 4 * seg + p1[s, m, seg]] += vals[s, m, 2 * seg + 1]
    return A


def tile_model(plan, dense, halo):
    kern = plan.kernel
    inf = plan.info()
    r = inf.r_dev or kern.r  # device radius: a radius-2 stencil runs embedded as radius 3
    L, n_tile = inf.L, inf.n_tile * (2 if inf.cg2 else 1)  # a CTA pair spans both x-halves
    a_img, e_words, starts = plan.operands()
    in_off, out_off = plan.geometry()
    lanes = plan.lane_map()  # accumulator row of (output row a, chunk position i)
    perm = sp.input_row_permutation(L, plan.parity).mapping
    A = decode_A(a_img, e_words)
    dense3 = dense if dense.ndim == 3 else dense[None]
    zh = halo if dense.ndim == 3 else 0
    kslots = 8 * inf.kchunks  # window slots per input row (2L padded with zeros)
    Bimg = np.zeros((inf.r_in, n_tile, kslots))
    for b in range(inf.r_in):
        dz, dy, dx = in_off[b]
        for n in range(n_tile):
            for q in range(2 * L):
                x = dx + n * L - r + perm[q]
                zz, yy, xx = dz + zh, dy + halo, x + halo
                if 0 <= zz < dense3.shape[0] and 0 <= yy < dense3.shape[1] and 0 <= xx < dense3.shape[2]:
                    Bimg[b, n, q] = dense3[zz, yy, xx]
    rpm = 32 // kslots
    out = {}
    # M-tile t runs the same MMA schedule (same A/E) on B rows shifted by
    # t * mt_rows and produces output rows t * r_out ..
    # CTA-pair mode: rank t runs every K-block with its own A images
    # An M = 64 MMA (half 1 / 2) only writes lanes 0-15 / 16-31 of each
    # quadrant: the model drops its rows on the other lanes, so a wrong half
    # assignment loses coefficients and breaks the comparison with the oracle.
    halves = plan.mma_halves()
    lane_half = np.where(np.arange(128) % 32 < 16, 1, 2)
    for t in range(2 if inf.cg2 else inf.m_tiles):
        D = np.zeros((128, n_tile))
        for s in range(inf.mmas_per_tile):
            b0 = starts[s] + (0 if inf.cg2 else t * inf.mt_rows)
            Bs = Bimg[b0 : b0 + rpm].transpose(0, 2, 1).reshape(32, n_tile)
            As = A[t * inf.mmas_per_tile + s if inf.cg2 else s]
            if halves[s]:
                As = np.where((lane_half == halves[s])[:, None], As, 0.0)
            D += As @ Bs
        for a in range(inf.r_out):
            dz, dy, dx = out_off[a + t * inf.r_out]
            for i in range(L):
                for n in range(n_tile):
                    out[(dz, dy, dx + n * L + i)] = D[lanes[L * a + i], n]
    return out


def f16(x):
    return np.asarray(x, dtype=np.float64).astype(np.float16).astype(np.float64)


CASES = [
    ("box", 2, 1),
    ("star", 2, 1),
    ("box", 2, 3),
    ("star", 2, 3),
    ("box", 3, 1),
    ("box", 1, 1),
    ("box", 1, 3),
    # generic radii (padded K-chunks, R_out = 128 // L)
    ("box", 2, 2),
    ("star", 2, 2),
    ("box", 2, 4),
    ("box", 2, 5),
    ("box", 2, 6),
    ("box", 2, 7),
    ("box", 1, 2),
    ("box", 1, 5),
]


@pytest.mark.parametrize("shape,d,r", CASES)
@pytest.mark.parametrize("parity", ["even", "odd"])
def test_tile_model_matches_oracle(shape, d, r, parity):
    rng = np.random.default_rng([d, r, 11])
    span = 2 * r + 1
    coeffs = rng.uniform(-1, 1, (span,) * d)
    if shape == "star" and d >= 2:
        mask = np.zeros_like(coeffs, dtype=bool)
        mask[r, :] = True
        mask[:, r] = True
        coeffs = np.where(mask, coeffs, 0.0)
    kern = sp.make_kernel_3d(shape, r, coeffs) if d == 3 else sp.make_kernel(shape, d, r, coeffs)
    plan = Plan(kern, parity, "fp16", device=-1)
    inf = plan.info()
    L = inf.L
    in_off, out_off = plan.geometry()
    if d == 3:
        shape3 = (inf.tile_z, inf.tile_y, inf.n_tile * L * (2 if inf.cg2 else 1))
    elif d == 2:
        shape3 = (inf.tile_y, inf.n_tile * L)
    else:
        shape3 = (1, inf.n_tile * L * inf.r_out)
    dense = f16(rng.uniform(-1, 1, tuple(s + 2 * r for s in shape3)))
    got = tile_model(plan, dense, r)
    want = naive.naive_apply(f16(coeffs), d, r, dense, r, 1)
    h = r
    err = 0.0
    for (z, y, x), v in got.items():
        w = want[z + h, y + h, x + h] if d == 3 else want[y + h, x + h]
        err = max(err, abs(v - w))
    assert len(got) == int(np.prod(shape3))
    assert err < 1e-12, err


def test_operand_bits_are_fp16_coefficients():
    k = sp.make_kernel("box", 2, 1, np.arange(1, 10) / 7.0)
    plan = Plan(k, "even", "fp16", device=-1)
    a_img, e_words, starts = plan.operands()
    vals = set(np.unique(a_img.view(np.float16).astype(np.float64)))
    want = set(f16(np.arange(1, 10) / 7.0)) | {0.0}
    assert vals <= want and vals >= want - {0.0}
    assert list(starts) == [0, 4, 8, 12, 16, 20, 24, 28, 30]


def test_bf16_operands():
    k = sp.make_kernel("box", 2, 1, np.full(9, 1 / 3))
    plan = Plan(k, "even", "bf16", device=-1)
    a_img, _, _ = plan.operands()
    nz = a_img[a_img != 0]
    # 1/3 in bf16 = 0x3EAB
    assert set(nz.tolist()) == {0x3EAB}


def test_unsupported_radius_rejected_by_device_plan():
    k = sp.make_kernel("box", 2, 8, np.ones(17 * 17))
    with pytest.raises(ValueError, match="unsupported"):
        Plan(k, "even", "fp16", device=-1)
    k3 = sp.make_kernel_3d("box", 2, np.ones(125))
    with pytest.raises(ValueError, match="unsupported"):
        Plan(k3, "even", "fp16", device=-1)


def test_lane_map_is_a_permutation():
    """L = 4 one-M-tile plans (2D, 1D) put output row a, chunk position i on
    accumulator lane 32*(j%4) + 16*(j/4) + 2*(a%4) + (i>>1) + 8*(i&1), j = a/4
    (the epilogue's tcgen05.ld.16x256b order; rows 0-15 on lanes 0-15 of the
    quadrants, rows 16-31 on lanes 16-31); 3D and other radii keep
    m = L*a + i."""
    for d, r in ((2, 1), (3, 1), (1, 1), (2, 3), (2, 2)):
        c = np.ones((2 * r + 1,) * d)
        kern = sp.make_kernel_3d("box", r, c) if d == 3 else sp.make_kernel("box", d, r, c)
        plan = Plan(kern, "even", "fp16", device=-1)
        inf = plan.info()
        lanes = plan.lane_map()
        assert sorted(lanes) == list(range(inf.r_out * inf.L))
        for a in range(inf.r_out):
            for i in range(inf.L):
                rows16 = 16 // inf.L
                j = a // rows16
                pair = 32 * (j % 4) + 16 * (j // 4) + (inf.L // 2) * (a % rows16) + (i >> 1) + 8 * (i & 1)
                if inf.L == 4 and inf.m_tiles == 1 and not inf.cg2:
                    assert lanes[inf.L * a + i] == pair
                elif inf.L == 8:
                    assert lanes[inf.L * a + i] == 32 * ((a % 8) // 2) + 16 * (a // 8) + 8 * (a % 2) + i
                elif d == 3:
                    z, y = a // 8, a % 8
                    assert lanes[inf.L * a + i] == 32 * (y // 2) + 16 * (z // 2) + 4 * (2 * (z % 2) + y % 2) + i
                else:
                    assert lanes[inf.L * a + i] == inf.L * a + i


def test_radius2_embeds_as_radius3():
    """1D / 2D radius 2 runs on the L = 8 fast path (zero ring); SPD_NO_EMBED
    keeps the generic L = 6 geometry."""
    import os

    for d in (1, 2):
        c = np.ones((5,) * d)
        kern = sp.make_kernel("box", d, 2, c)
        inf = Plan(kern, "even", "fp16", device=-1).info()
        assert inf.L == 8 and inf.r_dev == 3
        os.environ["SPD_NO_EMBED"] = "1"
        try:
            inf = Plan(kern, "even", "fp16", device=-1).info()
        finally:
            del os.environ["SPD_NO_EMBED"]
        assert inf.L == 6 and inf.r_dev == 2


def test_mma_halves():
    """K-blocks that feed only one half of the accumulator lanes run as M = 64
    MMAs (aot.cpp assign_mma_halves): every nonzero A row of such an MMA sits
    on that half; MMA 0 (accumulate = 0) is always M = 128; CTA-pair plans
    issue M = 128 only.  Expected schedules: 2D r = 1 (34 input
    rows, 4 per MMA) splits at output row 16; 3D r = 1 (z-planes 0-1 on lanes
    0-15 of each quadrant, 2-3 on lanes 16-31) has 9 of 15 half MMAs."""
    lane_half = np.where(np.arange(128) % 32 < 16, 1, 2)
    for d, r, want in ((2, 1, [0, 1, 1, 1, 0, 2, 2, 2, 2]), (1, 1, [0, 1, 1, 1, 2, 2, 2, 2]),
                       (3, 1, [0, 1, 1, 1, 1, 0, 0, 0, 0, 0, 2, 2, 2, 2, 2]),
                       (2, 3, [0, 1, 1, 1, 0, 0, 0, 2, 2, 2, 2]), (1, 3, [0, 1, 1, 1, 2, 2, 2, 2]),
                       (2, 2, [0, 1, 1, 1, 0, 0, 0, 2, 2, 2, 2]), (2, 5, None)):
        c = np.ones((2 * r + 1,) * d)
        kern = sp.make_kernel_3d("box", r, c) if d == 3 else sp.make_kernel("box", d, r, c)
        plan = Plan(kern, "even", "fp16", device=-1)
        halves = plan.mma_halves()
        if want is not None:
            assert list(halves) == want
        assert halves[0] == 0
        a_img, _, _ = plan.operands()
        for s, h in enumerate(halves):
            if h:
                nz = np.any(a_img[s] != 0, axis=1)
                assert np.all(lane_half[nz] == h), (d, r, s)
    k3 = sp.make_kernel_3d("box", 1, np.ones(27))
    assert not np.any(Plan(k3, "even", "fp16", device=-1, cta_pair=True).mma_halves())
