"""Device parity: the sm_100a sparse-tensor-core path against the CPU oracle.

Tolerances (fp16 storage, fp32 tensor-core accumulation), on
max|got-want|/max|want| (reference pipeline.py:265-267) against the fp64
oracle run on identically quantised inputs:
  * one step, fp16-rounded coefficients in the oracle too: every point within
    one fp16 rounding of the exact value (0.5 ulp + 1e-6 of the row scale)
  * T <= 4 steps vs the fp64-coefficient oracle: 1e-2 (fp16), 5e-2 (bf16)
Device naive_apply (fp64) is bit-identical to the oracle.
"""
import numpy as np
import pytest
import torch

import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid, mma_selftest
from paper_2506_22035_b200.pipeline import DeviceConfig, get_plan, max_rel_error
from oracle import cnaive

pytestmark = pytest.mark.gpu

TOL = {"fp16": 1e-2, "bf16": 5e-2}


def quant(x, dtype="fp16"):
    t = torch.from_numpy(np.array(x, dtype=np.float64))
    return t.to(torch.float16 if dtype == "fp16" else torch.bfloat16).to(torch.float64).numpy()


def heat2d(alpha=0.125):
    c = np.zeros((3, 3))
    c[1, 1] = 1 - 4 * alpha
    c[0, 1] = c[2, 1] = c[1, 0] = c[1, 2] = alpha
    return c


def heat3d(alpha=1 / 12):
    c = np.zeros((3, 3, 3))
    c[1, 1, 1] = 1 - 6 * alpha
    for a in ((0, 1, 1), (2, 1, 1), (1, 0, 1), (1, 2, 1), (1, 1, 0), (1, 1, 2)):
        c[a] = alpha
    return c


def rand_kernel(shape, d, r, seed):
    rng = np.random.default_rng(seed)
    n = 2 * r + 1
    c = rng.uniform(-1, 1, (n,) * d)
    if shape == "star" and d >= 2:
        m = np.zeros_like(c, dtype=bool)
        m[(r,) * (d - 1)] = True
        for ax in range(d):
            idx = [r] * d
            idx[ax] = slice(None)
            m[tuple(idx)] = True
        c = np.where(m, c, 0.0)
    return sp.make_kernel_3d(shape, r, c) if d == 3 else sp.make_kernel(shape, d, r, c)


def run_case(kern, shape, steps, dtype="fp16", parity="even", seed=0):
    h = kern.r
    rng = np.random.default_rng(seed)
    data = quant(rng.uniform(-1, 1, tuple(s + 2 * h for s in shape)), dtype)
    grid = sp.Grid3D(data, h) if kern.d == 3 else sp.Grid(data, h)
    got, stats = sp.execute(kern, grid, steps, DeviceConfig(parity=parity, dtype=dtype))
    want = cnaive.naive_apply(kern.coeffs, kern.d, kern.r, data, h, steps)
    return got, want, grid, stats


# --------------------------------------------------------------------------
def test_mma_selftest_matches_decode():
    rng = np.random.default_rng(3)
    for n in (8, 64, 128, 256):
        vals = rng.integers(-3, 4, (128, 16)).astype(np.float16)
        nib = np.zeros((128, 8), dtype=np.uint8)
        A = np.zeros((128, 32))
        for m in range(128):
            for s in range(8):
                p = np.sort(rng.choice(4, 2, replace=False))
                nib[m, s] = p[0] | (p[1] << 2)
                A[m, 4 * s + p[0]] = vals[m, 2 * s]
                A[m, 4 * s + p[1]] = vals[m, 2 * s + 1]
        B = rng.integers(-4, 5, (32, n)).astype(np.float16)
        D = mma_selftest(vals.view(np.uint16), nib, B.view(np.uint16))
        np.testing.assert_array_equal(D, (A @ B.astype(np.float64)).astype(np.float32))


def test_device_naive_bit_exact_vs_oracle(golden):
    g = golden("naive_golden.npz")
    for c in range(int(g["n_cases"])):
        d, r, steps, star = (int(v) for v in g[f"c{c}_meta"])
        coeffs = g[f"c{c}_coeffs"]
        k = sp.make_kernel("star" if star else "box", d, r, coeffs)
        out = sp.naive_apply(k, sp.Grid(g[f"c{c}_in"].copy(), r), steps)
        np.testing.assert_array_equal(out.data, g[f"c{c}_out"])


def test_device_naive_3d_pins(golden):
    g = golden("naive3d_golden.npz")
    k = sp.make_kernel_3d("box", 1, g["a_coeffs"])
    out = sp.naive_apply(k, sp.Grid3D(g["a_in"].copy(), 1), 1)
    np.testing.assert_array_equal(out.data, g["a_out"])


def test_s5_oracle_config(golden):
    """Star-2D5P (Heat-2D) 512^2, 4 steps — BASELINE configs[0]."""
    g = golden("naive_golden.npz")
    k = sp.make_kernel("star", 2, 1, g["s5_coeffs"])
    grid = sp.random_grid(512, 512, 1, seed=[1, 512, 512])
    # the device naive path reproduces the reference oracle exactly
    ref = sp.naive_apply(k, grid, 4)
    np.testing.assert_array_equal(ref.data[240:272, 240:272], g["s5_center"])
    q = sp.Grid(quant(grid.data), 1)
    got, stats = sp.execute(k, q, 4)
    want = cnaive.naive_apply(k.coeffs, 2, 1, q.data, 1, 4)
    err = max_rel_error(got.interior, want[1:-1, 1:-1])
    assert err < TOL["fp16"], err
    assert stats.dense_macs == 2 * stats.total_macs


@pytest.mark.parametrize("shape,d,r,dims", [
    ("box", 2, 1, (64, 512)),
    ("star", 2, 1, (37, 200)),      # ragged: partial tiles in y and x
    ("box", 2, 3, (48, 136)),
    ("star", 2, 3, (17, 64)),
    ("box", 3, 1, (9, 20, 72)),
    ("star", 3, 1, (4, 8, 256)),
    ("box", 1, 1, (1, 1000)),
    ("box", 1, 3, (1, 16384 + 40)),
    # generic radii (L = 2r+2 not in {4, 8})
    ("box", 2, 2, (50, 390)),
    ("star", 2, 2, (64, 768)),
    ("box", 2, 4, (30, 700)),
    ("box", 2, 5, (25, 840)),
    ("box", 2, 6, (20, 1064)),
    ("star", 2, 7, (17, 1024)),
    ("box", 1, 2, (1, 9000)),
    ("box", 1, 5, (1, 12000)),
])
@pytest.mark.parametrize("parity", ["even", "odd"])
def test_execute_matches_oracle(shape, d, r, dims, parity):
    k = rand_kernel(shape, d, r, seed=[d, r, 5])
    for steps in (1, 3):
        got, want, grid, _ = run_case(k, dims, steps, parity=parity, seed=steps)
        h = r
        gi = got.interior
        wi = want[h:-h, h:-h, h:-h] if d == 3 else want[h:-h, h:-h]
        err = max_rel_error(gi, wi)
        assert err < TOL["fp16"], (steps, err)
        # the halo is never written
        if d == 3:
            mask = np.ones(got.data.shape, bool)
            mask[h:-h, h:-h, h:-h] = False
        else:
            mask = np.ones(got.data.shape, bool)
            mask[h:-h, h:-h] = False
        np.testing.assert_array_equal(got.data[mask], grid.data[mask])


@pytest.mark.parametrize("d,r", [(2, 1), (2, 3), (3, 1), (1, 1), (2, 2), (2, 7), (1, 4)])
def test_single_step_within_one_fp16_rounding(d, r):
    """One step, fp16-rounded coefficients in the oracle: the device result is
    the fp16 rounding of an fp32-accumulated exact sum."""
    k = rand_kernel("box", d, r, seed=[d, r, 77])
    kq = quant(k.coeffs)
    L = 2 * r + 2
    dims = {1: (1, 96 * L * 16), 2: (40, 64 * L * 2 + 8 * L), 3: (8, 16, 256)}[d]
    got, _, grid, _ = run_case(k, dims, 1, seed=4)
    want = cnaive.naive_apply(kq, d, r, grid.data, r, 1)
    h = r
    gi = got.interior
    wi = want[h:-h, h:-h, h:-h] if d == 3 else want[h:-h, h:-h]
    ulp = np.spacing(np.abs(wi).astype(np.float16)).astype(np.float64)
    bound = 0.5 * ulp + 1e-6 * np.abs(wi).max()
    assert np.all(np.abs(gi - wi) <= bound), float(np.max(np.abs(gi - wi) / bound))


@pytest.mark.parametrize("d,r,dims", [(2, 1, (64, 256)), (2, 3, (32, 128)), (3, 1, (8, 16, 128))])
def test_bf16_matches_oracle(d, r, dims):
    k = rand_kernel("box", d, r, seed=[d, r, 9])
    got, want, grid, _ = run_case(k, dims, 2, dtype="bf16")
    h = r
    wi = want[h:-h, h:-h, h:-h] if d == 3 else want[h:-h, h:-h]
    assert max_rel_error(got.interior, wi) < TOL["bf16"]


def test_heat3d_and_contractive_100_steps():
    """Heat-3D, 100 steps (the B27 step count) on a small cube: measured bound."""
    k = sp.make_kernel_3d("star", 1, heat3d())
    got, want, grid, _ = run_case(k, (16, 24, 64), 100)
    err = max_rel_error(got.interior, want[1:-1, 1:-1, 1:-1])
    assert err < 2e-2, err


def test_identity_kernel_fixed_point_full_size():
    """10240^2 (the B9 size): the identity stencil is exact in fp16, so the
    device result must equal the input bit for bit (size-independent check)."""
    c = np.zeros((3, 3))
    c[1, 1] = 1.0
    k = sp.make_kernel("box", 2, 1, c)
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    dg = DeviceGrid(plan, (10240, 10240), 1)
    host = torch.randn(dg.dense_shape, dtype=torch.float16)
    dg.upload(host)
    dg.run(3)
    out = torch.empty_like(host)
    dg.download(out)
    torch.cuda.synchronize()
    assert torch.equal(out, host)


def test_linearity_full_size():
    """B9 shape, 2 steps: S(a*g1 + g2) == a*S(g1) + S(g2) within fp16 error."""
    k = rand_kernel("box", 2, 1, seed=1)
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    shape = (10240, 10240)
    outs = []
    g1 = torch.rand((10242, 10242), dtype=torch.float64, device="cuda") - 0.5
    g2 = torch.rand((10242, 10242), dtype=torch.float64, device="cuda") - 0.5
    for g in (g1, g2, 0.5 * g1 + g2):
        dg = DeviceGrid(plan, shape, 1)
        dg.load_dense_f64(g)
        dg.run(2)
        outs.append(dg.to_dense_f64())
    lhs, rhs = outs[2], 0.5 * outs[0] + outs[1]
    scale = lhs.abs().max().item()
    assert (lhs - rhs).abs().max().item() / scale < 1e-2


def test_step_range_composes_to_full_step():
    k = rand_kernel("box", 2, 1, seed=2)
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    dense = torch.rand((130 + 2, 512 + 2), dtype=torch.float64, device="cuda")
    a = DeviceGrid(plan, (130, 512), 1)
    b = DeviceGrid(plan, (130, 512), 1)
    a.load_dense_f64(dense)
    b.load_dense_f64(dense)
    a.run(1)
    b.step_range(0, 7)
    b.step_range(7, 100)
    b.step_range(100, 130)
    b.flip()
    assert torch.equal(a.bufs[a.cur], b.bufs[b.cur])


@pytest.mark.parametrize("d,r,shape", [(2, 3, (100, 264)), (2, 1, (37, 4096)), (3, 1, (9, 20, 72)), (1, 2, (1, 600))])
@pytest.mark.parametrize("staged", [False, True])
def test_upload_download_roundtrip(d, r, shape, staged):
    """Strided DMA and staged (linear DMA + repack kernel) transfers place
    every element, halo included, identically; the two are interchangeable."""
    k = rand_kernel("box", d, r, seed=3)
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    dg = DeviceGrid(plan, shape, r)
    host = torch.randn(dg.dense_shape, dtype=torch.float16).pin_memory()
    dg.upload(host, staged=staged)
    back = torch.empty_like(host).pin_memory()
    dg.download(back, staged=not staged)
    torch.cuda.synchronize()
    assert torch.equal(host, back)
    dense = dg.to_dense_f64().cpu()
    assert torch.equal(dense, host.to(torch.float64))
    dg.download(back.zero_(), staged=staged)
    torch.cuda.synchronize()
    assert torch.equal(host, back)


def test_reference_error_contract():
    k = sp.make_kernel("box", 2, 2, np.ones(25))
    with pytest.raises(ValueError, match="multiple"):
        sp.execute(k, sp.random_grid(32, 32, 2, seed=0), 1)  # 32 % L=6 != 0
    k8 = sp.make_kernel("box", 2, 8, np.ones(17 * 17))
    with pytest.raises(ValueError, match="halo"):
        sp.execute(rand_kernel("box", 2, 3, 0), sp.random_grid(32, 32, 1, seed=0), 1)
    with pytest.raises(ValueError, match="step"):
        sp.execute(rand_kernel("box", 2, 1, 0), sp.random_grid(32, 32, 1, seed=0), 0)
    with pytest.raises(ValueError, match="unsupported"):
        sp.execute(k8, sp.random_grid(36, 36, 8, seed=0), 1)


def test_verify_report():
    k = sp.make_kernel("star", 2, 1, heat2d())
    rep = sp.verify(k, [64, 128], seed=1, steps=2)
    assert rep["all_pass"], rep
    assert rep["cross_checks"]["parity_max_abs_diff"] < 1e-2
    assert sp.report_json(rep) == sp.report_json(sp.verify(k, [64, 128], seed=1, steps=2))


@pytest.mark.parametrize("d,shape,ranks", [(2, (160, 512), 2), (2, (224, 1024), 3), (3, (24, 16, 256), 2)])
def test_slab_driver_emulated_ranks_bit_exact(d, shape, ranks):
    """The slab driver's device path (band compute, halo pack/unpack) with
    `ranks` slabs emulated on one GPU equals the undecomposed run bit for bit
    (slab boundaries are tile-aligned, so every point sees the same MMAs)."""
    from paper_2506_22035_b200.distributed import DeviceSlabOps, SlabDriver, decompose, local_exchange

    k = rand_kernel("box", d, 1, seed=[d, 21])
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    h = 1
    dense = (torch.rand(tuple(n + 2 * h for n in shape), dtype=torch.float64, device="cuda") - 0.5)
    ref = DeviceGrid(plan, shape, h)
    ref.load_dense_f64(dense)
    steps = 5
    ref.run(steps)
    want = ref.to_dense_f64()
    band = plan.info().tile_z if d == 3 else plan.info().tile_y
    drivers = []
    for rk in range(ranks):
        slab = decompose(shape[0], ranks, rk, align=band)
        ops = DeviceSlabOps(plan, (slab.rows,) + tuple(shape[1:]), h)
        ops.grid.load_dense_f64(dense[slab.lo : slab.hi + 2 * h].contiguous())
        drivers.append(SlabDriver(slab, ops))
    for _ in range(steps):
        for drv in drivers:
            drv.step_boundary()
        for drv in drivers:
            drv.pack_messages()
        local_exchange(drivers)
        for drv in drivers:
            drv.unpack_messages()
        for drv in drivers:
            drv.step_interior_and_flip()
    for drv in drivers:
        got = drv.ops.grid.to_dense_f64()
        s = drv.slab
        assert torch.equal(got[h:-h], want[h + s.lo : h + s.hi]), (s.lo, s.hi)


@pytest.mark.parametrize(
    "d,r,shape,steps,sweep,lag",
    [
        (2, 1, (512, 512), 6, None, None),
        (2, 1, (100, 1000), 6, None, None),
        (3, 1, (16, 24, 128), 6, None, None),
        (1, 1, (1, 40000), 6, None, None),
        (2, 1, (1000, 2048), 13, 1, 2),
        (2, 1, (1000, 2048), 13, 4, 2),
        (2, 1, (1000, 2048), 13, 5, 3),
        (2, 1, (1000, 2048), 13, 13, 4),
        (2, 3, (600, 1024), 9, 4, 2),
        (2, 2, (300, 1536), 7, 3, 2),
        (3, 1, (64, 40, 256), 11, 3, 2),
        (1, 1, (1, 100000), 9, 4, 2),
    ],
)
@pytest.mark.timeout(180, method="thread")
def test_persistent_launch_matches_per_step(monkeypatch, d, r, shape, steps, sweep, lag):
    """One cooperative launch for all steps (sweep / wavefront order through
    L2, band-counter ordered) gives the same bits as one launch per step, for
    every sweep length and band lag (partial last sweeps included)."""
    if sweep is not None:
        monkeypatch.setenv("SPD_SWEEP", str(sweep))
        monkeypatch.setenv("SPD_LAG", str(lag))
    # normalised weights: many steps of un-normalised r = 3 weights overflow
    # fp16 to inf/NaN, and NaN != NaN
    k0 = rand_kernel("box", d, r, seed=[d, 31 + r])
    c = k0.coeffs / np.abs(k0.coeffs).sum()
    k = sp.make_kernel_3d("box", r, c) if d == 3 else sp.make_kernel("box", d, r, c)
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    dense = torch.rand(tuple(n + 2 * r for n in shape), dtype=torch.float64, device="cuda") - 0.5
    outs = []
    for persistent in (False, True):
        g = DeviceGrid(plan, shape, r)
        g.load_dense_f64(dense)
        g.run(steps, persistent=persistent)
        outs.append(g.bufs[g.cur].clone())
    assert torch.equal(outs[0], outs[1])


# --------------------------------------------------------------------------
# Many tiles per CTA: every ring (natural rows, B image, accumulators,
# publish) wraps around many times, on grids with ragged edges; per-step
# launches and the persistent wavefront launch, against the oracle.

@pytest.mark.parametrize(
    "d,r,shape,steps",
    [
        (2, 1, (1000, 4096), 3),     # B9 geometry, ragged last tile row
        (2, 1, (2048, 2000), 2),     # ragged right tiles
        (2, 3, (1000, 4096), 2),     # B49 geometry
        (2, 2, (600, 3072), 2),      # radius 2 embedded as radius 3 (L = 8 fast path)
        (2, 2, (600, 3066), 2),      # ... with a partial last 8-point chunk (width % 8 = 2)
        ("noembed", 2, (600, 3072), 2),  # radius 2 on the generic L = 6 path (SPD_NO_EMBED)
        (2, 4, (300, 4000), 1),      # generic L = 10
        (2, 7, (200, 4096), 1),      # generic L = 16
        (3, 1, (60, 72, 512), 2),    # B27 geometry, ragged z / y
        (1, 1, (1, 4 * 512 * 700), 2),
        (1, 2, (1, 419994), 2),      # 1D radius 2 embedded, partial last chunk
    ],
)
@pytest.mark.parametrize("persistent", [False, True])
@pytest.mark.timeout(180, method="thread")
def test_many_tiles_per_cta_match_oracle(monkeypatch, d, r, shape, steps, persistent):
    import os

    if d == "noembed":
        monkeypatch.setenv("SPD_NO_EMBED", "1")
        d = 2
    rng = np.random.default_rng([d, r, 11])
    c = rng.uniform(0.5, 1.5, (2 * r + 1,) * d)
    c /= c.sum()
    k = sp.make_kernel_3d("box", r, c) if d == 3 else sp.make_kernel("box", d, r, c)
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    dense = quant(rng.uniform(-1, 1, tuple(n + 2 * r for n in shape)))
    g = DeviceGrid(plan, shape, r)
    g.load_dense_f64(torch.from_numpy(dense).cuda())
    g.run(steps, persistent=persistent)
    got = g.to_dense_f64().cpu().numpy()
    want = cnaive.naive_apply(c, d, r, dense, r, steps, threads=os.cpu_count())
    assert max_rel_error(got, want) < TOL["fp16"]
    # fp32 accumulation + one fp16 rounding per step: far tighter than 1e-2
    assert np.abs(got - want).max() < 2e-3 * np.abs(want).max()


def test_cli_run_and_verify_on_device(tmp_path, capsys):
    """The reference CLI surface (cli.py:74-97, 185-203) over the device:
    make-grid -> run -> SPGR output vs the oracle; verify exits 0."""
    import json
    from pathlib import Path

    from paper_2506_22035_b200 import cli
    from paper_2506_22035_b200.io import load_grid, load_kernel

    gold = Path(__file__).resolve().parent / "golden" / "io"
    assert cli.main(["make-grid", "--size", "96x256", "--halo", "1", "--seed", "5",
                     "--out", str(tmp_path / "g.spgr")]) == cli.EXIT_OK
    capsys.readouterr()
    assert cli.main(["run", "--kernel", str(gold / "star2d_r1.json"), "--grid", str(tmp_path / "g.spgr"),
                     "--steps", "3", "--out", str(tmp_path / "o.spgr"), "--stats"]) == cli.EXIT_OK
    payload = json.loads(capsys.readouterr().out)
    assert payload["stats"]["steps"] == 3 and payload["stats"]["kernel_rows"] == 3
    k = load_kernel(gold / "star2d_r1.json")
    g = load_grid(tmp_path / "g.spgr")
    q = quant(g.data)
    want = cnaive.naive_apply(k.coeffs, 2, 1, q, 1, 3)
    got = load_grid(tmp_path / "o.spgr")
    assert max_rel_error(got.interior, want[1:-1, 1:-1]) < TOL["fp16"]
    assert abs(payload["output_checksum"] - float(got.interior.sum())) < 1e-6 * max(1.0, abs(payload["output_checksum"]))
    assert cli.main(["verify", "--kernel", str(gold / "box2d_r3.json"), "--sizes", "48,80", "--steps", "1"]) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert "all_pass:" in out


@pytest.mark.parametrize("d,shape", [(2, (130, 512)), (2, (96, 1024)), (3, (20, 24, 256)), (3, (40, 16, 128))])
def test_step_edges_plus_interior_is_a_full_step(d, shape):
    """The slab driver's boundary launch (first + last tile band in one
    launch, spd_step_edges) plus the interior range is one full step, bit for
    bit."""
    k = rand_kernel("box", d, 1, seed=[d, 3])
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    inf = plan.info()
    band = inf.tile_z if d == 3 else inf.tile_y
    dense = torch.rand(tuple(n + 2 for n in shape), dtype=torch.float64, device="cuda")
    a = DeviceGrid(plan, shape, 1)
    b = DeviceGrid(plan, shape, 1)
    a.load_dense_f64(dense)
    b.load_dense_f64(dense)
    a.run(1)
    b.step_edges()
    rows = shape[0]
    last = ((rows - 1) // band) * band
    if last > band:
        b.step_range(band, last)
    b.flip()
    assert torch.equal(a.bufs[a.cur], b.bufs[b.cur])


@pytest.mark.parametrize("d,r,shape,dtype,parity", [
    (2, 1, (1000, 4096), "bf16", "even"),
    (2, 1, (1000, 4096), "fp16", "odd"),
    (2, 3, (600, 2048), "bf16", "odd"),
    (3, 1, (40, 48, 256), "bf16", "even"),
])
def test_many_tiles_bf16_and_odd_parity(d, r, shape, dtype, parity):
    """The bf16 and ODD-parity kernel instantiations on grids with many tiles
    per CTA, against the oracle."""
    import os

    rng = np.random.default_rng([d, r, 13])
    c = rng.uniform(0.5, 1.5, (2 * r + 1,) * d)
    c /= c.sum()
    k = sp.make_kernel_3d("box", r, c) if d == 3 else sp.make_kernel("box", d, r, c)
    plan = get_plan(k, sp.Parity(parity), dtype)
    dense = quant(rng.uniform(-1, 1, tuple(n + 2 * r for n in shape)), dtype)
    g = DeviceGrid(plan, shape, r)
    g.load_dense_f64(torch.from_numpy(dense).cuda())
    g.run(2)
    got = g.to_dense_f64().cpu().numpy()
    want = cnaive.naive_apply(c, d, r, dense, r, 2, threads=os.cpu_count())
    assert max_rel_error(got, want) < TOL[dtype]


@pytest.mark.parametrize("shape", [(16, 16, 512), (40, 48, 256), (64, 64, 600)])
def test_cta_pair_3d_bit_identical(shape):
    """3D CTA-pair mode (SPD_PLAN_CTA_PAIR: one M = 256 tcgen05.mma.sp.cta_group::2
    per K-block, each CTA staging one x-half of B and holding one M-tile's
    A/E) gives the same bits as the default two-M-tile kernel."""
    from paper_2506_22035_b200.engine import Plan

    rng = np.random.default_rng(3)
    c = rng.uniform(0.5, 1.5, (3, 3, 3))
    c /= c.sum()
    k = sp.make_kernel_3d("box", 1, c)
    torch.manual_seed(0)
    dense = torch.rand(tuple(n + 2 for n in shape), dtype=torch.float64, device="cuda") - 0.5
    outs = []
    for cg2 in (0, 1):
        plan = Plan(k, sp.Parity.EVEN, "fp16", cta_pair=bool(cg2))
        assert plan.info().cg2 == int(cg2)
        g = DeviceGrid(plan, shape, 1)
        g.load_dense_f64(dense)
        g.run(3)
        outs.append(g.to_dense_f64())
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("d,r,dims", [(2, 1, (96, 1024)), (3, 1, (24, 24, 256))])
def test_concurrent_execute_callers(d, r, dims):
    """execute() from several host threads at once (each on its own stream,
    sharing one cached plan) gives the same bits as sequential calls."""
    import threading

    k = rand_kernel("box", d, r, seed=[d, 11])
    cls = sp.Grid3D if d == 3 else sp.Grid
    grids = []
    for i in range(4):
        data = quant(np.random.default_rng(i).uniform(-1, 1, tuple(n + 2 * r for n in dims))).astype(np.float16)
        grids.append(cls(data, r))
    want = [sp.execute(k, g, 5)[0].data.copy() for g in grids]
    got = [None] * len(grids)

    def worker(i):
        with torch.cuda.stream(torch.cuda.Stream()):
            for _ in range(3):
                got[i] = sp.execute(k, grids[i], 5)[0].data.copy()

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(grids))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for w, g in zip(want, got):
        np.testing.assert_array_equal(g, w)


@pytest.mark.parametrize("d,r,dims", [(2, 1, (64, 512)), (2, 3, (48, 256)), (3, 1, (16, 16, 256))])
def test_grid_cache_reuse_with_new_halo(d, r, dims):
    """execute() reuses cached device grids between calls: a second call with a
    different grid (different Dirichlet halo too) must give the same bits as a
    call on freshly allocated buffers, and both match the oracle."""
    from paper_2506_22035_b200.pipeline import release_device_grids

    c = np.random.default_rng([d, r, 5]).uniform(0.5, 1.5, (2 * r + 1,) * d)
    c /= c.sum()
    k = sp.make_kernel_3d("box", r, c) if d == 3 else sp.make_kernel("box", d, r, c)
    cls = sp.Grid3D if d == 3 else sp.Grid
    shape = tuple(n + 2 * r for n in dims)
    g1 = cls(quant(np.random.default_rng(1).uniform(-1, 1, shape)).astype(np.float16), r)
    g2 = cls(quant(np.random.default_rng(2).uniform(-1, 1, shape)).astype(np.float16), r)
    release_device_grids()
    sp.execute(k, g1, 3)
    reused = sp.execute(k, g2, 3)[0].data.copy()
    release_device_grids()
    fresh = sp.execute(k, g2, 3)[0].data.copy()
    np.testing.assert_array_equal(reused, fresh)
    want = cnaive.naive_apply(k.coeffs, d, r, g2.data.astype(np.float64), r, 3)
    assert max_rel_error(reused.astype(np.float64), want) < TOL["fp16"]


def test_device_stats_equal_host_counters():
    """The counters execute() returns are exec_stats()' plus the device block."""
    from paper_2506_22035_b200.pipeline import exec_stats

    k = rand_kernel("box", 2, 3, seed=4)
    g = sp.random_grid(64, 64, 3, seed=20)
    _, st = sp.execute(k, g, 2)
    host = exec_stats(k, g, 2).as_dict()
    dev = st.as_dict()
    assert dev.pop("device")["mma_instructions"] > 0
    host.pop("device")
    assert dev == host


@pytest.mark.gpu
@pytest.mark.parametrize("d,r,halves_per_tile", [(2, 1, 7), (2, 3, 7), (3, 1, 18), (1, 1, 7)])
def test_m64_half_lane_mmas_counted_and_exact(d, r, halves_per_tile):
    """The step schedule issues M = 64 MMAs on one half of the accumulator
    lanes where a K-block feeds only that half (aot.cpp assign_mma_halves,
    engine.cu ct_halves_mask); the device block counts them (per M-tile) and
    the result still matches the oracle."""
    kern = rand_kernel("box", d, r, seed=50 + d + r)
    shape = {1: (1, 3000), 2: (70, 600), 3: (12, 10, 200)}[d]  # 1D problems use A = 1
    got, want, _, stats = run_case(kern, shape, 2)
    dev = stats.device
    assert dev["m64_instructions"] == 2 * dev["tiles_per_step"] * halves_per_tile
    inner = tuple(slice(r, -r) for _ in range(max(d, 2)))
    assert max_rel_error(got.interior, want[inner]) < TOL["fp16"]
