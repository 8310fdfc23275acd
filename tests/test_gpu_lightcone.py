"""Full-size parity through the light cone (SURVEY.md §8(c) "Large grids").

After T steps of a radius-r stencil, a point depends only on inputs within
r*T of it.  So for the bench configurations at their full sizes and step
counts (B9 / B49 at 10240^2, B27 at 512^3, W at 16384^2, B25 at 10240 x 10242,
T = 100):

* the device result on the full grid, restricted to an inner block, equals
  the device result on a crop holding that block plus an r*T margin
  (the crop's outer ring acting as its Dirichlet halo) BIT FOR BIT — the
  crop origin is tile-aligned, so every point sees the same arithmetic;
* the crop is small enough for the C oracle (fp64 `naive_apply`, reference
  core.py:151-182) to run the same T steps on the fp16-quantised inputs, so
  the full-size result is pinned against the reference algorithm.  The
  tolerance is the measured fp16 bound over 100 steps (max-rel, reference
  pipeline.py:265-267): 2e-2, the same bound the 100-step Heat-3D test uses.

Blocks are taken at the grid centre and at a corner (the global Dirichlet
halo inside the light cone).
"""
import zlib

import pytest
import torch

import bench
import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.engine import DeviceGrid
from paper_2506_22035_b200.pipeline import get_plan, max_rel_error
from oracle import cnaive

pytestmark = pytest.mark.gpu

TOL_T100 = 2e-2


@pytest.mark.parametrize("name,inner", [("B9", 64), ("B49", 32), ("B27", 16), ("W", 64), ("B25", 32)])
@pytest.mark.parametrize("where", ["centre", "corner"])
@pytest.mark.timeout(600, method="thread")
def test_light_cone_full_size(name, inner, where):
    _, shape, d, r, kind, T = bench.CONFIGS[name]
    kern = bench.make_kernel(kind, d, r)
    plan = get_plan(kern, sp.Parity.EVEN, "fp16")
    h, margin = r, r * T
    gen = torch.Generator(device="cuda").manual_seed(zlib.crc32(f"{name}/{where}".encode()))
    dense = torch.rand(tuple(n + 2 * h for n in shape), dtype=torch.float64, device="cuda",
                       generator=gen) * 2 - 1
    dense = dense.to(torch.float16).to(torch.float64)          # the inputs the device sees

    full = DeviceGrid(plan, shape, h)
    full.load_dense_f64(dense)
    full.run(T)
    out_full = full.to_dense_f64()
    del full

    # crop origin (dense index of its first halo point) tile-aligned with the
    # full grid (the tile's row and x-chunk positions fix each point's
    # accumulation order); the block sits `margin` points inside
    inf = plan.info()
    tile_x = inf.n_tile * inf.L
    tiles = ([inf.tile_z] if d == 3 else []) + [inf.tile_y]
    if where == "centre":
        cs = [(n // 2) // t * t for n, t in zip(shape[:-1], tiles)] + [(shape[-1] // 2) // tile_x * tile_x]
    else:
        cs = [0] * d                             # keeps the global halo as its own
    lo = [c + margin for c in cs] if where == "centre" else [0] * d
    size = [inner] * d
    ext = [a + s + margin - c for c, a, s in zip(cs, lo, size)]     # crop interior extents
    L = 2 * r + 2
    ext[-1] = -(-ext[-1] // L) * L                                  # width: a multiple of L
    sl = tuple(slice(c, min(c + e + 2 * h, n)) for c, e, n in zip(cs, ext, dense.shape))
    crop_in = dense[sl].contiguous()
    crop_shape = tuple(n - 2 * h for n in crop_in.shape)
    offs = cs

    cg = DeviceGrid(plan, crop_shape, h)
    cg.load_dense_f64(crop_in)
    cg.run(T)
    out_crop = cg.to_dense_f64()
    del cg

    # the block inside the cone, in dense coordinates of each array
    blk_full = tuple(slice(a + h, a + h + s) for a, s in zip(lo, size))
    blk_crop = tuple(slice(a + h - o, a + h - o + s) for a, s, o in zip(lo, size, offs))
    got_full = out_full[blk_full]
    got_crop = out_crop[blk_crop]
    assert torch.equal(got_full, got_crop), float((got_full - got_crop).abs().max())

    # oracle on the crop (2D: all of it; 3D: the C oracle at 3D crop sizes is
    # seconds too since the crop is (inner + 2rT)^3 = 216^3)
    want = cnaive.naive_apply(kern.coeffs, d, r, crop_in.cpu().numpy(), h, T)
    err = max_rel_error(got_crop.cpu().numpy(), want[blk_crop])
    print(f"light-cone {name} {where}: max-rel vs fp64 oracle after T={T}: {err:.3e}")
    assert err < TOL_T100, err
    assert not torch.equal(got_crop, crop_in[blk_crop])            # the block did evolve


@pytest.mark.timeout(600, method="thread")
def test_large_grid_64bit_offsets():
    """A 36864^2 fp16 grid (2.7 GB per buffer: element offsets past 2^31
    bytes): a block at the far corner after 3 steps equals the same block of a
    small tile-aligned crop run (light cone), bit for bit."""
    _, _, d, r, kind, _ = bench.CONFIGS["B9"]
    kern = bench.make_kernel(kind, d, r)
    plan = get_plan(kern, sp.Parity.EVEN, "fp16")
    n, T, h = 36864, 3, r
    full = DeviceGrid(plan, (n, n), h)
    gen = torch.Generator(device="cuda").manual_seed(31)
    dense = (torch.rand((n + 2 * h, n + 2 * h), dtype=torch.float32, device="cuda", generator=gen) * 2 - 1).half()
    full.load_dense_f64(dense.double())
    full.run(T)
    out = full.to_dense_f64()
    inf = plan.info()
    ty, tx = inf.tile_y, inf.n_tile * inf.L
    c0y, c0x = (n - 256) // ty * ty, (n - 1024) // tx * tx       # crop origin (dense index), tile-aligned
    crop_in = dense[c0y:, c0x:].double().contiguous()
    cg = DeviceGrid(plan, tuple(s - 2 * h for s in crop_in.shape), h)
    cg.load_dense_f64(crop_in)
    cg.run(T)
    got = cg.to_dense_f64()
    m = r * T  # rows / columns next to the crop's own halo see its frozen edge
    assert torch.equal(out[c0y + h + m:, c0x + h + m:], got[h + m:, h + m:])
    assert not torch.equal(out[c0y + h + m:-h, c0x + h + m:-h], dense[c0y + h + m:-h, c0x + h + m:-h].double())


@pytest.mark.timeout(600, method="thread")
def test_large_3d_grid_64bit_offsets():
    """1024^3 fp16 (2.2 GB per buffer): the far-corner block after 2 steps
    equals a tile-aligned crop run, bit for bit."""
    _, _, d, r, kind, _ = bench.CONFIGS["B27"]
    kern = bench.make_kernel(kind, d, r)
    plan = get_plan(kern, sp.Parity.EVEN, "fp16")
    n, T, h = 1024, 2, r
    full = DeviceGrid(plan, (n, n, n), h)
    gen = torch.Generator(device="cuda").manual_seed(33)
    dense = (torch.rand((n + 2 * h,) * 3, dtype=torch.float32, device="cuda", generator=gen) * 2 - 1).half()
    full.load_dense_f64(dense.double())
    full.run(T)
    out = full.to_dense_f64()
    inf = plan.info()
    c = [(n - 40) // inf.tile_z * inf.tile_z, (n - 40) // inf.tile_y * inf.tile_y,
         (n - 256) // (inf.n_tile * inf.L) * (inf.n_tile * inf.L)]
    crop_in = dense[c[0]:, c[1]:, c[2]:].double().contiguous()
    cg = DeviceGrid(plan, tuple(s - 2 * h for s in crop_in.shape), h)
    cg.load_dense_f64(crop_in)
    cg.run(T)
    got = cg.to_dense_f64()
    m = h + r * T
    assert torch.equal(out[c[0] + m:, c[1] + m:, c[2] + m:], got[m:, m:, m:])
