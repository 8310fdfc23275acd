"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `sparsestencil` from /root/reference/pkg/src (read-only) and writes
small fixtures next to this script.  The GPU box never needs the reference:
the tests read only these committed files.

Fixtures
  transform_golden.npz  transform_stencil rows (values, metadata bytes, swapped
                        matrix, decoded matrix) and the row permutations for
                        r in 1..8, both parities, for tap-identifying rows
                        [1..2r+1], random rows, star off-centre rows (one tap),
                        rows with zeros and negative zeros; encode_segment KATs.
  naive_golden.npz      reference naive_apply outputs on seeded grids: the
                        oracle config (Star-2D5P / Heat-2D, 512^2, 4 steps —
                        stored as statistics + sampled points) plus full
                        outputs for small 1D/2D box/star cases, r in 1..3.
  naive3d_golden.npz    3D pins (no 3D in the reference): (a) a 3D kernel whose
                        only nonzero plane is rho_z = 0 equals the reference 2D
                        naive_apply per z-plane; (b) a separable kernel
                        a(rho_z) * b(rho_y, delta) equals sum_rz a * (2D
                        reference on plane z + rz), recorded for one step.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _ref():
    if not REF.exists():
        raise SystemExit("reference tree not found; golden vectors can only be regenerated in the build container")
    sys.path.insert(0, str(REF))
    import sparsestencil as ss  # noqa: E402

    return ss


def transform_cases(ss):
    rng = np.random.default_rng(20250617)
    out = {}
    n = 0
    for r in range(1, 9):
        span = 2 * r + 1
        rows = {
            "taps": np.arange(1, span + 1, dtype=np.float64),
            "rand": rng.uniform(-1, 1, span),
            "star": np.where(np.arange(span) == r, 0.75, 0.0),
            "zeros": np.where(rng.uniform(size=span) < 0.4, 0.0, rng.uniform(-2, 2, span)),
            "negzero": np.where(np.arange(span) % 2 == 0, -0.0, rng.uniform(-1, 1, span)),
        }
        for name, row in rows.items():
            for parity in ("even", "odd"):
                band = ss.build_kernel_matrix(row, r)
                sw = ss.strided_swap(band, parity)
                ck = ss.encode(sw)
                key = f"r{r}_{name}_{parity}"
                out[key + "_row"] = row
                out[key + "_band"] = band.values
                out[key + "_swapped"] = sw.values
                out[key + "_values"] = ck.values
                out[key + "_meta"] = ck.metadata
                out[key + "_metabytes"] = np.frombuffer(ss.transform.metadata_to_bytes(ck.metadata), dtype=np.uint8)
                out[key + "_decoded"] = ss.decode(ck).values
                out[key + "_check_unswapped"] = np.array(ss.check_2to4(band).violations, dtype=np.int64).reshape(-1, 2)
                n += 1
        L = 2 * r + 2
        for parity in ("even", "odd"):
            out[f"perm_L{L}_{parity}"] = ss.input_row_permutation(L, parity).mapping
    segs = np.array(
        [[1.5, 0, 2.5, 0], [0, 3, 0, 0], [0, 0, 0, 0], [0, 0, 0, 4], [5, 0, 0, 0], [0, 0, 6, 0], [7, 8, 0, 0],
         [0, 0, 9, 1], [0, 2, 0, 3], [-0.0, 0, 0, 1]],
        dtype=np.float64,
    )
    enc = np.array([ss.transform.encode_segment(s) for s in segs], dtype=np.float64)
    out["segments"] = segs
    out["segments_encoded"] = enc
    np.savez_compressed(OUT / "transform_golden.npz", **out)
    print(f"transform_golden.npz: {n} row cases")


def heat2d(alpha=0.125):
    c = np.zeros((3, 3))
    c[1, 1] = 1 - 4 * alpha
    c[0, 1] = c[2, 1] = c[1, 0] = c[1, 2] = alpha
    return c


def naive_cases(ss):
    out = {}
    # Oracle config: Star-2D5P (Heat-2D) 512^2, 4 steps, random_grid seed [1, 512, 512]
    k = ss.make_kernel("star", 2, 1, heat2d())
    g = ss.random_grid(512, 512, 1, seed=[1, 512, 512])
    res = ss.naive_apply(k, g, 4).data
    rng = np.random.default_rng(7)
    idx = rng.integers(0, 514, size=(4096, 2))
    out["s5_coeffs"] = k.coeffs
    out["s5_seed"] = np.array([1, 512, 512])
    out["s5_sum"] = np.array(res.sum())
    out["s5_sumsq"] = np.array((res * res).sum())
    out["s5_idx"] = idx
    out["s5_samples"] = res[idx[:, 0], idx[:, 1]]
    out["s5_center"] = res[240:272, 240:272]
    # small full cases
    case = 0
    for shape in ("box", "star"):
        for d in (1, 2):
            for r in (1, 2, 3):
                kr = np.random.default_rng([case, d, r])
                span = 2 * r + 1
                if d == 1 or shape == "box":
                    coeffs = kr.uniform(-1, 1, span**d)
                else:
                    coeffs = np.zeros((span, span))
                    coeffs[r, :] = kr.uniform(-1, 1, span)
                    coeffs[:, r] = kr.uniform(-1, 1, span)
                kern = ss.make_kernel(shape, d, r, coeffs)
                a, b = (1, 96) if d == 1 else (24, 40)
                grid = ss.random_grid(a, b, r, seed=[case, a, b])
                steps = 1 + case % 3
                res = ss.naive_apply(kern, grid, steps).data
                key = f"c{case}"
                out[key + "_meta"] = np.array([d, r, steps, 0 if shape == "box" else 1])
                out[key + "_coeffs"] = kern.coeffs.ravel()
                out[key + "_in"] = grid.data
                out[key + "_out"] = res
                # the reference's own SpTC-emulation path on the same input
                if b % (2 * r + 2) == 0:
                    ex, _ = ss.execute(kern, grid, steps)
                    out[key + "_execute"] = ex.data
                case += 1
    out["n_cases"] = np.array(case)
    np.savez_compressed(OUT / "naive_golden.npz", **out)
    print(f"naive_golden.npz: S5 + {case} small cases")


def naive3d_cases(ss):
    out = {}
    rng = np.random.default_rng(31337)
    Z, A, B, h, r = 6, 10, 16, 1, 1
    g3 = rng.uniform(-1, 1, (Z + 2 * h, A + 2 * h, B + 2 * h))
    # (a) only the rho_z = 0 plane is nonzero
    plane = rng.uniform(-1, 1, (3, 3))
    c3 = np.zeros((3, 3, 3))
    c3[1] = plane
    k2 = ss.make_kernel("box", 2, 1, plane)
    want = g3.copy()
    for z in range(h, h + Z):
        want[z] = ss.naive_apply(k2, ss.Grid(g3[z].copy(), h), 1).data
    out["a_coeffs"] = c3
    out["a_in"] = g3
    out["a_out"] = want
    # (b) separable: c[rz, ry, dx] = a[rz] * b[ry, dx]
    av = rng.uniform(-1, 1, 3)
    bv = rng.uniform(-1, 1, (3, 3))
    cs = av[:, None, None] * bv[None, :, :]
    kb = ss.make_kernel("box", 2, 1, bv)
    planes2d = np.stack([ss.naive_apply(kb, ss.Grid(g3[z].copy(), h), 1).data for z in range(Z + 2 * h)])
    wantb = g3.copy()
    for z in range(h, h + Z):
        acc = np.zeros((A, B))
        for i, rz in enumerate((-1, 0, 1)):
            acc += av[i] * planes2d[z + rz, h : h + A, h : h + B]
        wantb[z, h : h + A, h : h + B] = acc
    out["b_coeffs"] = cs
    out["b_in"] = g3
    out["b_out"] = wantb
    np.savez_compressed(OUT / "naive3d_golden.npz", **out)
    print("naive3d_golden.npz: rho_z=0 and separable pins")


def io_cases(ss):
    """Reference-written files for the byte-compatibility tests of io.py."""
    from sparsestencil import transform as st

    d = OUT / "io"
    d.mkdir(exist_ok=True)
    ss.save_grid(ss.random_grid(5, 7, 2, seed=3), d / "grid.spgr")
    rng = np.random.default_rng(7)
    k = ss.make_kernel("box", 2, 3, rng.uniform(-1, 1, (7, 7)))
    ss.save_kernel(k, d / "box2d_r3.json")
    star = np.zeros((3, 3))
    star[1, :] = [0.25, -0.5, 0.25]
    star[:, 1] = [0.125, -0.5, 0.125]
    ss.save_kernel(ss.make_kernel("star", 2, 1, star), d / "star2d_r1.json")
    for name in ("box2d_r3", "star2d_r1"):
        kern = ss.load_kernel(d / f"{name}.json")
        for par in ("even", "odd"):
            ts = ss.transform_stencil(kern, ss.Parity(par))
            cks = [ck for _rho, ck in ts.rows]
            st.save_compressed_set(cks, d / f"{name}_{par}.spck")
            st.save_compressed_json(cks, d / f"{name}_{par}.spck.json")
    print("io/: SPGR grid, kernel JSON, SPCK records + JSON mirrors")


STATS_CASES = [
    # (name, shape, d, r, A, B, steps, ExecConfig kwargs)
    ("box2d_r1_64", "box", 2, 1, 64, 64, 1, {}),
    ("box2d_r3_64_t2", "box", 2, 3, 64, 64, 2, {}),
    ("star2d_r1_32_t2", "star", 2, 1, 32, 32, 2, {}),
    ("box2d_r2_48_odd_unpacked", "box", 2, 2, 48, 48, 1, {"parity": "odd", "packing": False}),
    ("box2d_r1_64_blocks32", "box", 2, 1, 64, 64, 1, {"a_block": 32, "b_block": 32}),
    ("box2d_r1_30_noauto", "box", 2, 1, 30, 64, 1, {}),
    ("box1d_r2_48_t3", "box", 1, 2, 1, 48, 3, {}),
    ("box2d_r7_32", "box", 2, 7, 32, 32, 1, {}),
]


def stats_cases(ss):
    """ExecStats.as_dict() of the reference execute on small grids (the
    counter KATs: reference pipeline.py:200-259, tests/test_pipeline.py:140-192)."""
    import json

    out = {}
    for name, shape, d, r, A, B, steps, kw in STATS_CASES:
        span = 2 * r + 1
        rng = np.random.default_rng([7, d, r, A, B])
        coeffs = rng.uniform(0.5, 1.5, (span,) * d)
        if shape == "star":
            idx = np.indices((span,) * d)
            on_axis = np.zeros((span,) * d, dtype=bool)
            for ax in range(d):
                on_axis |= np.all([idx[o] == r for o in range(d) if o != ax], axis=0) if d > 1 else True
            coeffs = np.where(on_axis, coeffs, 0.0)
        k = ss.make_kernel(shape, d, r, coeffs)
        g = ss.random_grid(A, B, r, seed=[3, A, B])
        cfg = ss.ExecConfig(**{k2: (ss.Parity(v) if k2 == "parity" else v) for k2, v in kw.items()})
        _, st = ss.execute(k, g, steps, cfg)
        out[name] = {"shape": shape, "d": d, "r": r, "A": A, "B": B, "steps": steps, "cfg": kw,
                     "coeffs": np.asarray(coeffs).tolist(), "stats": st.as_dict()}
    (OUT / "stats_golden.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    print(f"stats_golden.json: {len(out)} cases")


if __name__ == "__main__":
    ss = _ref()
    only = sys.argv[1:]
    for fn in (transform_cases, naive_cases, naive3d_cases, io_cases, stats_cases):
        if not only or fn.__name__ in only:
            fn(ss)
