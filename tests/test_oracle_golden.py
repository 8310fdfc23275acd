"""Pin the CPU oracle (oracle/) against vectors produced by the reference itself
(tests/golden/make_golden.py).  Bit-exact for the transform and for naive_apply."""
import numpy as np
import pytest

from oracle import cnaive, naive
from oracle import transform as otr


def _row_keys(g):
    return sorted(k[: -len("_row")] for k in g.files if k.endswith("_row"))


def test_transform_oracle_matches_reference(golden):
    g = golden("transform_golden.npz")
    keys = _row_keys(g)
    assert len(keys) == 80
    for key in keys:
        r = int(key.split("_")[0][1:])
        parity = 0 if key.endswith("even") else 1
        row = g[key + "_row"]
        band = otr.kernel_matrix(row, r)
        np.testing.assert_array_equal(band, g[key + "_band"])
        sw = otr.swap(band, parity)
        np.testing.assert_array_equal(sw, g[key + "_swapped"])
        vals, meta = otr.encode(sw)
        np.testing.assert_array_equal(vals, g[key + "_values"])
        np.testing.assert_array_equal(meta, g[key + "_meta"])
        assert otr.metadata_bytes(meta) == g[key + "_metabytes"].tobytes()
        np.testing.assert_array_equal(otr.decode(vals, meta), g[key + "_decoded"])
        got = np.array(otr.check_2to4(band), dtype=np.int64).reshape(-1, 2)
        np.testing.assert_array_equal(got, g[key + "_check_unswapped"])
        assert otr.check_2to4(sw) == []


def test_permutation_oracle_matches_reference(golden):
    g = golden("transform_golden.npz")
    for r in range(1, 9):
        L = 2 * r + 2
        for p, name in ((0, "even"), (1, "odd")):
            np.testing.assert_array_equal(otr.permutation(L, p), g[f"perm_L{L}_{name}"])


def test_encode_segment_kats(golden):
    g = golden("transform_golden.npz")
    for seg, want in zip(g["segments"], g["segments_encoded"]):
        assert np.array_equal(np.array(otr.encode_segment(seg), dtype=np.float64), want)


def _small_cases(g):
    for c in range(int(g["n_cases"])):
        d, r, steps, star = (int(v) for v in g[f"c{c}_meta"])
        yield c, d, r, steps, g[f"c{c}_coeffs"], g[f"c{c}_in"], g[f"c{c}_out"]


@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_naive_oracle_small_cases_bit_exact(golden, impl):
    g = golden("naive_golden.npz")
    n = 0
    for c, d, r, steps, coeffs, grid, want in _small_cases(g):
        if impl == "numpy":
            got = naive.naive_apply(coeffs, d, r, grid, r, steps)
        else:
            got = cnaive.naive_apply(coeffs, d, r, grid, r, steps, threads=3)
        np.testing.assert_array_equal(got, want, err_msg=f"case {c}")
        n += 1
    assert n == 12


@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_naive_oracle_s5_config(golden, impl):
    """The oracle config: Star-2D5P (Heat-2D) 512^2, 4 steps."""
    g = golden("naive_golden.npz")
    rng = np.random.default_rng([1, 512, 512])
    grid = rng.uniform(-1.0, 1.0, size=(514, 514))
    coeffs = g["s5_coeffs"]
    if impl == "numpy":
        got = naive.naive_apply(coeffs, 2, 1, grid, 1, 4)
    else:
        got = cnaive.naive_apply(coeffs, 2, 1, grid, 1, 4)
    idx = g["s5_idx"]
    np.testing.assert_array_equal(got[idx[:, 0], idx[:, 1]], g["s5_samples"])
    np.testing.assert_array_equal(got[240:272, 240:272], g["s5_center"])
    assert got.sum() == g["s5_sum"]


@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_naive3d_oracle_pins(golden, impl):
    g = golden("naive3d_golden.npz")
    fn = naive.naive_apply if impl == "numpy" else cnaive.naive_apply
    got = fn(g["a_coeffs"], 3, 1, g["a_in"], 1, 1)
    np.testing.assert_array_equal(got, g["a_out"])  # rho_z = 0: exact reduction
    got = fn(g["b_coeffs"], 3, 1, g["b_in"], 1, 1)
    np.testing.assert_allclose(got, g["b_out"], rtol=0, atol=1e-13)  # separable: reassociated


def test_reference_execute_agrees_with_oracle(golden):
    """The reference's own SpTC-emulation path (execute) on the same inputs
    lands within its 1e-10 bar of the oracle."""
    g = golden("naive_golden.npz")
    seen = 0
    for c, d, r, steps, coeffs, grid, want in _small_cases(g):
        key = f"c{c}_execute"
        if key in g.files:
            assert naive.max_rel_error(g[key][r:-r, r:-r], want[r:-r, r:-r]) < 1e-10
            seen += 1
    assert seen >= 6
