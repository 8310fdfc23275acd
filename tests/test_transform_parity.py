"""The product's AOT transform (C++ in libspider.so, via the drop-in Python
API) against the reference's own outputs: exact index / permutation / value /
metadata equality (BASELINE north star)."""
import numpy as np
import pytest

import paper_2506_22035_b200 as sp
from oracle import transform as otr


def _row_keys(g):
    return sorted(k[: -len("_row")] for k in g.files if k.endswith("_row"))


def test_transform_rows_exact(golden):
    g = golden("transform_golden.npz")
    for key in _row_keys(g):
        r = int(key.split("_")[0][1:])
        parity = sp.Parity.EVEN if key.endswith("even") else sp.Parity.ODD
        row = g[key + "_row"]
        band = sp.build_kernel_matrix(row, r)
        assert band.values.tobytes() == g[key + "_band"].tobytes()
        sw = sp.strided_swap(band, parity)
        assert sw.values.tobytes() == g[key + "_swapped"].tobytes()  # -0.0 preserved
        ck = sp.encode(sw)
        assert ck.values.tobytes() == g[key + "_values"].tobytes()
        np.testing.assert_array_equal(ck.metadata, g[key + "_meta"])
        assert sp.metadata_to_bytes(ck.metadata) == g[key + "_metabytes"].tobytes()
        assert sp.decode(ck).values.tobytes() == g[key + "_decoded"].tobytes()
        rep = sp.check_2to4(band)
        want = [tuple(v) for v in g[key + "_check_unswapped"].tolist()]
        assert rep.violations == want and rep.valid == (not want)
        assert sp.check_2to4(sw).valid
        # one-call builder used by the device plan
        ck2 = sp.transform.transform_row(row, r, parity)
        assert ck2.values.tobytes() == ck.values.tobytes()
        np.testing.assert_array_equal(ck2.metadata, ck.metadata)


def test_permutations_exact(golden):
    g = golden("transform_golden.npz")
    for r in range(1, 9):
        L = 2 * r + 2
        for parity in ("even", "odd"):
            perm = sp.input_row_permutation(L, parity)
            np.testing.assert_array_equal(perm.mapping, g[f"perm_L{L}_{parity}"])
            assert not perm.mapping.flags.writeable
            # involution
            np.testing.assert_array_equal(perm.mapping[perm.mapping], np.arange(2 * L))


def test_encode_segment_kats(golden):
    g = golden("transform_golden.npz")
    for seg, want in zip(g["segments"], g["segments_encoded"]):
        assert np.array_equal(np.array(sp.encode_segment(seg), dtype=np.float64), want)
    with pytest.raises(ValueError, match="2:4"):
        sp.encode_segment([1.0, 2.0, 3.0, 0.0])


def test_random_rows_match_oracle():
    rng = np.random.default_rng(5)
    for trial in range(200):
        r = int(rng.integers(1, 9))
        row = rng.uniform(-1, 1, 2 * r + 1)
        row[rng.uniform(size=row.size) < 0.3] = 0.0
        for parity in (0, 1):
            v, m = otr.transform_row(row, r, parity)
            ck = sp.transform.transform_row(row, r, sp.Parity.EVEN if parity == 0 else sp.Parity.ODD)
            assert ck.values.tobytes() == v.tobytes()
            np.testing.assert_array_equal(ck.metadata, m)


def test_equivalence_identity():
    """swapped-K @ permuted-X == K @ X (reference tests/test_transform.py:283-297)."""
    rng = np.random.default_rng(9)
    for r in (1, 2, 3, 7):
        row = rng.uniform(-1, 1, 2 * r + 1)
        band = sp.build_kernel_matrix(row, r)
        for parity in ("even", "odd"):
            sw = sp.strided_swap(band, parity)
            perm = sp.input_row_permutation(band.L, parity)
            X = rng.uniform(-1, 1, (2 * band.L, 7))
            np.testing.assert_allclose(sw.values @ perm.apply(X), band.values @ X, rtol=0, atol=1e-12)


def test_error_messages():
    band = sp.build_kernel_matrix([1.0, 2.0, 3.0], 1)
    sw = sp.strided_swap(band)
    with pytest.raises(ValueError, match="already swapped"):
        sp.strided_swap(sw)
    with pytest.raises(ValueError, match="swapped"):
        sp.encode(band)
    with pytest.raises(ValueError, match="radius"):
        sp.band_rows(0)
    with pytest.raises(ValueError, match="even"):
        sp.input_row_permutation(5)
    with pytest.raises(ValueError, match="2r\\+1"):
        sp.build_kernel_matrix([1.0, 2.0], 1)
    bad = sp.CompressedKernel(values=np.zeros((4, 4)), metadata=np.array([[[1, 0], [0, 1]]] * 4, dtype=np.uint8),
                              r=1, parity=sp.Parity.EVEN)
    with pytest.raises(ValueError, match="ascending"):
        sp.decode(bad)
