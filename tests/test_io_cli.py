"""File formats and the CLI against files written by the reference itself
(tests/golden/io, made by tests/golden/make_golden.py): byte-identical SPGR
and SPCK output, JSON mirrors, and the reference's exit-code contract
(cli.py:281-291).  Device subcommands are exercised in the gpu tier."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2506_22035_b200 as sp
from paper_2506_22035_b200 import cli
from paper_2506_22035_b200.io import (
    load_compressed_set,
    load_grid,
    load_kernel,
    save_compressed_json,
    save_compressed_set,
    save_grid,
    save_kernel,
)

GOLD = Path(__file__).resolve().parent / "golden" / "io"
KERNELS = ["box2d_r3", "star2d_r1"]


def test_spgr_roundtrip_is_byte_identical(tmp_path):
    g = load_grid(GOLD / "grid.spgr")
    assert (g.A, g.B, g.halo) == (5, 7, 2)
    save_grid(g, tmp_path / "g.spgr")
    assert (tmp_path / "g.spgr").read_bytes() == (GOLD / "grid.spgr").read_bytes()


def test_random_grid_matches_reference_file(tmp_path):
    # the reference random_grid (core.py:144-148) wrote grid.spgr
    save_grid(sp.random_grid(5, 7, 2, seed=3), tmp_path / "g.spgr")
    assert (tmp_path / "g.spgr").read_bytes() == (GOLD / "grid.spgr").read_bytes()


def test_spg3_roundtrip(tmp_path):
    g = sp.random_grid_3d(3, 4, 8, 1, seed=1)
    save_grid(g, tmp_path / "g.spg3")
    h = load_grid(tmp_path / "g.spg3")
    assert isinstance(h, sp.Grid3D) and np.array_equal(h.data, g.data)


@pytest.mark.parametrize("name", KERNELS)
@pytest.mark.parametrize("parity", ["even", "odd"])
def test_spck_bytes_match_reference(tmp_path, name, parity):
    from paper_2506_22035_b200.pipeline import transform_stencil

    k = load_kernel(GOLD / f"{name}.json")
    ts = transform_stencil(k, sp.Parity(parity))
    cks = [ck for _rho, ck in ts.rows]
    save_compressed_set(cks, tmp_path / "k.spck")
    assert (tmp_path / "k.spck").read_bytes() == (GOLD / f"{name}_{parity}.spck").read_bytes()
    save_compressed_json(cks, tmp_path / "k.json")
    assert json.loads((tmp_path / "k.json").read_text()) == json.loads((GOLD / f"{name}_{parity}.spck.json").read_text())
    back = load_compressed_set(GOLD / f"{name}_{parity}.spck")
    assert len(back) == len(cks)
    for a, b in zip(back, cks):
        assert np.array_equal(a.values, b.values) and np.array_equal(a.metadata, b.metadata)
        assert a.r == b.r and a.parity == b.parity


def test_kernel_json_roundtrip(tmp_path):
    for name in KERNELS:
        k = load_kernel(GOLD / f"{name}.json")
        save_kernel(k, tmp_path / "k.json")
        assert json.loads((tmp_path / "k.json").read_text()) == json.loads((GOLD / f"{name}.json").read_text())
    k3 = sp.make_kernel_3d("box", 1, np.arange(27.0))
    save_kernel(k3, tmp_path / "k3.json")
    assert np.array_equal(load_kernel(tmp_path / "k3.json").coeffs, k3.coeffs)


def test_bad_files_raise_value_error(tmp_path):
    (tmp_path / "bad.spgr").write_bytes(b"XXXX" + bytes(12))
    with pytest.raises(ValueError, match="bad magic"):
        load_grid(tmp_path / "bad.spgr")
    (tmp_path / "short.spgr").write_bytes(b"SPG")
    with pytest.raises(ValueError, match="truncated"):
        load_grid(tmp_path / "short.spgr")
    raw = (GOLD / "grid.spgr").read_bytes()
    (tmp_path / "cut.spgr").write_bytes(raw[:-8])
    with pytest.raises(ValueError, match="expected"):
        load_grid(tmp_path / "cut.spgr")
    (tmp_path / "empty.spck").write_bytes(b"")
    with pytest.raises(ValueError, match="no compressed-kernel records"):
        load_compressed_set(tmp_path / "empty.spck")


def test_cli_transform_and_make_grid(tmp_path, capsys):
    rc = cli.main(["transform", "--kernel", str(GOLD / "box2d_r3.json"), "--parity", "odd",
                   "--out", str(tmp_path / "o.spck"), "--json", str(tmp_path / "o.json")])
    assert rc == cli.EXIT_OK
    assert (tmp_path / "o.spck").read_bytes() == (GOLD / "box2d_r3_odd.spck").read_bytes()
    summary = json.loads(capsys.readouterr().out)
    assert summary["kernel_rows"] == 7 and summary["L"] == 8
    assert summary["permutation"] == [0, 9, 2, 11, 4, 13, 6, 15, 8, 1, 10, 3, 12, 5, 14, 7]
    rc = cli.main(["make-grid", "--size", "5x7", "--halo", "2", "--seed", "3", "--out", str(tmp_path / "g.spgr")])
    assert rc == cli.EXIT_OK
    assert (tmp_path / "g.spgr").read_bytes() == (GOLD / "grid.spgr").read_bytes()


def test_cli_exit_codes(tmp_path):
    assert cli.main(["frobnicate"]) == cli.EXIT_CONFIG_ERROR
    assert cli.main(["transform", "--kernel", str(tmp_path / "missing.json"), "--out", "x"]) == cli.EXIT_CONFIG_ERROR
    (tmp_path / "bad.json").write_text(json.dumps({"shape": "box", "d": 4, "r": 1, "coeffs": [0] * 81}))
    assert cli.main(["transform", "--kernel", str(tmp_path / "bad.json"), "--out", "x"]) == cli.EXIT_CONFIG_ERROR
    assert cli.main(["analyze", "--r", "3"]) == cli.EXIT_CONFIG_ERROR
