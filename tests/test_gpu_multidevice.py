"""execute(..., DeviceConfig(devices=...)): one process, the grid cut into
slabs over several devices with the peer-memory halo exchange.  The box has
one GPU, so the slabs share cuda:0 (listed several times); the exchange runs
the same code as between NVLink peers (plain device pointers, copy engine,
stream memory operations).  Results must equal the one-device execute bit
for bit."""
import numpy as np
import pytest

import paper_2506_22035_b200 as sp
from paper_2506_22035_b200.pipeline import DeviceConfig

gpu = pytest.mark.gpu


def _kernel(d, r, seed=3):
    rng = np.random.default_rng([d, r, seed])
    c = rng.uniform(0.5, 1.5, (2 * r + 1,) * d)
    c /= c.sum()
    return sp.make_kernel_3d("box", r, c) if d == 3 else sp.make_kernel("box", d, r, c)


def _grid(d, r, shape, dtype):
    rng = np.random.default_rng([len(shape), *shape])
    data = rng.uniform(-1, 1, tuple(s + 2 * r for s in shape)).astype(dtype)
    return sp.Grid3D(data, r) if d == 3 else sp.Grid(data, r)


@gpu
@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("d,r,shape,n,steps,dtype", [
    (2, 1, (256, 1024), 2, 7, np.float16),
    (2, 1, (224, 512), 3, 4, np.float16),      # ragged last slab
    (2, 3, (96, 1024), 2, 3, np.float16),
    (2, 1, (128, 512), 2, 5, np.float64),      # quantised on the device, fp64 result
    (3, 1, (48, 24, 256), 3, 3, np.float16),
    (3, 1, (32, 16, 128), 2, 2, np.float32),
    (2, 4, (200, 1000), 2, 3, np.float16),     # generic radius (L = 10): staged epilogue + peer copies
])
def test_multidevice_execute_matches_one_device(d, r, shape, n, steps, dtype):
    k = _kernel(d, r)
    g = _grid(d, r, shape, dtype)
    before = g.data.copy()
    want, _ = sp.execute(k, g, steps, DeviceConfig())
    got, stats = sp.execute(k, g, steps, DeviceConfig(devices=(0,) * n))
    assert np.array_equal(g.data, before), "input grid modified"
    assert got.data.dtype == want.data.dtype
    assert got.step == want.step == steps
    assert np.array_equal(got.data, want.data)
    assert stats.device["devices"] == [0] * n


@gpu
@pytest.mark.timeout(300, method="thread")
def test_multidevice_execute_into_out_grid_repeated():
    k = _kernel(2, 1)
    g = _grid(2, 1, (512, 1024), np.float16)
    want, _ = sp.execute(k, g, 9)
    out = sp.Grid(np.empty_like(g.data), 1)
    for _ in range(2):  # fresh slabs and counters per call
        got, _ = sp.execute(k, g, 9, DeviceConfig(devices=(0, 0)), out=out)
        assert got.data is out.data
        assert np.array_equal(out.data, want.data)


@gpu
def test_multidevice_rejects_too_many_slabs():
    k = _kernel(2, 1)
    g = _grid(2, 1, (64, 512), np.float16)  # two 32-row bands
    with pytest.raises(ValueError):
        sp.execute(k, g, 2, DeviceConfig(devices=(0, 0, 0)))


@gpu
@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("d,r,shape,steps,halo,windows", [
    (2, 1, (4096, 4096), 8, 1, None),     # default window count from the cost model
    (2, 1, (1000, 512), 7, 1, 3),         # ragged extent
    (2, 3, (384, 1024), 3, 3, 3),
    (2, 1, (256, 512), 2, 2, 2),          # grid halo > r
    (3, 1, (64, 32, 256), 2, 1, None),    # 3D: staged window uploads
])
def test_streamed_execute_matches_whole_grid(monkeypatch, d, r, shape, steps, halo, windows):
    k = _kernel(d, r)
    rng = np.random.default_rng([7, *shape])
    data = rng.uniform(-1, 1, tuple(s + 2 * halo for s in shape)).astype(np.float16)
    g = sp.Grid3D(data, halo) if d == 3 else sp.Grid(data, halo)
    monkeypatch.setenv("SPD_STREAM_WINDOWS", "0")
    want, st0 = sp.execute(k, g, steps)
    assert "streamed_windows" not in st0.device
    monkeypatch.setenv("SPD_STREAM_WINDOWS", str(windows) if windows else "")
    if windows is None:
        monkeypatch.delenv("SPD_STREAM_WINDOWS")
    for _ in range(2):
        got, st = sp.execute(k, g, steps)
        assert st.device["streamed_windows"] >= 2
        assert np.array_equal(got.data, want.data)


@gpu
@pytest.mark.timeout(300, method="thread")
def test_multidevice_bf16_matches_one_device():
    k = _kernel(2, 1)
    g = _grid(2, 1, (256, 512), np.float64)
    want, _ = sp.execute(k, g, 3, DeviceConfig(dtype="bf16"))
    got, _ = sp.execute(k, g, 3, DeviceConfig(dtype="bf16", devices=(0, 0)))
    assert np.array_equal(got.data, want.data)


@gpu
@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("two_launch", ["0", "1"])
def test_multidevice_long_run_both_slab_forms(monkeypatch, two_launch):
    """64 steps on 3 slabs: the in-kernel peer copies and the flag protocol
    stay exact over many exchanges, in both slab launch forms."""
    monkeypatch.setenv("SPD_SLAB_TWO_LAUNCH", two_launch)
    k = _kernel(2, 1)
    g = _grid(2, 1, (1536, 2048), np.float16)
    monkeypatch.setenv("SPD_STREAM_WINDOWS", "0")
    want, _ = sp.execute(k, g, 64)
    got, _ = sp.execute(k, g, 64, DeviceConfig(devices=(0, 0, 0)))
    assert np.array_equal(got.data, want.data)
