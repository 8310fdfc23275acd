"""Multi-rank slab driver on CPU: world_size 2 (and 3) over gloo.

The same SlabDriver orchestration the GPUs run (boundary bands first, halo
exchange, interior, flip) drives a host double whose per-step compute is the
oracle; the gathered result must equal the oracle on the undecomposed grid bit
for bit (every point sees identical fp64 arithmetic)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import naive
from paper_2506_22035_b200.distributed import SlabDriver, SlabOps, decompose


class HostSlabOps(SlabOps):
    def __init__(self, coeffs, d, r, local_dense, band):
        self.coeffs, self.d, self.r = coeffs, d, r
        self.cur = torch.from_numpy(local_dense.copy())
        self.nxt = self.cur.clone()
        self.rows = local_dense.shape[0] - 2 * r
        self.band = band
        self._full = None

    def compute(self, lo, hi):
        if self._full is None:
            self._full = torch.from_numpy(naive.naive_apply(self.coeffs, self.d, self.r, self.cur.numpy(), self.r, 1))
        h = self.r
        if self.d == 3:
            self.nxt[h + lo : h + hi, h:-h, h:-h] = self._full[h + lo : h + hi, h:-h, h:-h]
        else:
            self.nxt[h + lo : h + hi, h:-h] = self._full[h + lo : h + hi, h:-h]

    def flip(self):
        self.cur, self.nxt = self.nxt, self.cur
        self._full = None

    def new_message(self):
        return torch.empty((self.r,) + tuple(self.cur.shape[1:]), dtype=torch.float64)

    def pack(self, which, msg):
        h = self.r
        rows = slice(h, 2 * h) if which == "up" else slice(h + self.rows - h, h + self.rows)
        msg.copy_(self.nxt[rows])

    def unpack(self, which, msg):
        h = self.r
        rows = slice(0, h) if which == "up" else slice(h + self.rows, 2 * h + self.rows)
        self.nxt[rows] = msg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, d, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r = 1
        rng = np.random.default_rng(123)
        shape = (12, 10, 16) if d == 3 else (40, 24)
        dense = rng.uniform(-1, 1, tuple(s + 2 * r for s in shape))
        coeffs = rng.uniform(-1, 1, (3,) * d)
        band = 2
        slab = decompose(shape[0], world, rank, align=band)
        local = dense[slab.lo : slab.hi + 2 * r]
        ops = HostSlabOps(coeffs, d, r, local, band)
        drv = SlabDriver(slab, ops)
        for _ in range(steps):
            drv.step()
        res = ops.cur.numpy()[r : r + slab.rows]
        q.put((rank, slab.lo, slab.hi, res))
        if rank == 0:
            want = naive.naive_apply(coeffs, d, r, dense, r, steps)
            q.put(("want", want))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,d", [(2, 2), (3, 2), (2, 3)])
def test_slab_driver_matches_global_oracle(world, d):
    steps = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, d, steps, q)) for rk in range(world)]
    for p in procs:
        p.start()
    got = {}
    want = None
    for _ in range(world + 1):
        item = q.get(timeout=120)
        if item[0] == "want":
            want = item[1]
        else:
            got[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r = 1
    for rank, (lo, hi, res) in got.items():
        if d == 3:
            np.testing.assert_array_equal(res[:, r:-r, r:-r], want[r + lo : r + hi, r:-r, r:-r])
        else:
            np.testing.assert_array_equal(res[:, r:-r], want[r + lo : r + hi, r:-r])


def test_decompose_tile_aligned():
    s = [decompose(10240, 8, k, align=32) for k in range(8)]
    assert s[0].lo == 0 and s[-1].hi == 10240
    assert all(a.hi == b.lo for a, b in zip(s, s[1:]))
    assert all(x.lo % 32 == 0 for x in s)
    assert {x.rows for x in s} == {1280}
    with pytest.raises(ValueError):
        decompose(40, 8, 0, align=32)
