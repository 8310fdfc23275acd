"""Peer-memory slab exchange (csrc/peer.cu): 2-3 processes, one slab each,
halos written into the neighbours' buffers through CUDA IPC and signalled with
stream memory operations.  All processes share cuda:0 here (IPC between
processes on one device uses the same mechanism as between NVLink peers);
the result must equal the undecomposed single-grid run bit for bit."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _kernel(d, r):
    import paper_2506_22035_b200 as sp

    rng = np.random.default_rng([d, r, 77])
    c = rng.uniform(0.5, 1.5, (2 * r + 1,) * d)
    c /= c.sum()
    return sp.make_kernel_3d("box", r, c) if d == 3 else sp.make_kernel("box", d, r, c)


def _dense(d, r, shape):
    g = torch.Generator().manual_seed(5)
    return torch.rand(tuple(n + 2 * r for n in shape), dtype=torch.float64, generator=g) - 0.5


def _worker(rank, world, port, d, r, shape, steps, outdir):
    import torch.distributed as dist

    import paper_2506_22035_b200 as sp
    from paper_2506_22035_b200.distributed import PeerSlab, decompose
    from paper_2506_22035_b200.engine import DeviceGrid
    from paper_2506_22035_b200.pipeline import get_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    k = _kernel(d, r)
    plan = get_plan(k, sp.Parity.EVEN, "fp16")
    inf = plan.info()
    band = inf.tile_z if d == 3 else inf.tile_y
    slab = decompose(shape[0], world, rank, align=band)
    dense = _dense(d, r, shape)
    grid = DeviceGrid(plan, (slab.rows,) + tuple(shape[1:]), r)
    grid.load_dense_f64(dense[slab.lo : slab.hi + 2 * r].contiguous().cuda())
    ps = PeerSlab(plan, slab, grid)
    for _ in range(steps):
        ps.step()
    torch.cuda.synchronize()
    out = grid.to_dense_f64().cpu()
    torch.save({"lo": slab.lo, "hi": slab.hi, "data": out}, os.path.join(outdir, f"{rank}.pt"))
    dist.barrier()
    ps.close()
    dist.destroy_process_group()


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("d,r,shape,world,steps,launch", [
    (2, 1, (256, 1024), 2, 5, None),
    (2, 1, (224, 512), 3, 4, None),    # ragged last slab
    (2, 3, (96, 1024), 2, 3, None),
    (3, 1, (48, 24, 256), 3, 3, None),
    (2, 1, (256, 1024), 2, 5, "1"),    # edge launch + interior launch (large 2D slabs)
    (3, 1, (48, 24, 256), 3, 3, "0"),  # one edge-first launch (small 2D slabs)
])
def test_peer_slab_matches_single_grid(monkeypatch, d, r, shape, world, steps, launch):
    import torch.multiprocessing as mp

    if launch is not None:
        monkeypatch.setenv("SPD_SLAB_TWO_LAUNCH", launch)

    import paper_2506_22035_b200 as sp
    from paper_2506_22035_b200.engine import DeviceGrid
    from paper_2506_22035_b200.pipeline import get_plan

    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), d, r, shape, steps, tmp), nprocs=world, join=True)
        plan = get_plan(_kernel(d, r), sp.Parity.EVEN, "fp16")
        ref = DeviceGrid(plan, shape, r)
        ref.load_dense_f64(_dense(d, r, shape).cuda())
        ref.run(steps)
        want = ref.to_dense_f64().cpu()
        for rank in range(world):
            part = torch.load(os.path.join(tmp, f"{rank}.pt"))
            lo, hi, got = part["lo"], part["hi"], part["data"]
            assert torch.equal(got[r:-r], want[r + lo : r + hi]), (rank, lo, hi)
