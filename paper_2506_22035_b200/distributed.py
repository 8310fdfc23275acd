"""Multi-GPU slab driver: domain decomposition with one halo exchange per step.

The reference has no distribution; per SURVEY.md §8(e) the
grid is cut into contiguous slabs along the slowest axis (y in 2D, z in 3D),
one rank per GPU.  Each step:

  1. the two boundary tile bands of the slab are computed first
     (compute stream);
  2. their r outermost rows are packed and exchanged with the y-1 / y+1 ranks
     by NCCL send/recv on a communication stream, then unpacked into the halo
     rows of the freshly written buffer — overlapped with
  3. the interior bands (compute stream);
  4. the compute stream waits for the exchange before the next step reads the
     halos.

Outer ranks keep the global Dirichlet halo.  The orchestration is written
against `SlabOps` so the exchange logic is tested with gloo on CPU
(tests/test_distributed.py) while the device ops call libspider.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from ._lib import check, lib
from .engine import DeviceGrid, Plan, _stream_ptr


@dataclass(frozen=True)
class Slab:
    """Rows [lo, hi) of a global extent owned by `rank` of `world`."""

    rank: int
    world: int
    lo: int
    hi: int

    @property
    def rows(self) -> int:
        return self.hi - self.lo

    @property
    def up(self) -> int | None:
        return self.rank - 1 if self.rank > 0 else None

    @property
    def down(self) -> int | None:
        return self.rank + 1 if self.rank < self.world - 1 else None


def decompose(global_rows: int, world: int, rank: int, align: int = 1) -> Slab:
    """Contiguous split; slab boundaries are multiples of `align` (the tile
    height) except the last, so boundary bands are whole tiles."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    units = -(-global_rows // align)
    if units < world:
        raise ValueError(f"{global_rows} rows cannot be split into {world} slabs of {align}-row tiles")
    lo = (units * rank // world) * align
    hi = min(global_rows, (units * (rank + 1) // world) * align)
    return Slab(rank, world, lo, hi)


def exchange(slab: Slab, send_up, send_down, recv_up, recv_down, group=None) -> None:
    """Post the neighbour sends/receives of one step and wait for them.
    Works on CUDA tensors (NCCL) and CPU tensors (gloo)."""
    ops = []
    if slab.up is not None:
        ops.append(dist.P2POp(dist.isend, send_up, slab.up, group))
        ops.append(dist.P2POp(dist.irecv, recv_up, slab.up, group))
    if slab.down is not None:
        ops.append(dist.P2POp(dist.isend, send_down, slab.down, group))
        ops.append(dist.P2POp(dist.irecv, recv_down, slab.down, group))
    if not ops:
        return
    for req in dist.batch_isend_irecv(ops):
        req.wait()


class SlabOps:
    """What the driver needs from a local slab (device or test double)."""

    r: int
    rows: int
    band: int

    def compute(self, lo: int, hi: int) -> None:  # one step over local rows [lo, hi)
        raise NotImplementedError

    def flip(self) -> None:
        raise NotImplementedError

    def pack(self, which: str, msg) -> None:  # 'up': rows [0, r); 'down': rows [rows-r, rows)
        raise NotImplementedError

    def unpack(self, which: str, msg) -> None:  # 'up': halo rows [-r, 0); 'down': [rows, rows+r)
        raise NotImplementedError

    def new_message(self):
        raise NotImplementedError


class SlabDriver:
    """Runs steps of a slab with boundary-first compute and overlapped exchange."""

    def __init__(self, slab: Slab, ops: SlabOps, group=None, comm_stream=None, compute_stream=None):
        # an interior slab face must sit on a tile-band boundary: otherwise the
        # 'down' pack reads rows of the interior band, which is computed
        # concurrently with (or after) the exchange
        if slab.down is not None and ops.rows % ops.band != 0:
            raise ValueError(f"slab of {ops.rows} rows has an interior face off the {ops.band}-row tile bands "
                             f"(use decompose(..., align={ops.band}))")
        self.slab, self.ops, self.group = slab, ops, group
        self.msgs = {k: ops.new_message() for k in ("send_up", "send_down", "recv_up", "recv_down")}
        self.comm_stream = comm_stream
        self.compute_stream = compute_stream

    def _bands(self):
        """(boundary, interior) row ranges: the first and the last tile band,
        and everything between (slab boundaries are tile-aligned except the
        global bottom, which exchanges nothing downward)."""
        rows, band = self.ops.rows, self.ops.band
        last = ((rows - 1) // band) * band  # first row of the last tile band
        if last <= band:
            return [(0, rows)], []
        return [(0, band), (last, rows)], [(band, last)]

    def _compute_boundary(self, boundary) -> None:
        if len(boundary) == 2 and hasattr(self.ops, "compute_edges"):
            self.ops.compute_edges()  # both edge bands in one launch
        else:
            for lo, hi in boundary:
                self.ops.compute(lo, hi)

    def step(self) -> None:
        """One timestep: boundary bands, exchange (overlapped on the comm
        stream when CUDA), interior bands, flip."""
        boundary, interior = self._bands()
        self._compute_boundary(boundary)
        if self.comm_stream is not None:
            done = torch.cuda.Event()
            done.record(self.compute_stream)
            with torch.cuda.stream(self.comm_stream):
                self.comm_stream.wait_event(done)
                self._exchange()
                exchanged = torch.cuda.Event()
                exchanged.record(self.comm_stream)
            for lo, hi in interior:
                self.ops.compute(lo, hi)
            self.compute_stream.wait_event(exchanged)
        else:
            self._exchange()
            for lo, hi in interior:
                self.ops.compute(lo, hi)
        self.ops.flip()

    # phase API (used to emulate several ranks in one process)
    def step_boundary(self) -> None:
        self._compute_boundary(self._bands()[0])

    def pack_messages(self) -> None:
        m, s = self.msgs, self.slab
        if s.up is not None:
            self.ops.pack("up", m["send_up"])
        if s.down is not None:
            self.ops.pack("down", m["send_down"])

    def unpack_messages(self) -> None:
        m, s = self.msgs, self.slab
        if s.up is not None:
            self.ops.unpack("up", m["recv_up"])
        if s.down is not None:
            self.ops.unpack("down", m["recv_down"])

    def step_interior_and_flip(self) -> None:
        for lo, hi in self._bands()[1]:
            self.ops.compute(lo, hi)
        self.ops.flip()

    def _exchange(self) -> None:
        m, s = self.msgs, self.slab
        self.pack_messages()
        exchange(s, m["send_up"], m["send_down"], m["recv_up"], m["recv_down"], self.group)
        self.unpack_messages()


def local_exchange(drivers) -> None:
    """Exchange halos between SlabDrivers living in one process (ranks
    emulated on one device): rank k's send_down -> rank k+1's recv_up etc."""
    for a, b in zip(drivers, drivers[1:]):
        b.msgs["recv_up"].copy_(a.msgs["send_down"])
        a.msgs["recv_down"].copy_(b.msgs["send_up"])


class DeviceSlabOps(SlabOps):
    """libspider-backed slab: a DeviceGrid whose halo rows at inner slab faces
    are refreshed by the exchange (outer faces keep the global Dirichlet halo)."""

    def __init__(self, plan: Plan, local_shape, halo: int, stream=None):
        self.grid = DeviceGrid(plan, local_shape, halo)
        self.plan = plan
        self.r = plan.kernel.r
        self.rows = int(local_shape[0])
        self.band = plan.info().tile_z if plan.kernel.d == 3 else plan.info().tile_y
        self.stream = stream
        d = self.grid.desc
        self.unit = d.plane if plan.kernel.d == 3 else d.pitch

    def compute(self, lo: int, hi: int) -> None:
        self.grid.step_range(lo, hi, self.stream)

    def compute_edges(self) -> None:
        self.grid.step_edges(self.stream)

    def flip(self) -> None:
        self.grid.flip()

    def new_message(self):
        return torch.empty(self.r * self.unit, dtype=self.grid.bufs[0].dtype, device=self.grid.bufs[0].device)

    def _out(self):
        return self.grid.bufs[1 - self.grid.cur]  # buffer being written this step

    def pack(self, which: str, msg) -> None:
        check(lib.spd_halo_pack(C.byref(self.grid.desc), C.c_void_p(self._out().data_ptr()), self.r,
                                0 if which == "up" else 1, C.c_void_p(msg.data_ptr()), _stream_ptr()))

    def unpack(self, which: str, msg) -> None:
        check(lib.spd_halo_unpack(C.byref(self.grid.desc), C.c_void_p(self._out().data_ptr()), self.r,
                                  0 if which == "up" else 1, C.c_void_p(msg.data_ptr()), _stream_ptr()))


__all__ = ["Slab", "decompose", "exchange", "local_exchange", "SlabOps", "SlabDriver", "DeviceSlabOps"]


# ---------------------------------------------------------------------------
# Peer-memory exchange (CUDA IPC + stream memory operations), csrc/peer.cu


def _desc_tuple(d) -> tuple:
    return (d.nz, d.ny, d.nx, d.halo, d.dims, d.pitch, d.plane, d.origin, d.alloc_elems)


def _desc_from(t):
    from ._lib import spd_grid_desc

    d = spd_grid_desc()
    d.nz, d.ny, d.nx, d.halo, d.dims, d.pitch, d.plane, d.origin, d.alloc_elems = t
    return d


def _ipc_export(t: torch.Tensor):
    handle = C.create_string_buffer(64)
    off = C.c_int64(0)
    check(lib.spd_ipc_export(C.c_void_p(t.data_ptr()), handle, C.byref(off)))
    return handle.raw, int(off.value)


def _check_peer_access(dev: torch.device, peer_uuid: str) -> None:
    """Raise unless this process can map memory of the GPU `peer_uuid` (the
    same device, or a peer-capable visible one: NVLink / PCIe P2P)."""
    for i in range(torch.cuda.device_count()):
        if str(torch.cuda.get_device_properties(i).uuid) == peer_uuid:
            if i == dev.index or torch.cuda.can_device_access_peer(dev.index, i):
                return
            raise RuntimeError(f"cuda:{dev.index} cannot access peer cuda:{i}")
    raise RuntimeError(f"neighbour GPU {peer_uuid} is not visible to this process")


class PeerSlab:
    """One rank's slab whose halo rows are exchanged through peer memory: the
    neighbours' grid buffers and flag words are mapped with CUDA IPC, the
    boundary rows go by copy engine straight into the neighbours' halos and a
    stream memory operation signals them (spd_slab_step).  One host call per
    step, no NCCL and no host synchronisation on the data path.  Setup is a
    collective over `group` (any backend: it only all-gathers the handles).

    The grid must be fully initialised (both buffers, halos included) before
    construction: the constructor synchronises and barriers, after which the
    neighbours may write into this rank's halos."""

    def __init__(self, plan: Plan, slab: Slab, grid: DeviceGrid, group=None, compute_stream=None, comm_stream=None):
        self.plan, self.slab, self.grid = plan, slab, grid
        dev = grid.bufs[0].device
        self.flags = torch.zeros(2, dtype=torch.int32, device=dev)
        self.compute_stream = compute_stream or torch.cuda.current_stream(dev)
        self.comm_stream = comm_stream or torch.cuda.Stream(dev)
        self._bases = []
        self._descs = {}
        self._h = None
        try:
            mine = {
                "bufs": [_ipc_export(b) for b in grid.bufs],
                "flags": _ipc_export(self.flags),
                "desc": _desc_tuple(grid.desc),
                "uuid": str(torch.cuda.get_device_properties(dev).uuid),
            }
        except Exception as exc:  # every rank must reach the all-gather
            mine = {"error": f"rank {dist.get_rank(group)}: {exc}"}
        torch.cuda.synchronize(dev)
        world = dist.get_world_size(group)
        everyone = [None] * world
        dist.all_gather_object(everyone, mine, group=group)
        failed = [e["error"] for e in everyone if "error" in e]
        if failed:
            raise RuntimeError("peer-memory exchange unavailable: " + "; ".join(failed))

        def open_peer(rank):
            if rank is None:
                return None, None, None, None
            info = everyone[rank]
            _check_peer_access(dev, info["uuid"])
            ptrs = []
            for handle, off in info["bufs"] + [info["flags"]]:
                p, base = C.c_void_p(), C.c_void_p()
                check(lib.spd_ipc_open(C.create_string_buffer(handle, 64), off, C.byref(p), C.byref(base)))
                self._bases.append(base)
                ptrs.append(p)
            desc = _desc_from(info["desc"])
            self._descs[rank] = desc
            return ptrs[0], ptrs[1], desc, ptrs[2]

        err = None
        try:
            ub0, ub1, ud, uf = open_peer(slab.up)
            db0, db1, dd, df = open_peer(slab.down)
            h = C.c_void_p()
            check(lib.spd_slab_create(
                plan.handle, C.byref(grid.desc), C.c_void_p(grid.bufs[0].data_ptr()),
                C.c_void_p(grid.bufs[1].data_ptr()), C.c_void_p(self.flags.data_ptr()), ub0, ub1,
                C.byref(ud) if ud is not None else None, uf, db0, db1, C.byref(dd) if dd is not None else None, df,
                C.byref(h)))
            self._h = h
        except Exception as exc:  # decided collectively below: all ranks or none
            err = f"rank {dist.get_rank(group)}: {exc}"
        errors = [None] * world
        dist.all_gather_object(errors, err, group=group)
        errors = [e for e in errors if e]
        if errors:
            self.close()
            raise RuntimeError("peer-memory exchange unavailable: " + "; ".join(errors))
        self.t = 0
        dist.barrier(group=group)

    def step(self) -> None:
        if self.grid.cur != (self.t & 1):
            raise RuntimeError("the slab grid was stepped outside PeerSlab")
        check(lib.spd_slab_step(self._h, self.t, C.c_void_p(self.compute_stream.cuda_stream),
                                C.c_void_p(self.comm_stream.cuda_stream)))
        self.t += 1
        self.grid.flip()

    def close(self) -> None:
        torch.cuda.synchronize(self.grid.bufs[0].device)
        if getattr(self, "_h", None):
            lib.spd_slab_destroy(self._h)
            self._h = None
        for b in getattr(self, "_bases", []):
            lib.spd_ipc_close(b)
        self._bases = []


__all__ += ["PeerSlab"]


# ---------------------------------------------------------------------------
# Several devices driven by one process: execute(..., DeviceConfig(devices=...))


def enable_peer_access(devices) -> None:
    """Direct peer access between neighbouring devices of a slab chain (both
    directions); raises ValueError when a pair has no peer path."""
    for a, b in zip(devices, devices[1:]):
        if a != b:
            check(lib.spd_peer_enable(int(a), int(b)))
            check(lib.spd_peer_enable(int(b), int(a)))


class LocalSlabs:
    """A grid cut into slabs along y (2D) / z (3D), one per entry of
    `devices` (entries may repeat: several slabs on one device), all driven
    by this process.  The halo exchange is the peer-memory one of PeerSlab
    (csrc/peer.cu: boundary bands published by the step kernel, copy engine
    into the neighbour's halo rows, stream-memory-op flags), with the
    neighbours' buffers passed as plain device pointers instead of IPC
    mappings.  Each slab's steps are issued by one native call
    (spd_slab_run) on its own host thread, so the host cost does not grow
    with the device count.

    `plans` maps device -> Plan; `shape` is the global interior shape."""

    def __init__(self, plans: dict, devices, shape, halo: int):
        devices = [int(v) for v in devices]
        if not devices:
            raise ValueError("no devices given")
        plan0 = plans[devices[0]]
        d = plan0.kernel.d
        if d == 1:
            raise ValueError("1D grids cannot be cut into slabs")
        info = plan0.info()
        self.band = info.tile_z if d == 3 else info.tile_y
        self.devices, self.shape, self.halo, self.d = devices, tuple(int(v) for v in shape), int(halo), d
        world = len(devices)
        self.slabs = [decompose(self.shape[0], world, k, align=self.band) for k in range(world)]
        if any(s.rows < self.halo for s in self.slabs):
            raise ValueError(f"{self.shape[0]} rows give slabs thinner than the halo ({self.halo})")
        enable_peer_access(devices)
        self.grids = []
        self.flags = []
        self.streams = []
        for dev, slab in zip(devices, self.slabs):
            with torch.cuda.device(dev):
                self.grids.append(DeviceGrid(plans[dev], (slab.rows,) + self.shape[1:], self.halo))
                self.flags.append(torch.zeros(2, dtype=torch.int32, device=torch.device("cuda", dev)))
                self.streams.append((torch.cuda.Stream(dev), torch.cuda.Stream(dev)))
        self.handles = []

    def _create_handles(self) -> None:
        """Exchange handles over the neighbours' buffers; only once every
        slab holds its initial state (both buffers, halos included)."""
        null = None
        for k, (dev, g) in enumerate(zip(self.devices, self.grids)):
            up = self.grids[k - 1] if k > 0 else None
            dn = self.grids[k + 1] if k + 1 < len(self.grids) else None

            def ptrs(n, j):
                if n is None:
                    return null, null, null, null
                return (C.c_void_p(n.bufs[0].data_ptr()), C.c_void_p(n.bufs[1].data_ptr()), C.byref(n.desc),
                        C.c_void_p(self.flags[j].data_ptr()))

            h = C.c_void_p()
            with torch.cuda.device(dev):
                check(lib.spd_slab_create(g.plan.handle, C.byref(g.desc), C.c_void_p(g.bufs[0].data_ptr()),
                                          C.c_void_p(g.bufs[1].data_ptr()), C.c_void_p(self.flags[k].data_ptr()),
                                          *ptrs(up, k - 1), *ptrs(dn, k + 1), C.byref(h)))
            self.handles.append(h)

    def _each(self, fn) -> None:
        """fn(k) on one host thread per slab, each with its device current;
        the first failure is re-raised."""
        errors = []

        def body(k):
            try:
                with torch.cuda.device(self.devices[k]):
                    fn(k)
            except BaseException as exc:  # noqa: BLE001 - re-raised below
                errors.append(exc)

        threads = [threading.Thread(target=body, args=(k,)) for k in range(len(self.devices))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]

    def run(self, data, steps: int, native16: bool, out):
        """`steps` steps of the dense host grid `data` (halo included);
        returns the dense result (written into `out` when given)."""
        h = self.halo
        if out is not None:
            res = out
        elif native16:  # pinned: the per-slab downloads run asynchronously
            res = torch.empty(data.shape, dtype=torch.float16, pin_memory=True).numpy()
        else:
            res = np.empty(data.shape, dtype=np.float64)

        def load(k):
            s, g, (cs, _) = self.slabs[k], self.grids[k], self.streams[k]
            part = np.ascontiguousarray(data[s.lo : s.hi + 2 * h])
            if native16:
                g.upload(torch.from_numpy(part), stream=cs)
            else:
                g.load_dense_f64(torch.from_numpy(part.astype(np.float64, copy=False)).to(g.device), stream=cs)
            cs.synchronize()

        self._each(load)  # every halo holds its initial neighbour rows before any exchange writes
        self._create_handles()
        try:
            def steps_of(k):
                cs, xs = self.streams[k]
                check(lib.spd_slab_run(self.handles[k], 0, int(steps), C.c_void_p(cs.cuda_stream),
                                       C.c_void_p(xs.cuda_stream)))
                cs.synchronize()
                xs.synchronize()

            self._each(steps_of)
        finally:
            for dev, hd in zip(self.devices, self.handles):
                with torch.cuda.device(dev):
                    torch.cuda.synchronize(dev)
                    lib.spd_slab_destroy(hd)
            self.handles = []
        for g in self.grids:
            g.cur, g.step = steps % 2, g.step + steps

        def store(k):
            s, g, (cs, _) = self.slabs[k], self.grids[k], self.streams[k]
            lo, hi = s.lo + h, s.hi + h  # dense rows of the slab interior
            if k == 0:
                lo = 0
            if k == len(self.slabs) - 1:
                hi = res.shape[0]
            if native16:
                # only this slab's rows, straight into the result (pinned: async)
                row_elems = int(np.prod(res.shape[1:]))
                g.download_rows(res.ctypes.data + s.lo * row_elems * 2, lo - s.lo, hi - s.lo, stream=cs)
                cs.synchronize()
            else:
                with torch.cuda.stream(cs):
                    part = g.to_dense_f64(stream=cs).cpu().numpy()
                res[lo:hi] = part[lo - s.lo : hi - s.lo].astype(res.dtype, copy=False)

        self._each(store)
        return res


def execute_slabs(plans: dict, devices, shape, halo: int, data, steps: int, native16: bool, out=None):
    """One-process multi-device run (see LocalSlabs)."""
    return LocalSlabs(plans, devices, shape, halo).run(data, steps, native16, out)


__all__ += ["LocalSlabs", "enable_peer_access", "execute_slabs"]
