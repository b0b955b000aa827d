"""Screen-band sharding with an exact exchange.

Each rank renders a contiguous band of image rows.  The learned cut state
must evolve exactly as in one render_pass over the whole image, and the
ordered, floored EMA of update_q (proj/src/cut.cpp:76-86) cannot be merged by
summing deltas.  Each rank files its update records (cell, cluster, v;
32 B) in canonical order into a fixed-size block; the blocks are all-gathered
(rank-major order is canonical order: bands are consecutive); every rank
inserts the pass's new keys in that order, so the hash tables stay identical
(and a record can name its cell by table slot).  The records are then folded
in canonical order per cut entry, either by every rank (replicated) or only
by the owner of the cell, table slot % nranks (owner mode): the owners'
per-record q_before values and per-entry record counts are summed over the
ranks and every rank advances the other owners' entries on its copy.  Each
rank then forms the radiance of its own band.

Three drivers of the same protocol:
  * NcclFrame -- the C++ data plane (rlc_shard_frame): NCCL all-gather and
    all-reduce on the context stream, no host synchronization per frame; or
    (peer=True) every rank storing its records straight into every rank's
    receive buffer over NVLink, one barrier all-reduce per frame;
  * ShardedFrame -- the same steps with torch.distributed collectives (gloo
    stages through host memory: functional multi-process runs);
  * local_exchange -- N ranks emulated as N contexts on one device, the
    collectives done by the host between the steps (no kernel waits on
    another rank);
and OracleFrame, the CPU restatement's model of the replicated protocol over
gloo (tests/test_dist.py).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import rlcuts

RECORD_BYTES = rlcuts.RECORD_DTYPE.itemsize  # 32


def band(height: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [r0, r1) of `rank`: consecutive bands in rank order."""
    return (height * rank) // world, (height * (rank + 1)) // world


def record_capacity(cfg, width: int, height: int, world: int) -> int:
    """Record slots per rank block: the largest band's path vertices."""
    rows = max(b - a for a, b in (band(height, r, world) for r in range(world)))
    return max(1, rows * width * (cfg.spp // cfg.passes) * max(cfg.max_depth, 1))


class _CudaView:
    """Zero-copy torch view of device memory owned by the C library."""

    def __init__(self, ptr: int, nbytes: int, typestr: str = "|u1"):
        self.__cuda_array_interface__ = {"shape": (nbytes // int(typestr[-1]),), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class GpuEngine:
    """One rank's B200 path: rlc_shard_trace / _fold / _finish, end_of_pass."""

    def __init__(self, ctx, grid, fb, cfg, device: torch.device, cap: int | None = None,
                 world: int = 1):
        self.ctx, self.grid, self.fb, self.cfg, self.device = ctx, grid, fb, cfg, device
        cam = ctx.scene.camera
        self.cap = cap or record_capacity(cfg, cam.width, cam.height, world)

    def trace(self, pass_index: int, rows) -> torch.Tensor:
        ptr, nbytes = rlcuts.shard_trace(self.ctx, self.cfg, pass_index, self.grid, rows, self.cap)
        return torch.as_tensor(_CudaView(ptr, nbytes), device=self.device)

    def trace_to(self, pass_index: int, rows, rank: int, dsts) -> None:
        """The band's records stored straight into every buffer of `dsts`
        (each nranks blocks) at block `rank`."""
        rlcuts.shard_trace_to(self.ctx, self.cfg, pass_index, self.grid, rows, self.cap, rank,
                              [d.data_ptr() for d in dsts])

    def fold(self, gathered: torch.Tensor, nranks: int, rank: int, owner: bool):
        """-> the arrays owner mode sums over the ranks: q_before per exchange
        slot, then either the records per cut entry at its last slot or (the
        entry exchange) each entry's final q and record count.  `gathered`
        must stay alive until finish()."""
        ptr, seg, n = rlcuts.shard_fold(self.ctx, self.cfg, self.grid, gathered.data_ptr(), nranks,
                                        rank, owner)
        out = [torch.as_tensor(_CudaView(ptr, 8 * n, "<f8"), device=self.device)]
        if seg:
            out.append(torch.as_tensor(_CudaView(seg, 4 * n, "<i4"), device=self.device))
        else:
            eq, en, m = rlcuts.shard_entry_arrays(self.ctx)
            if m:
                out.append(torch.as_tensor(_CudaView(eq, 8 * m, "<f8"), device=self.device))
                out.append(torch.as_tensor(_CudaView(en, 4 * m, "<i4"), device=self.device))
        return out

    def finish(self, rank: int, owner: bool):
        rlcuts.shard_finish(self.ctx, self.grid, self.fb, rank, owner)

    def end_of_pass(self) -> int:
        return rlcuts.end_of_pass_update(self.grid, self.ctx, self.cfg.cut)


class ShardedFrame:
    """One rank's share of a sharded frame over torch.distributed."""

    def __init__(self, engine: GpuEngine, height: int, rank: int, world: int, group=None,
                 host_staging: bool = False, owner: bool = True):
        self.engine, self.rank, self.world, self.group = engine, rank, world, group
        self.rows = band(height, rank, world)
        self.owner = owner
        # gloo cannot all-gather device tensors: stage through host memory
        self.host_staging = host_staging

    def _sync(self):
        # the library's stream -> torch's collective (same stream under the
        # bench; a full sync keeps the functional gloo path simple)
        self.engine.ctx.synchronize()

    def step(self, pass_index: int) -> int:
        """render_pass + end_of_pass_update for this rank's band; returns the
        split-collapse change count (identical on every rank)."""
        e = self.engine
        block = e.trace(pass_index, self.rows)
        self._sync()
        dev = torch.device("cpu") if self.host_staging else e.device
        send = block.to(dev)
        parts = [torch.empty_like(send) for _ in range(self.world)]
        dist.all_gather(parts, send, group=self.group)
        gathered = torch.cat(parts).to(e.device)
        torch.cuda.synchronize(e.device)
        arrays = e.fold(gathered, self.world, self.rank, self.owner)
        if self.owner and self.world > 1:
            self._sync()
            for a in arrays:  # (the uint32 counts viewed as int32: they stay below 2^31)
                t = a.to(dev)
                dist.all_reduce(t, group=self.group)
                a.copy_(t.to(e.device))
            torch.cuda.synchronize(e.device)
        e.finish(self.rank, self.owner)
        out = e.end_of_pass()
        del gathered  # read by finish() on the context stream (end_of_pass synchronized)
        return out


class NcclFrame:
    """One rank's share of a sharded frame over the C++ NCCL data plane
    (rlc_shard_frame): one library call per frame, no host synchronization."""

    def __init__(self, engine: GpuEngine, height: int, rank: int, world: int, device_index: int,
                 owner: bool = True, peer: bool = False):
        self.engine, self.rank, self.world = engine, rank, world
        self.rows = band(height, rank, world)
        self.owner = owner
        obj = [rlcuts.Comm.unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        self.comm = rlcuts.Comm(device_index, world, rank, obj[0])
        if peer:  # records by peer memory (CUDA IPC), one barrier all-reduce per frame
            self.comm.enable_peer_exchange(engine.cap)

    def step(self, pass_index: int) -> None:
        e = self.engine
        rlcuts.shard_frame(e.ctx, e.cfg, pass_index, e.grid, e.fb, self.comm, self.rows, e.cap,
                           self.owner)

    def run(self, first_pass: int, count: int, graph: bool = True) -> None:
        """`count` frames in one call, replayed from a captured CUDA graph."""
        e = self.engine
        rlcuts.shard_frames(e.ctx, e.cfg, first_pass, count, e.grid, e.fb, self.comm, self.rows,
                            e.cap, self.owner, graph)


def local_exchange(engines, heights_rows, pass_index: int, owner: bool = True,
                   serial: bool = False, peer_buffers=None):
    """Single-process emulation of the exchange for N engines (tests on one
    device): every engine traces its band, the blocks are concatenated in
    rank order, every engine folds; in owner mode the per-slot q_before
    arrays are summed and handed back.  No kernel waits on another.
    serial: one rank's work at a time (per-rank timing without the other
    ranks' kernels sharing the device)."""
    n = len(engines)
    if peer_buffers is not None:
        # the peer exchange's data path: every rank stores its records into
        # every rank's buffer (here all on one device), each folds its own
        for r, (e, rows) in enumerate(zip(engines, heights_rows)):
            e.trace_to(pass_index, rows, r, peer_buffers)
            if serial:
                e.ctx.synchronize()
        for e in engines:
            e.ctx.synchronize()
        sources = list(peer_buffers)
    else:
        blocks = []
        for e, rows in zip(engines, heights_rows):
            blocks.append(e.trace(pass_index, rows))
            if serial:
                e.ctx.synchronize()
        for e in engines:
            e.ctx.synchronize()
        gathered = torch.cat([b.clone() for b in blocks])
        sources = [gathered] * n
    torch.cuda.synchronize()
    arrays = []
    for r, e in enumerate(engines):
        arrays.append(e.fold(sources[r], n, r, owner))
        if serial:
            e.ctx.synchronize()
    for e in engines:
        e.ctx.synchronize()
    if owner and n > 1:
        for k in range(len(arrays[0])):  # q_before, then the counts (or entry finals)
            total = torch.stack([a[k].clone() for a in arrays]).sum(0)
            for a in arrays:
                a[k].copy_(total.to(a[k].dtype))
        torch.cuda.synchronize()
    for r, e in enumerate(engines):
        e.finish(r, owner)
        if serial:
            e.ctx.synchronize()
    return [e.end_of_pass() for e in engines]


class OracleEngine:
    """The CPU restatement (oracle/): the replicated protocol on host memory."""

    def __init__(self, run):
        self.run = run

    def trace(self, pass_index: int, rows) -> torch.Tensor:
        n = self.run.trace(pass_index, rows)
        return torch.from_numpy(self.run.records().view(np.uint8).copy()), n

    def fold(self, all_records: torch.Tensor, counts, rank: int, stride: int):
        self.run.fold(all_records.numpy().view(rlcuts.RECORD_DTYPE), counts, rank, stride)

    def end_of_pass(self) -> int:
        return self.run.end_of_pass()


class OracleFrame:
    """One rank's share of a sharded frame of the CPU model over gloo."""

    def __init__(self, engine: OracleEngine, height: int, rank: int, world: int, group=None):
        self.engine, self.rank, self.world, self.group = engine, rank, world, group
        self.rows = band(height, rank, world)

    def step(self, pass_index: int) -> int:
        recs, n = self.engine.trace(pass_index, self.rows)
        cnt = torch.tensor([n], dtype=torch.int64)
        counts_t = [torch.zeros_like(cnt) for _ in range(self.world)]
        dist.all_gather(counts_t, cnt, group=self.group)
        counts = [int(c.item()) for c in counts_t]
        stride = max(max(counts), 1)
        send = torch.zeros(stride * RECORD_BYTES, dtype=torch.uint8)
        if n:
            send[: n * RECORD_BYTES] = recs
        parts = [torch.empty_like(send) for _ in range(self.world)]
        dist.all_gather(parts, send, group=self.group)
        self.engine.fold(torch.cat(parts), counts, self.rank, stride)
        return self.engine.end_of_pass()
