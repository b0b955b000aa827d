"""Screen-band sharding with an exact exchange.

Each rank renders a contiguous band of image rows.  The learned cut state
must evolve exactly as in one render_pass over the whole image, and the
ordered, floored EMA of update_q (proj/src/cut.cpp:76-86) cannot be merged
by summing deltas.  So every rank all-gathers the ranks' update records
(cell key, cluster, v; 32 B each) and folds all of them in canonical order
-- rank-major order is canonical because bands are consecutive -- which
keeps the cut tables bit-identical on every rank.  Each rank then forms the
radiance of its own band.

The protocol is written once over an *engine* (GpuEngine: the B200 path,
NCCL over NVLink; OracleEngine: the CPU restatement, gloo) so the multi-rank
logic is exercised on CPU by the test-suite.
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


class _CudaView:
    """Zero-copy torch view of device memory owned by the C library."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class GpuEngine:
    """The B200 path: rlc_pass_trace / rlc_pass_fold / rlc_end_of_pass_update."""

    def __init__(self, ctx, grid, fb, cfg, device: torch.device):
        self.ctx, self.grid, self.fb, self.cfg, self.device = ctx, grid, fb, cfg, device
        self._ptr, self._n = 0, 0

    def trace(self, pass_index: int, rows) -> int:
        self._ptr, self._n = rlcuts.pass_trace(self.ctx, self.cfg, pass_index, self.grid, rows)
        return self._n

    def records(self) -> torch.Tensor:
        if self._n == 0:
            return torch.zeros(0, dtype=torch.uint8, device=self.device)
        return torch.as_tensor(_CudaView(self._ptr, self._n * RECORD_BYTES), device=self.device)

    def fold(self, all_records: torch.Tensor, counts, rank: int, stride: int):
        # the gather ran on torch's stream; the library works on its own stream
        torch.cuda.current_stream(self.device).synchronize()
        rlcuts.pass_fold(self.ctx, self.cfg, self.grid, self.fb, all_records.data_ptr(), counts,
                         rank, stride)

    def end_of_pass(self) -> int:
        return rlcuts.end_of_pass_update(self.grid, self.ctx, self.cfg.cut)


class OracleEngine:
    """The CPU restatement (oracle/): the same protocol on host memory."""

    def __init__(self, run):
        self.run = run
        self.device = torch.device("cpu")

    def trace(self, pass_index: int, rows) -> int:
        return self.run.trace(pass_index, rows)

    def records(self) -> torch.Tensor:
        return torch.from_numpy(self.run.records().view(np.uint8).copy())

    def fold(self, all_records: torch.Tensor, counts, rank: int, stride: int):
        self.run.fold(all_records.numpy().view(rlcuts.RECORD_DTYPE), counts, rank, stride)

    def end_of_pass(self) -> int:
        return self.run.end_of_pass()


class ShardedFrame:
    """One rank's share of a sharded frame."""

    def __init__(self, engine, height: int, rank: int, world: int, group=None,
                 host_staging: bool = False):
        self.engine, self.rank, self.world, self.group = engine, rank, world, group
        self.rows = band(height, rank, world)
        self.last_counts = [0] * world
        # gloo cannot all-gather device tensors: stage through host memory
        self.host_staging = host_staging

    def exchange(self, n: int) -> tuple[torch.Tensor, list, int]:
        dev = torch.device("cpu") if self.host_staging else self.engine.device
        cnt = torch.tensor([n], dtype=torch.int64, device=dev)
        counts_t = [torch.zeros_like(cnt) for _ in range(self.world)]
        dist.all_gather(counts_t, cnt, group=self.group)
        counts = [int(c.item()) for c in counts_t]
        stride = max(max(counts), 1)
        send = torch.zeros(stride * RECORD_BYTES, dtype=torch.uint8, device=dev)
        if n:
            send[: n * RECORD_BYTES] = self.engine.records().to(dev)
        parts = [torch.empty_like(send) for _ in range(self.world)]
        dist.all_gather(parts, send, group=self.group)
        return torch.cat(parts).to(self.engine.device), counts, stride

    def step(self, pass_index: int) -> int:
        """render_pass + end_of_pass_update for this rank's band; returns the
        split-collapse change count (identical on every rank)."""
        n = self.engine.trace(pass_index, self.rows)
        all_records, counts, stride = self.exchange(n)
        self.last_counts = counts
        self.engine.fold(all_records, counts, self.rank, stride)
        return self.engine.end_of_pass()


def local_exchange(engines, heights_rows, pass_index: int):
    """Single-process emulation of the exchange for N engines (tests on one
    device): every engine traces its band, records are concatenated in rank
    order, every engine folds all of them.  No kernel waits on another."""
    counts = [e.trace(pass_index, rows) for e, rows in zip(engines, heights_rows)]
    stride = max(max(counts), 1)
    parts = []
    for e, n in zip(engines, counts):
        buf = torch.zeros(stride * RECORD_BYTES, dtype=torch.uint8, device=e.device)
        if n:
            buf[: n * RECORD_BYTES] = e.records()
        parts.append(buf)
    all_records = torch.cat(parts)
    for r, e in enumerate(engines):
        e.fold(all_records, counts, r, stride)
    return [e.end_of_pass() for e in engines]
