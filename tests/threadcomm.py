"""Thread-backed stand-in for engine.Comm (TEST INFRASTRUCTURE ONLY).

Runs G "ranks" as Python threads in one process on one GPU, so the
product's sharded run_pipeline orchestration (symmetric super-tile ranges,
the all-to-alls, the fold-stack all-gather, the MIN all-reduces of every
Boruvka round) executes end to end on the real CUDA kernels.  Collectives
are host-level barriers over device tensors: no rank's kernel ever waits on
another's, so this is a functional check of the multi-GPU path, not a
stand-in for its performance.
"""
from __future__ import annotations

import threading

import torch


class ThreadGroup:
    def __init__(self, world: int):
        self.world = world
        self.slots = [None] * world
        self.barrier = threading.Barrier(world)

    def exchange(self, rank: int, value):
        """Every rank posts `value`; returns the list of all ranks' values."""
        torch.cuda.synchronize()
        self.slots[rank] = value
        self.barrier.wait()
        out = list(self.slots)
        self.barrier.wait()
        return out


class ThreadComm:
    """Same interface as engine.Comm for one rank of a ThreadGroup."""

    def __init__(self, group: ThreadGroup, rank: int):
        self.g, self.rank, self.world = group, rank, group.world

    def rows(self, n: int, rank=None):
        r = self.rank if rank is None else rank
        return n * r // self.world, n * (r + 1) // self.world

    def allreduce_min_(self, t) -> None:
        vals = self.g.exchange(self.rank, t.clone())
        t.copy_(torch.stack(vals).min(dim=0).values)

    def allreduce_sum_(self, t) -> None:
        vals = self.g.exchange(self.rank, t.clone())
        t.copy_(torch.stack(vals).sum(dim=0))

    def allgather_rows(self, local, n: int):
        return torch.cat(self.g.exchange(self.rank, local.clone()))

    def alltoall_rows(self, t, n: int):
        lo, hi = self.rows(n)
        parts = self.g.exchange(self.rank, t)
        out = torch.stack([p[lo:hi] for p in parts]).contiguous()
        self.g.exchange(self.rank, None)   # senders keep their buffers until all have read
        return out

    def alltoall_chunks(self, t):
        parts = self.g.exchange(self.rank, t)
        out = torch.stack([p[self.rank] for p in parts]).contiguous()
        self.g.exchange(self.rank, None)
        return out

    def alltoall_var(self, t, send_counts, recv_counts):
        parts = self.g.exchange(self.rank, (t, list(send_counts)))
        segs = []
        for buf, cnts in parts:
            off = sum(cnts[: self.rank])
            segs.append(buf[off: off + cnts[self.rank]])
        out = torch.cat(segs).contiguous()
        self.g.exchange(self.rank, None)
        return out

    def allgather_stack(self, stack):
        return torch.stack(self.g.exchange(self.rank, stack.clone()))
