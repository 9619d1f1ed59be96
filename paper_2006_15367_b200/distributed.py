"""Multi-GPU evaluation: one process per GPU, torch.distributed for the plumbing.

Decomposition: leaves are split along the Morton curve
exactly as the reference's ``partition_leaves`` (tree.cpp:19-75).  Rank r holds
every node whose leaf range meets its own; the upward pass (C2M, M2M) runs on
held nodes and yields PARTIAL multipoles -- M2M is linear, so the partials of
a plural node sum to its full multipole and no data moves on the way up.  Two
static exchanges then suffice:

* kind 1, ghosts: the particles of neighbouring ranks' leaves that this rank's
  near lists touch (the reference's near plan, comm_plan.cpp:84-109);
* kind 0, multipoles: for every far source a held observer needs, the partials
  of the source's other users, added in rank order (this replaces the
  reference's sliced aggregation, parallel interpolation and M2L halo,
  traversal.cpp:350-426, parallel_interp.cpp:151-226, comm_plan.cpp:31-82).

The downward pass (M2L, L2L, L2T, P2P) is then rank-local.  Buffers move with
``torch.distributed.batch_isend_irecv`` (NCCL over NVLink on B200; gloo in the
CPU tests).  The engine is pluggable: :class:`paper_2006_15367_b200.RankEngine`
on a GPU, or a CPU restatement in the tests.
"""
from __future__ import annotations

import time

import numpy as np

from .hfmm import Phase

KIND_MULTIPOLE = 0
KIND_GHOST = 1


class DistributedEvaluator:
    """Drives one rank's engine through an evaluation with the two exchanges."""

    def __init__(self, engine, rank: int, world: int, device, group=None):
        import torch
        self.torch = torch
        self.eng = engine
        self.rank = rank
        self.world = world
        self.device = device
        self.group = group
        self.send = {}
        self.recv = {}
        for kind in (KIND_MULTIPOLE, KIND_GHOST):
            for q in range(world):
                if q == rank:
                    continue
                s, r = engine.exchange_sizes(kind, q)
                self.send[kind, q] = torch.empty(int(s), dtype=torch.float64, device=device)
                self.recv[kind, q] = torch.empty(int(r), dtype=torch.float64, device=device)

    def exchange_bytes(self, kind: int) -> int:
        return 8 * sum(int(self.send[kind, q].numel()) for q in range(self.world) if q != self.rank)

    def exchange(self, kind: int) -> None:
        if self.world == 1:  # nothing to exchange (single-rank engines have no plan)
            return
        dist = self.torch.distributed
        if kind == KIND_MULTIPOLE:
            self.eng.exchange_begin(kind)
        ops = []
        for q in range(self.world):
            if q == self.rank:
                continue
            if self.send[kind, q].numel():
                self.eng.pack(kind, q, self.send[kind, q])
        for q in range(self.world):
            if q == self.rank:
                continue
            if self.send[kind, q].numel():
                ops.append(dist.P2POp(dist.isend, self.send[kind, q], q, group=self.group))
            if self.recv[kind, q].numel():
                ops.append(dist.P2POp(dist.irecv, self.recv[kind, q], q, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for q in range(self.world):  # fixed (rank) order: deterministic sums
            if q != self.rank and self.recv[kind, q].numel():
                self.eng.unpack(kind, q, self.recv[kind, q])

    def step(self, mark=None) -> None:
        """One evaluation from the charges already loaded into the engine.

        `mark(name)` (optional) is called after every stage, e.g. to record
        CUDA events for per-phase device timing."""
        mark = mark or (lambda name: None)
        self.exchange(KIND_GHOST)
        mark("ghosts")
        self.eng.run_phase(Phase.NearStart)  # near field overlaps the far-field chain
        self.eng.run_phase(Phase.C2M)
        mark("C2M")
        self.eng.run_phase(Phase.M2M)
        mark("M2M")
        self.exchange(KIND_MULTIPOLE)
        mark("multipoles")
        self.eng.run_phase(Phase.M2L)
        mark("M2L")
        self.eng.run_phase(Phase.L2L)
        mark("L2L")
        self.eng.run_phase(Phase.L2T)
        mark("L2T")
        self.eng.run_phase(Phase.Near)
        mark("Near")


def gpu_rank_engine(setup, rank: int, device: int):
    """A :class:`RankEngine` bound to torch's current stream on `device`."""
    import torch
    from .hfmm import RankEngine
    eng = RankEngine(setup, rank, device)
    eng.set_stream(torch.cuda.current_stream(device).cuda_stream)
    return eng
