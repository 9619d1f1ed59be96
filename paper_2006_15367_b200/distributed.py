"""Multi-GPU evaluation: one process per GPU, torch.distributed for the plumbing.

Decomposition, following the reference's distributed
algorithm (arXiv 2006.15367; traversal.cpp:322-707):

* leaves are split along the Morton curve exactly as ``partition_leaves``
  (tree.cpp:19-75); rank r holds every node whose leaf range meets its own;
* the upward pass (C2M, M2M) runs on held nodes and yields PARTIAL
  multipoles -- M2M is linear, so a plural node's partials sum to its full
  multipole;
* plural (shared) nodes are SLICED across their users by theta rows
  (``assign_sample_slices``, tree.cpp:180-239): a reduce-scatter (kind 2)
  leaves every user the full multipole on its own slice;
* M2L runs per observer slice; the missing source rows arrive through the
  reference's M2L CommPlan (kind 0, comm_plan.cpp:31-82), sent in
  ``buffer_limit``-byte chunks (M_S, traversal.cpp:449-470) and level by
  level, so the transfer of level l+1 overlaps the translations of level l;
* before the L2L from level l, the users of each plural node gather its
  local slices (kind 3) -- the role of the reference's parallel
  anterpolation (parallel_interp.cpp:151-226, traversal.cpp:596-707);
* ghost particles of neighbouring ranks (kind 1) feed the near field (the
  reference's near plan, comm_plan.cpp:84-109).

Buffers move with ``torch.distributed`` point-to-point operations (NCCL over
NVLink on B200; gloo in the CPU tests).  The engine is pluggable:
:class:`paper_2006_15367_b200.RankEngine` on a GPU, or a CPU restatement in
the tests.  :func:`run_emulated` drives several engines in one process through
the same schedule with in-process copies (one GPU standing in for P).
"""
from __future__ import annotations

from .hfmm import Phase

KIND_HALO = 0     # M2L halo: reference CommPlan rows, overwrite
KIND_GHOST = 1    # ghost particles
KIND_REDUCE = 2   # plural multipole reduce-scatter, add (ascending peer order)
KIND_GATHER = 3   # plural local all-gather, overwrite
KIND_MULTIPOLE = KIND_HALO  # (name kept for callers of the previous scheme)


def schedule(top: int, levels: int):
    """The per-evaluation stage list shared by every driver: ("x", kind, level)
    exchanges and ("run", phase, level) compute steps (level -1 = all)."""
    st = [("x", KIND_GHOST, -1), ("run", Phase.NearStart, -1), ("run", Phase.C2M, -1),
          ("run", Phase.M2M, -1), ("x", KIND_REDUCE, -1), ("run", Phase.TBuild, -1)]
    for lvl in range(top, levels + 1):
        st += [("x", KIND_HALO, lvl), ("run", Phase.M2L, lvl)]
    for lvl in range(top, levels):
        st += [("x", KIND_GATHER, lvl), ("run", Phase.L2L, lvl)]
    st += [("run", Phase.L2T, -1), ("run", Phase.Near, -1)]
    return st


def _run(eng, phase, level):
    if level < 0:
        eng.run_phase(phase)
    else:
        eng.run_level(phase, level)


def _chunks(n_doubles: int, buffer_limit: int | None):
    """[begin, end) double ranges of one message stream cut into buffer_limit
    byte chunks (PairPlan::num_chunks, comm_plan.cpp:19-23)."""
    if n_doubles == 0:
        return []
    step = n_doubles if not buffer_limit or buffer_limit >= 8 * n_doubles else max(1, buffer_limit // 8)
    return [(b, min(n_doubles, b + step)) for b in range(0, n_doubles, step)]


class DistributedEvaluator:
    """Drives one rank's engine through an evaluation over torch.distributed."""

    def __init__(self, engine, rank: int, world: int, device, group=None, buffer_limit: int | None = None,
                 top: int | None = None, levels: int | None = None):
        import torch
        self.torch = torch
        self.eng = engine
        self.rank = rank
        self.world = world
        self.device = device
        self.group = group
        setup = getattr(engine, "setup", None) or getattr(engine, "s", None)
        self.top = top if top is not None else setup.top_level
        self.levels = levels if levels is not None else setup.levels
        if buffer_limit is None and setup is not None and hasattr(setup, "config"):
            buffer_limit = int(setup.config.buffer_limit)
        self.buffer_limit = buffer_limit if buffer_limit and buffer_limit < 2**63 else None
        self.peers = [q for q in range(world) if q != rank]
        self.send, self.recv, self.off = {}, {}, {}
        for kind in (KIND_HALO, KIND_GHOST, KIND_REDUCE, KIND_GATHER):
            for q in self.peers:
                s, r = engine.exchange_sizes(kind, q)
                self.send[kind, q] = torch.empty(int(s), dtype=torch.float64, device=device)
                self.recv[kind, q] = torch.empty(int(r), dtype=torch.float64, device=device)
                if kind in (KIND_HALO, KIND_GATHER):  # level-major offsets
                    so = ro = 0
                    for lvl in range(self.top, self.levels + 1):
                        sl, rl = engine.exchange_sizes(kind, q, lvl)
                        self.off[kind, q, lvl] = (so, so + int(sl), ro, ro + int(rl))
                        so += int(sl)
                        ro += int(rl)
        self._halo_works = {}

    def exchange_bytes(self, kind: int) -> int:
        return 8 * sum(int(self.send[kind, q].numel()) for q in self.peers)

    def _post(self, pairs):
        """pairs: [(peer, send view, recv view)] -> started works (chunked)."""
        dist = self.torch.distributed
        ops = []
        for q, sv, rv in pairs:
            for b, e in _chunks(int(sv.numel()), self.buffer_limit):
                ops.append(dist.P2POp(dist.isend, sv[b:e], q, group=self.group))
            for b, e in _chunks(int(rv.numel()), self.buffer_limit):
                ops.append(dist.P2POp(dist.irecv, rv[b:e], q, group=self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def _views(self, kind, q, level):
        if level < 0 or kind in (KIND_GHOST, KIND_REDUCE):
            return self.send[kind, q], self.recv[kind, q]
        sb, se, rb, re_ = self.off[kind, q, level]
        return self.send[kind, q][sb:se], self.recv[kind, q][rb:re_]

    def exchange(self, kind: int, level: int = -1) -> None:
        if self.world == 1:
            return
        if kind == KIND_HALO:
            self._halo(level)
            return
        for q in self.peers:
            sv, _ = self._views(kind, q, level)
            if sv.numel():
                self.eng.pack(kind, q, sv, level)
        works = self._post([(q, *self._views(kind, q, level)) for q in self.peers])
        for w in works:
            w.wait()
        for q in self.peers:  # ascending peer rank: deterministic sums (kind 2)
            _, rv = self._views(kind, q, level)
            if rv.numel():
                self.eng.unpack(kind, q, rv, level)

    def _halo(self, level: int) -> None:
        """M2L halo: at the first level, pack every level and post one batch per
        level; each level then waits only for its own batch, so later levels
        stay in flight while this level's translations run."""
        if level == self.top or not self._halo_works:
            for q in self.peers:
                if self.send[KIND_HALO, q].numel():
                    self.eng.pack(KIND_HALO, q, self.send[KIND_HALO, q], -1)
            self._halo_works = {lvl: self._post([(q, *self._views(KIND_HALO, q, lvl)) for q in self.peers])
                                for lvl in range(self.top, self.levels + 1)}
        for w in self._halo_works.pop(level, []):
            w.wait()
        for q in self.peers:
            _, rv = self._views(KIND_HALO, q, level)
            if rv.numel():
                self.eng.unpack(KIND_HALO, q, rv, level)

    def step(self, mark=None) -> None:
        """One evaluation from the charges already loaded into the engine.

        `mark(name)` (optional) is called after every stage, e.g. to record
        CUDA events for per-phase device timing."""
        mark = mark or (lambda name: None)
        for what, a, lvl in schedule(self.top, self.levels):
            if what == "x":
                self.exchange(a, lvl)
                mark(f"x{a}" if lvl < 0 else f"x{a}.L{lvl}")
            else:
                _run(self.eng, a, lvl)
                mark(Phase(a).name if lvl < 0 else f"{Phase(a).name}.L{lvl}")


def run_emulated(engines, alloc, mark=None) -> None:
    """All P ranks' engines in one process (one GPU standing in for P): the
    same schedule, each exchange done by packing every rank's send buffers and
    unpacking them on the receivers in ascending sender order.  No kernel ever
    waits on another rank.  `alloc(n)` returns a float64 buffer of n doubles
    on the engines' device."""
    P = len(engines)
    e0 = engines[0]
    setup = e0.setup
    for what, a, lvl in schedule(setup.top_level, setup.levels):
        if what == "run":
            for e in engines:
                _run(e, a, lvl)
        else:
            bufs = {}
            for r, e in enumerate(engines):
                for q in range(P):
                    if q == r:
                        continue
                    s, _ = e.exchange_sizes(a, q, lvl)
                    if s:
                        bufs[r, q] = alloc(s)
                        e.pack(a, q, bufs[r, q], lvl)
                e.synchronize()
            for q, e in enumerate(engines):
                for r in range(P):
                    if (r, q) in bufs:
                        assert e.exchange_sizes(a, r, lvl)[1] == bufs[r, q].numel()
                        e.unpack(a, r, bufs[r, q], lvl)
                e.synchronize()
        if mark:
            mark(what, a, lvl)


def gpu_rank_engine(setup, rank: int, device: int):
    """A :class:`RankEngine` bound to torch's current stream on `device`."""
    import torch
    from .hfmm import RankEngine
    eng = RankEngine(setup, rank, device)
    eng.set_stream(torch.cuda.current_stream(device).cuda_stream)
    return eng
