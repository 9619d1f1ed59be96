"""Host-side mirror of the reference's evaluation API, backed by the B200 engine.

Names, argument meaning and error behaviour follow the reference C++ API:

* :class:`RunConfig`      -- hfmm::RunConfig   (traversal.hpp:21-38)
* :func:`build_setup`     -- hfmm::build_setup (traversal.hpp:120, traversal.cpp:66-238)
* :class:`RankEngine`     -- hfmm::RankEngine phase drivers (traversal.hpp:125-156)
* :func:`evaluate_with_setup` / :func:`evaluate_potential`
                          -- traversal.hpp:163-166, traversal.cpp:790-823
* :func:`direct_potential` -- kernel.hpp:15-20 (device O(N M) sum)

Particles are given as ``positions`` (N, 3) float64 and ``intensities`` (N,)
complex128 (or (N, 2) float64), in input order.  Potentials come back as
complex128 in input order, like ``EvalResult::potentials``.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import check, lib, ptr


class AlignPolicy(enum.IntEnum):
    RankOrdered = 0
    Aligned = 1


class SchedulerKind(enum.IntEnum):
    Deterministic = 0
    Adversarial = 1
    Threaded = 2


class Phase(enum.IntEnum):
    C2M = 1
    M2M = 2
    M2L = 3
    L2L = 4
    L2T = 5
    Near = 6
    NearStart = 7
    TBuild = 8


@dataclass
class RunConfig:
    lambda_: float = 1.0
    digits: float = 3.0
    leaf_lambda: float = 0.25
    num_ranks: int = 1
    buffer_limit: int = 2**64 - 1
    policy: AlignPolicy = AlignPolicy.Aligned
    one_particle_per_leaf: bool = False
    seed: int = 0
    scheduler: SchedulerKind = SchedulerKind.Deterministic
    top_level: int = 3
    d_override: int = 0
    # Morton-partition leaf weights: 0 = particles (the reference's rule,
    # bit-exact setup), 1 = near-field pairs per leaf (opt-in P2P load balance)
    partition_weight: int = 0
    # 1 = Morton keys / sort and the far / near lists built on the device
    # (bit-exact with the host build)
    setup_device: int = 0

    def validate(self) -> None:
        """RunConfig::validate (traversal.cpp:42-46)."""
        if (not self.lambda_ > 0 or not self.digits > 0 or not self.leaf_lambda > 0
                or self.num_ranks < 1 or self.buffer_limit == 0 or self.top_level < 1):
            raise _native.InvalidArgument("RunConfig: invalid fields")

    def to_c(self) -> _native.RunConfigC:
        return _native.RunConfigC(
            float(self.lambda_), float(self.digits), float(self.leaf_lambda), int(self.num_ranks),
            int(self.policy), int(self.buffer_limit), int(bool(self.one_particle_per_leaf)),
            int(self.top_level), int(self.d_override), int(self.scheduler), int(self.seed),
            int(self.partition_weight), int(self.setup_device))


def _as_particles(positions, intensities):
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    if pos.ndim != 2 or pos.shape[1] != 3:
        raise _native.InvalidArgument("positions must have shape (N, 3)")
    q = np.asarray(intensities)
    if np.iscomplexobj(q):
        q = np.ascontiguousarray(np.stack([q.real, q.imag], axis=-1), dtype=np.float64)
    else:
        q = np.ascontiguousarray(q, dtype=np.float64)
    if q.shape != (pos.shape[0], 2):
        raise _native.InvalidArgument("intensities must have shape (N,) complex or (N, 2)")
    return pos, q


class GlobalSetup:
    """Host setup built by the native library; read-only during evaluation."""

    def __init__(self, handle: ctypes.c_void_p, config: RunConfig, n: int):
        self._h = handle
        self.config = config
        self.n = n
        meta = self.array("meta_i64", np.int64)
        self.levels, self.top_level, self.d_class = int(meta[0]), int(meta[1]), int(meta[2])
        self.num_leaves, self.num_ranks = int(meta[4]), int(meta[5])
        f = self.array("meta_f64", np.float64)
        self.root_side, self.leaf_side = float(f[0]), float(f[1])
        self.root_corner = f[2:5].copy()
        self.k = float(f[5])

    def array(self, name: str, dtype=np.uint8) -> np.ndarray:
        """Named flat view ('setup arrays')."""
        nb = ctypes.c_size_t(0)
        check(lib().hfmm_setup_get(self._h, name.encode(), None, 0, ctypes.byref(nb)))
        out = np.empty(nb.value, dtype=np.uint8)
        if nb.value:
            check(lib().hfmm_setup_get(self._h, name.encode(), ptr(out), nb.value, ctypes.byref(nb)))
        return out.view(dtype)

    def sampling(self, level: int):
        tr, nt, nphi = self.array(f"L{level}.sampling", np.int64)
        return int(tr), int(nt), int(nphi)

    def num_nodes(self, level: int) -> int:
        return int(self.array(f"L{level}.codes", np.uint64).size)

    @property
    def original_index(self) -> np.ndarray:
        return self.array("original_index", np.uint64).astype(np.int64)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _native._lib is not None:
            _native._lib.hfmm_setup_destroy(h)


def build_setup(positions, intensities, config: RunConfig | None = None) -> GlobalSetup:
    """hfmm::build_setup: Morton sort, tree, partition, slices, lists, plans (bit-exact)."""
    config = config or RunConfig()
    pos, q = _as_particles(positions, intensities)
    h = ctypes.c_void_p()
    c = config.to_c()
    check(lib().hfmm_setup_build(ptr(pos), ptr(q), pos.shape[0], ctypes.byref(c), ctypes.byref(h)))
    return GlobalSetup(h, config, pos.shape[0])


@dataclass
class EvalResult:
    potentials: np.ndarray  # complex128, input order
    phase_ms: dict = field(default_factory=dict)
    kernel_launches: int = 0


_PHASE_NAMES = ("Tbuild", "C2M", "M2M", "M2L", "L2L", "L2T", "Near", "total")


class RankEngine:
    """Device engine for one logical rank (hfmm::RankEngine on a B200)."""

    def __init__(self, setup: GlobalSetup, rank: int = 0, device: int = 0):
        self.setup = setup  # keeps the host setup alive for the engine's lifetime
        self.rank = rank
        self.device = device
        h = ctypes.c_void_p()
        check(lib().hfmm_gpu_create(setup._h, device, rank, ctypes.byref(h)))
        self._h = h

    # phase drivers (traversal.hpp:129-140)
    def set_intensities(self, intensities) -> None:
        _, q = _as_particles(np.zeros((self.setup.n, 3)), intensities)
        check(lib().hfmm_gpu_set_charges(self._h, ptr(q)))

    def c2m_phase(self):
        check(lib().hfmm_gpu_run_phase(self._h, Phase.C2M))

    def m2m_pass(self):
        check(lib().hfmm_gpu_run_phase(self._h, Phase.M2M))

    def m2l_pass(self):
        check(lib().hfmm_gpu_run_phase(self._h, Phase.M2L))

    def l2l_pass(self):
        check(lib().hfmm_gpu_run_phase(self._h, Phase.L2L))

    def l2o_near_phase(self) -> np.ndarray:
        """L2T + near field; returns sorted-order potentials (all particles)."""
        check(lib().hfmm_gpu_run_phase(self._h, Phase.L2T))
        check(lib().hfmm_gpu_run_phase(self._h, Phase.Near))
        return self.potentials_sorted()

    def potentials_sorted(self) -> np.ndarray:
        out = np.empty((self.setup.n, 2))
        check(lib().hfmm_gpu_get_potentials_sorted(self._h, ptr(out), out.size))
        return out[:, 0] + 1j * out[:, 1]

    def _expansion(self, kind: int, level: int) -> np.ndarray:
        _, nt, nphi = self.setup.sampling(level)
        nn = self.setup.num_nodes(level)
        out = np.empty((nn, nt * nphi, 2))
        check(lib().hfmm_gpu_get_expansion(self._h, kind, level, ptr(out), out.size))
        return out[..., 0] + 1j * out[..., 1]

    def multipole(self, level: int) -> np.ndarray:
        """(n_nodes, S) multipole samples of a level (RankEngine::multipole)."""
        return self._expansion(0, level)

    def local_expansion(self, level: int) -> np.ndarray:
        """(n_nodes, S) local samples of a level (RankEngine::local_expansion)."""
        return self._expansion(1, level)

    def evaluate(self, intensities=None) -> EvalResult:
        """All phases; host intensities in, host potentials (input order) out."""
        q = None
        if intensities is not None:
            _, q = _as_particles(np.zeros((self.setup.n, 3)), intensities)
        out = np.zeros((self.setup.n, 2))
        t = _native.TimingC()
        check(lib().hfmm_gpu_evaluate(self._h, ptr(q), ptr(out), ctypes.byref(t)))
        return EvalResult(out[:, 0] + 1j * out[:, 1],
                          {k: float(v) for k, v in zip(_PHASE_NAMES, t.ms)}, int(t.kernel_launches))

    def evaluate_device(self, d_q_sorted_ptr: int, d_pot_sorted_ptr: int, stream_ptr: int = 0):
        """Device-resident evaluation (raw device pointers, sorted order)."""
        check(lib().hfmm_gpu_evaluate_device(self._h, ctypes.c_void_p(d_q_sorted_ptr),
                                             ctypes.c_void_p(d_pot_sorted_ptr),
                                             ctypes.c_void_p(stream_ptr)))

    # distributed mode (paper_2006_15367_b200.distributed)
    def run_phase(self, phase: int) -> None:
        check(lib().hfmm_gpu_run_phase(self._h, int(phase)))

    def run_level(self, phase: int, level: int) -> None:
        """One level of M2L (observer level) or L2L (parent level)."""
        check(lib().hfmm_gpu_run_level(self._h, int(phase), int(level)))

    def exchange_sizes(self, kind: int, peer: int, level: int = -1) -> tuple[int, int]:
        """(send, recv) doubles of exchange `kind` with `peer` (level -1: all levels)."""
        s = ctypes.c_int64()
        r = ctypes.c_int64()
        check(lib().hfmm_gpu_exchange_sizes(self._h, kind, peer, level, ctypes.byref(s), ctypes.byref(r)))
        return s.value, r.value

    def pack(self, kind: int, peer: int, buf, level: int = -1) -> None:
        """Packs this rank's outgoing data for `peer` into a device tensor (float64)."""
        check(lib().hfmm_gpu_pack(self._h, kind, peer, level, ctypes.c_void_p(buf.data_ptr())))

    def unpack(self, kind: int, peer: int, buf, level: int = -1) -> None:
        check(lib().hfmm_gpu_unpack(self._h, kind, peer, level, ctypes.c_void_p(buf.data_ptr())))

    def set_stream(self, stream_ptr: int) -> None:
        check(lib().hfmm_gpu_set_stream(self._h, ctypes.c_void_p(stream_ptr)))

    def synchronize(self) -> None:
        check(lib().hfmm_gpu_synchronize(self._h))

    def load_charges_device(self, d_q_sorted_ptr: int) -> None:
        check(lib().hfmm_gpu_load_charges_device(self._h, ctypes.c_void_p(d_q_sorted_ptr)))

    def store_potentials_device(self, d_pot_sorted_ptr: int) -> None:
        """Async device copy of this rank's potentials (sorted, own range)."""
        check(lib().hfmm_gpu_store_potentials_device(self._h, ctypes.c_void_p(d_pot_sorted_ptr)))

    def set_overlap(self, on: bool) -> None:
        """Phase overlap in evaluate (default on); off = sequential phases whose
        last_timing() entries are each phase's own kernel time."""
        check(lib().hfmm_gpu_set_overlap(self._h, 1 if on else 0))

    def launch_count(self) -> int:
        """Kernels launched by this engine so far (cumulative)."""
        n = ctypes.c_int64()
        check(lib().hfmm_gpu_launch_count(self._h, ctypes.byref(n)))
        return n.value

    def particle_range(self) -> tuple[int, int]:
        b = ctypes.c_int64()
        e = ctypes.c_int64()
        check(lib().hfmm_gpu_particle_range(self._h, ctypes.byref(b), ctypes.byref(e)))
        return b.value, e.value

    def last_timing(self) -> tuple[dict, int]:
        """Per-phase device ms and kernel launches of the last evaluation."""
        t = _native.TimingC()
        check(lib().hfmm_gpu_last_timing(self._h, ctypes.byref(t)))
        return {k: float(v) for k, v in zip(_PHASE_NAMES, t.ms)}, int(t.kernel_launches)

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _native._lib is not None:
            _native._lib.hfmm_gpu_destroy(h)

    def __del__(self):
        self.close()


LEDGER_PHASES = ("Setup", "C2M", "M2M", "M2L", "L2L", "L2O", "Near")  # ledger.hpp


class World:
    """Every logical rank of the setup's partition in this process (the
    reference's run_world + evaluate_with_setup, runtime.cpp:274-290,
    traversal.cpp:790-817): rank r on devices[r % len(devices)], exchanges by
    device (peer) copies inside the native library."""

    def __init__(self, setup: GlobalSetup, devices=(0,)):
        self.setup = setup  # keeps the host setup alive
        devs = (ctypes.c_int * len(devices))(*devices)
        h = ctypes.c_void_p()
        check(lib().hfmm_world_create(setup._h, devs, len(devices), ctypes.byref(h)))
        self._h = h

    def set_intensities(self, intensities) -> None:
        _, q = _as_particles(np.zeros((self.setup.n, 3)), intensities)
        check(lib().hfmm_world_set_charges(self._h, ptr(q)))

    def run_phase(self, phase: int) -> None:
        """One reference RankEngine phase on every rank (C2M, M2M, M2L, L2L,
        L2T = l2o_near_phase), with the exchanges it owns."""
        check(lib().hfmm_world_run_phase(self._h, int(phase)))

    def evaluate(self, intensities=None) -> EvalResult:
        q = None
        if intensities is not None:
            _, q = _as_particles(np.zeros((self.setup.n, 3)), intensities)
        out = np.zeros((self.setup.n, 2))
        ms = np.zeros((self.setup.num_ranks, len(LEDGER_PHASES)))
        check(lib().hfmm_world_evaluate(self._h, ptr(q), ptr(out), ptr(ms)))
        res = EvalResult(out[:, 0] + 1j * out[:, 1],
                         {k: float(v) for k, v in zip(LEDGER_PHASES, ms.max(axis=0))})
        res.rank_ms = ms
        return res

    def potentials(self) -> np.ndarray:
        out = np.zeros((self.setup.n, 2))
        check(lib().hfmm_world_potentials(self._h, ptr(out)))
        return out[:, 0] + 1j * out[:, 1]

    def expansion(self, rank: int, kind: int, level: int) -> np.ndarray:
        """(n_nodes, S) expansions as held by `rank` (its slice rows valid)."""
        _, nt, nphi = self.setup.sampling(level)
        out = np.empty((self.setup.num_nodes(level), nt * nphi, 2))
        check(lib().hfmm_world_get_expansion(self._h, rank, kind, level, ptr(out), out.size))
        return out[..., 0] + 1j * out[..., 1]

    def assembled(self, kind: int, level: int) -> np.ndarray:
        """Every node's expansion assembled from its users' slices, as the
        reference's RankEngine::multipole / local_expansion expose them."""
        so = self.setup.array(f"L{level}.slices_off", np.uint64).astype(np.int64)
        sl = self.setup.array(f"L{level}.slices", np.int64).reshape(-1, 3)
        per = [self.expansion(r, kind, level) for r in range(self.setup.num_ranks)]
        out = np.zeros_like(per[0])
        for n in range(out.shape[0]):
            for z in range(so[n], so[n + 1]):
                r, b, e = (int(v) for v in sl[z])
                out[n, b:e] = per[r][n, b:e]
        return out

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _native._lib is not None:
            _native._lib.hfmm_world_destroy(h)

    def __del__(self):
        self.close()


def evaluate_with_setup(setup: GlobalSetup, device: int = 0, devices=None) -> EvalResult:
    """hfmm::evaluate_with_setup (traversal.cpp:790-817).  One logical rank
    runs as a single engine on `device`; num_ranks > 1 runs every rank in this
    process (:class:`World`, ranks round-robin over `devices`, default
    [device]) -- the reference's own in-process simulation of its ranks.  The
    one-process-per-GPU NCCL runner is :mod:`paper_2006_15367_b200.distributed`."""
    if setup.num_ranks == 1:
        eng = RankEngine(setup, 0, device)
        try:
            return eng.evaluate()
        finally:
            eng.close()
    w = World(setup, list(devices) if devices else [device])
    try:
        return w.evaluate()
    finally:
        w.close()


def evaluate_potential(positions, intensities, config: RunConfig | None = None,
                       device: int = 0) -> EvalResult:
    """hfmm::evaluate_potential: build_setup + evaluate_with_setup."""
    return evaluate_with_setup(build_setup(positions, intensities, config), device)


def direct_potential(positions, intensities, observer_index, lam: float = 1.0,
                     device: int = 0) -> np.ndarray:
    """Device O(N M) direct sum for observers given as particle indices
    (hfmm::direct_potential, kernel.cpp:16-41, self term skipped)."""
    pos, q = _as_particles(positions, intensities)
    obs = np.ascontiguousarray(observer_index, dtype=np.int64)
    out = np.empty((obs.size, 2))
    k = 2.0 * np.pi / lam
    check(lib().hfmm_gpu_direct(ptr(pos), ptr(q), pos.shape[0], ptr(obs), obs.size, k, device,
                                ptr(out)))
    return out[:, 0] + 1j * out[:, 1]


def generate_inputs(shape: str, n: int, extent: float, seed: int):
    """Frozen seeded generator; shape 'cube' (side) or 'sphere' (radius)."""
    pos = np.empty((n, 3))
    q = np.empty((n, 2))
    lib().hfmm_generate_inputs(0 if shape == "cube" else 1, n, float(extent), int(seed), ptr(pos), ptr(q))
    return pos, q[:, 0] + 1j * q[:, 1]


def resample_matrix(n_in: int, s_in: float, n_out: int, s_out: float) -> np.ndarray:
    """Dense (n_out, n_in) complex matrix of resample_circle (sphere_grid.cpp:128-155)
    as applied by the device M2M/L2L kernels."""
    out = np.empty((n_out, n_in, 2))
    check(lib().hfmm_resample_matrix(int(n_in), float(s_in), int(n_out), float(s_out), ptr(out)))
    return out[..., 0] + 1j * out[..., 1]


def m2m_operands(nc: int, npar: int):
    """Packed operands of the device M2M passes of a level pair (host logic, csrc/interp.hpp):
    (bphi (Kp, Np), vphi (nc,), bth (2 KH, NH), vth (2 KH,), KH)."""
    import ctypes
    dims = (ctypes.c_int * 4)()
    check(lib().hfmm_m2m_operands(int(nc), int(npar), None, None, None, None, dims))
    kp, n_p, kh, nh = list(dims)
    bphi, vphi = np.empty((kp, n_p)), np.empty(nc)
    bth, vth = np.empty((2 * kh, nh)), np.empty(2 * kh)
    check(lib().hfmm_m2m_operands(int(nc), int(npar), ptr(bphi), ptr(vphi), ptr(bth), ptr(vth), dims))
    return bphi, vphi, bth, vth, kh


def l2l_operands(nc: int, npar: int, row_scale: np.ndarray, col_scale: np.ndarray):
    """Packed operands of the device L2L passes: (bth (2 KH, NH), vth (2 KH,), bphi (Kp, Np), vphi (np,), KH)."""
    import ctypes
    rs = np.ascontiguousarray(row_scale, dtype=np.float64)
    cs = np.ascontiguousarray(col_scale, dtype=np.float64)
    if rs.size != 2 * nc or cs.size != 2 * npar:
        raise _native.InvalidArgument("l2l_operands: row_scale has 2 nc entries, col_scale 2 np")
    dims = (ctypes.c_int * 4)()
    check(lib().hfmm_l2l_operands(int(nc), int(npar), ptr(rs), ptr(cs), None, None, None, None, dims))
    kh, nh, kp, n_p = list(dims)
    bth, vth = np.empty((2 * kh, nh)), np.empty(2 * kh)
    bphi, vphi = np.empty((kp, n_p)), np.empty(npar)
    check(lib().hfmm_l2l_operands(int(nc), int(npar), ptr(rs), ptr(cs), ptr(bth), ptr(vth), ptr(bphi), ptr(vphi), dims))
    return bth, vth, bphi, vphi, kh
