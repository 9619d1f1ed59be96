"""ctypes wrapper of oracle/_ref/libhfmm_ref.so (the UNMODIFIED reference).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's reference / cpu_baseline legs, as the checker or the timed CPU
baseline.  Never imported by the product package.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libhfmm_ref.so")

_lib = None
_P = ctypes.c_void_p


class RefCfg(ctypes.Structure):
    _fields_ = [
        ("lambda_", ctypes.c_double), ("digits", ctypes.c_double), ("leaf_lambda", ctypes.c_double),
        ("num_ranks", ctypes.c_int32), ("policy", ctypes.c_int32), ("buffer_limit", ctypes.c_uint64),
        ("one_particle_per_leaf", ctypes.c_int32), ("top_level", ctypes.c_int32),
        ("d_override", ctypes.c_int32), ("scheduler", ctypes.c_int32), ("seed", ctypes.c_uint64),
    ]


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"reference oracle {LIB_PATH} not built (make -C oracle)")
        h = ctypes.CDLL(LIB_PATH)
        h.ref_last_error.restype = ctypes.c_char_p
        _lib = h
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class RefError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[{status}] {msg}")
        self.status = status


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def config(lambda_=1.0, digits=3.0, leaf_lambda=0.25, num_ranks=1, policy=1,
           buffer_limit=2**64 - 1, one_particle_per_leaf=0, top_level=3, d_override=0,
           scheduler=0, seed=0) -> RefCfg:
    return RefCfg(lambda_, digits, leaf_lambda, num_ranks, policy, buffer_limit,
                  one_particle_per_leaf, top_level, d_override, scheduler, seed)


def generate_inputs(shape: str, n: int, extent: float, seed: int):
    pos = np.empty((n, 3))
    q = np.empty((n, 2))
    lib().ref_generate_inputs(0 if shape == "cube" else 1, ctypes.c_size_t(n), ctypes.c_double(extent),
                              ctypes.c_uint64(seed), _p(pos), _p(q))
    return pos, q


def generate_geometry(kind: str, extent: float, spacing: float, lam: float = 1.0,
                      random: bool = True, seed: int = 0):
    """hfmm::generate_geometry (geometry.cpp:75-127): 'grid', 'sphere' or 'volume'."""
    k = {"grid": 0, "sphere": 1, "volume": 2}[kind]
    cnt = ctypes.c_size_t()
    _check(lib().ref_generate_geometry(ctypes.c_int(k), ctypes.c_double(extent), ctypes.c_double(spacing),
                                       ctypes.c_double(lam), ctypes.c_int(int(random)), ctypes.c_uint64(seed),
                                       ctypes.c_size_t(0), None, None, ctypes.byref(cnt)))
    n = cnt.value
    pos = np.empty((n, 3))
    q = np.empty((n, 2))
    _check(lib().ref_generate_geometry(ctypes.c_int(k), ctypes.c_double(extent), ctypes.c_double(spacing),
                                       ctypes.c_double(lam), ctypes.c_int(int(random)), ctypes.c_uint64(seed),
                                       ctypes.c_size_t(n), _p(pos), _p(q), ctypes.byref(cnt)))
    return pos, q


_IO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "particles_io")


def read_particles(path: str):
    """hfmm::read_particles (geometry.cpp:128-148) -> (positions (n, 3), charges (n, 2)).
    Runs out of process (oracle/particles_io.cpp); parse errors raise RefError."""
    import subprocess
    import tempfile
    with tempfile.NamedTemporaryFile(suffix=".bin") as tmp:
        r = subprocess.run([_IO, "read", path, tmp.name], capture_output=True, text=True)
        if r.returncode != 0:
            raise RefError(r.returncode, r.stderr.strip())
        raw = open(tmp.name, "rb").read()
    n = int(np.frombuffer(raw[:8], np.uint64)[0])
    v = np.frombuffer(raw[8:], np.float64)
    return v[:3 * n].reshape(n, 3).copy(), v[3 * n:5 * n].reshape(n, 2).copy()


def write_particles(path: str, pos, q, header: str = "") -> None:
    """hfmm::write_particles (geometry.cpp:150-159), out of process."""
    import subprocess
    import tempfile
    pos = np.ascontiguousarray(pos, np.float64)
    q = np.ascontiguousarray(q, np.float64)
    with tempfile.NamedTemporaryFile(suffix=".bin") as tmp:
        tmp.write(np.uint64(pos.shape[0]).tobytes() + pos.tobytes() + q.tobytes())
        tmp.flush()
        r = subprocess.run([_IO, "write", tmp.name, path, header], capture_output=True, text=True)
        if r.returncode != 0:
            raise RefError(r.returncode, r.stderr.strip())


class RefSetup:
    """hfmm::build_setup on the reference, with the flat dump accessors."""

    def __init__(self, pos, q, cfg: RefCfg):
        pos = np.ascontiguousarray(pos, np.float64)
        q = np.ascontiguousarray(q, np.float64)
        if np.iscomplexobj(q):
            q = np.ascontiguousarray(np.stack([q.real, q.imag], -1))
        self.n = pos.shape[0]
        self.cfg = cfg
        h = ctypes.c_void_p()
        _check(lib().ref_setup_build(_p(pos), _p(q), ctypes.c_size_t(self.n), ctypes.byref(cfg),
                                     ctypes.byref(h)))
        self._h = h
        meta = self.array("meta_i64", np.int64)
        self.levels, self.top_level = int(meta[0]), int(meta[1])
        self.num_leaves, self.num_ranks = int(meta[4]), int(meta[5])

    def array(self, name, dtype=np.uint8):
        nb = ctypes.c_size_t(0)
        _check(lib().ref_setup_get(self._h, name.encode(), None, ctypes.c_size_t(0), ctypes.byref(nb)))
        out = np.empty(nb.value, np.uint8)
        if nb.value:
            _check(lib().ref_setup_get(self._h, name.encode(), _p(out), ctypes.c_size_t(nb.value),
                                       ctypes.byref(nb)))
        return out.view(dtype)

    def sampling(self, level):
        return tuple(int(v) for v in self.array(f"L{level}.sampling", np.int64))

    def evaluate(self):
        """evaluate_with_setup -> (potentials complex input order, phase_sec[7], phase_flops[7])."""
        pot = np.empty((self.n, 2))
        sec = np.zeros(7)
        fl = np.zeros(7)
        _check(lib().ref_evaluate(self._h, _p(pot), _p(sec), _p(fl)))
        return pot[:, 0] + 1j * pot[:, 1], sec, fl

    def expansions(self, stop_phase: int, kind: int, level: int, want_pot=False):
        """Expansions of `level` after RankEngine phases 1..stop_phase (1 c2m .. 5 l2o_near)."""
        _, nt, nphi = self.sampling(level)
        nn = self.array(f"L{level}.codes", np.uint64).size
        out = np.zeros((nn, nt * nphi, 2))
        pot = np.zeros((self.n, 2)) if want_pot else None
        _check(lib().ref_expansions(self._h, ctypes.c_int(stop_phase), ctypes.c_int(kind),
                                    ctypes.c_int(level), _p(out), _p(pot)))
        e = out[..., 0] + 1j * out[..., 1]
        if want_pot:
            return e, pot[:, 0] + 1j * pot[:, 1]
        return e

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:
            _lib.ref_setup_destroy(h)


def direct(pos, q, obs_idx, lam=1.0, nthreads=8):
    pos = np.ascontiguousarray(pos, np.float64)
    q = np.ascontiguousarray(q)
    if np.iscomplexobj(q):
        q = np.ascontiguousarray(np.stack([q.real, q.imag], -1))
    obs = np.ascontiguousarray(obs_idx, np.int64)
    out = np.empty((obs.size, 2))
    _check(lib().ref_direct(_p(pos), _p(q), ctypes.c_size_t(pos.shape[0]), _p(obs), ctypes.c_size_t(obs.size),
                            ctypes.c_double(lam), ctypes.c_int(nthreads), _p(out)))
    return out[:, 0] + 1j * out[:, 1]


def green(k, r):
    out = np.empty(2)
    _check(lib().ref_green(ctypes.c_double(k), _p(np.ascontiguousarray(r, np.float64)), _p(out)))
    return complex(out[0], out[1])


def truncation_order(diameter, k, digits):
    v = ctypes.c_int()
    _check(lib().ref_truncation_order(ctypes.c_double(diameter), ctypes.c_double(k), ctypes.c_double(digits),
                                      ctypes.byref(v)))
    return v.value


def quadrature(nt, nphi):
    w = np.empty(nt)
    pw = ctypes.c_double()
    _check(lib().ref_quadrature(ctypes.c_size_t(nt), ctypes.c_size_t(nphi), _p(w), ctypes.byref(pw)))
    return w, pw.value


def translation_operator(trunc, nt, nphi, D, side, k):
    out = np.empty((nt * nphi, 2))
    _check(lib().ref_translation_operator(ctypes.c_int(trunc), ctypes.c_size_t(nt), ctypes.c_size_t(nphi),
                                          _p(np.ascontiguousarray(D, np.float64)), ctypes.c_double(side),
                                          ctypes.c_double(k), _p(out)))
    return out[:, 0] + 1j * out[:, 1]


def resample_grid(mode, grid, nt, nphi, nt_dst, nphi_dst):
    g = np.ascontiguousarray(np.stack([grid.real, grid.imag], -1), np.float64)
    out = np.empty((nt_dst * nphi_dst, 2))
    _check(lib().ref_resample_grid(ctypes.c_int(mode), _p(g), ctypes.c_size_t(nt), ctypes.c_size_t(nphi),
                                   ctypes.c_size_t(nt_dst), ctypes.c_size_t(nphi_dst), _p(out)))
    return out[:, 0] + 1j * out[:, 1]


def resample_circle(x, n_out, shift_in, shift_out):
    a = np.ascontiguousarray(np.stack([x.real, x.imag], -1), np.float64)
    out = np.empty((n_out, 2))
    _check(lib().ref_resample_circle(_p(a), ctypes.c_size_t(x.size), ctypes.c_double(shift_in), _p(out),
                                     ctypes.c_size_t(n_out), ctypes.c_double(shift_out)))
    return out[:, 0] + 1j * out[:, 1]


def c2m(pos, q, center, nt, nphi, k):
    pos = np.ascontiguousarray(pos, np.float64)
    qq = np.ascontiguousarray(np.stack([q.real, q.imag], -1), np.float64)
    out = np.empty((nt * nphi, 2))
    _check(lib().ref_c2m(_p(pos), _p(qq), ctypes.c_size_t(pos.shape[0]), _p(np.asarray(center, np.float64)),
                         ctypes.c_size_t(nt), ctypes.c_size_t(nphi), ctypes.c_double(k), _p(out)))
    return out[:, 0] + 1j * out[:, 1]


def l2o(local, nt, nphi, center, obs, k):
    g = np.ascontiguousarray(np.stack([local.real, local.imag], -1), np.float64)
    obs = np.ascontiguousarray(obs, np.float64)
    out = np.empty((obs.shape[0], 2))
    _check(lib().ref_l2o(_p(g), ctypes.c_size_t(nt), ctypes.c_size_t(nphi), _p(np.asarray(center, np.float64)),
                         _p(obs), ctypes.c_size_t(obs.shape[0]), ctypes.c_double(k), _p(out)))
    return out[:, 0] + 1j * out[:, 1]
