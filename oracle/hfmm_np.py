"""NumPy restatement of the reference MLFMA evaluation phase.

TEST INFRASTRUCTURE ONLY (the checker, never the product path).  Each function
restates the reference algorithm and cites the file:line it follows
(/root/reference/proj/...).  Parity of this restatement is pinned two ways:
against the compiled, unmodified reference (oracle/_ref, tests/test_oracle.py)
and against committed golden fixtures made from it (tests/golden/).

Third-party arithmetic on the path: the reference resamples with FFTW3 (no
version pinned anywhere in the reference; not vendored).  Its published
algorithm is an unnormalised DFT (FFTW_FORWARD = exp(-2 pi i jk/n),
FFTW_BACKWARD = exp(+2 pi i jk/n)); numpy.fft computes the same transform
(ifft carries 1/n, undone here).  The spherical Bessel functions come from
libstdc++ (std::sph_bessel / std::sph_neumann) in the reference and from
scipy.special here; both are accurate to a few ulps.

The restatement evaluates one logical rank (the reference is
rank-transparent to ~1e-14, proj/tests/acceptance.cpp:96-126).
"""
from __future__ import annotations

import numpy as np
from scipy.special import spherical_jn, spherical_yn

KC2M = 12  # operators.hpp:18


def truncation_order(diameter: float, k: float, digits: float) -> int:
    """sphere_grid.cpp:13-23."""
    kd = k * diameter
    return max(4, int(np.ceil(kd + 1.8 * digits ** (2.0 / 3.0) * np.cbrt(kd))))


def directions(nt: int, nphi: int) -> np.ndarray:
    """LevelSampling::direction, sphere_grid.cpp:25-37 -> (S, 3), theta-major."""
    th = (np.arange(nt) + 0.5) * np.pi / nt
    ph = np.arange(nphi) * 2.0 * np.pi / nphi
    st = np.sin(th)[:, None]
    d = np.stack([st * np.cos(ph)[None, :], st * np.sin(ph)[None, :],
                  np.broadcast_to(np.cos(th)[:, None], (nt, nphi))], axis=-1)
    return d.reshape(-1, 3)


def quadrature(nt: int, nphi: int):
    """make_quadrature, sphere_grid.cpp:52-70 -> (theta weights, phi weight)."""
    th = (np.arange(nt) + 0.5) * np.pi / nt
    m = np.arange(1, nt // 2 + 1)
    s = (np.cos(2.0 * m[None, :] * th[:, None]) / (4.0 * m * m - 1.0)[None, :]).sum(axis=1)
    return (2.0 / nt) * (1.0 - 2.0 * s), 2.0 * np.pi / nphi


def resample_circle(x: np.ndarray, n_out: int, s_in: float, s_out: float) -> np.ndarray:
    """resample_circle, sphere_grid.cpp:128-155, batched over leading axes."""
    n_in = x.shape[-1]
    spec = np.fft.fft(x, axis=-1)
    K = min(n_in, n_out)
    q = np.arange(K)
    m = np.where(q <= (K - 1) // 2, q, q - K)
    ang = m * 2.0 * np.pi * (s_out / n_out - s_in / n_in)
    dst = np.zeros(x.shape[:-1] + (n_out,), dtype=complex)
    dst[..., m % n_out] = spec[..., m % n_in] * np.exp(1j * ang) / n_in
    return np.fft.ifft(dst, axis=-1) * n_out


def fold(g: np.ndarray) -> np.ndarray:
    """fold_transpose, sphere_grid.cpp:72-83: (..., nt, np) -> (..., np/2, 2 nt)."""
    nt, nphi = g.shape[-2], g.shape[-1]
    half = nphi // 2
    first = np.swapaxes(g[..., :, :half], -1, -2)             # rows i < nt
    second = np.swapaxes(g[..., ::-1, half:], -1, -2)         # rows 2nt-1-i
    return np.concatenate([first, second], axis=-1)


def unfold(f: np.ndarray, nt: int, nphi: int) -> np.ndarray:
    """unfold_transpose, sphere_grid.cpp:85-102."""
    half = nphi // 2
    g = np.empty(f.shape[:-2] + (nt, nphi), dtype=complex)
    g[..., :, :half] = np.swapaxes(f[..., :, :nt], -1, -2)
    g[..., :, half:] = np.swapaxes(f[..., :, nt:], -1, -2)[..., ::-1, :]
    return g


def fft_interpolate(g: np.ndarray, nt_dst: int, np_dst: int) -> np.ndarray:
    """sphere_grid.cpp:183-192."""
    wide = resample_circle(g, np_dst, 0.0, 0.0)
    tall = resample_circle(fold(wide), 2 * nt_dst, 0.5, 0.5)
    return unfold(tall, nt_dst, np_dst)


def fft_anterpolate(g: np.ndarray, nt_dst: int, np_dst: int) -> np.ndarray:
    """sphere_grid.cpp:194-204."""
    nphi = g.shape[-1]
    short = resample_circle(fold(g), 2 * nt_dst, 0.5, 0.5)
    narrow = unfold(short, nt_dst, nphi)
    return resample_circle(narrow, np_dst, 0.0, 0.0)


def translation_operator(trunc: int, dirs: np.ndarray, D: np.ndarray, k: float) -> np.ndarray:
    """operators.cpp:39-80 (Legendre recurrence, coefficients (-i)^l (2l+1) h_l^(2))."""
    dist = float(np.sqrt(D @ D))
    x = k * dist
    ell = np.arange(trunc + 1)
    h2 = spherical_jn(ell, x) - 1j * spherical_yn(ell, x)
    coef = (-1j) ** ell * (2 * ell + 1) * h2
    u = dirs @ (D * (1.0 / dist))
    pm1 = np.zeros_like(u)
    p0 = np.ones_like(u)
    acc = np.full(u.shape, coef[0], dtype=complex)
    for l in range(1, trunc + 1):
        p1 = ((2 * l - 1) * u * p0 - (l - 1) * pm1) / l
        pm1, p0 = p0, p1
        acc += coef[l] * p0
    return acc


def _cells(codes: np.ndarray, level: int) -> np.ndarray:
    """MortonKey::cell_{x,y,z}, morton.hpp:29-39 -> (n, 3)."""
    codes = codes.astype(np.uint64)
    out = np.zeros((codes.size, 3), dtype=np.int64)
    for t in range(level - 1):
        for a in range(3):
            out[:, a] |= ((codes >> np.uint64(3 * t + a)) & np.uint64(1)).astype(np.int64) << t
    return out


def evaluate(setup, charges_sorted: np.ndarray | None = None, return_expansions: bool = False):
    """Single-rank evaluate_with_setup (traversal.cpp:306-788) on a setup object
    exposing the flat arrays (oracle.ref.RefSetup or the product GlobalSetup).
    Returns sorted-order potentials (and per-level expansions if asked)."""
    meta = setup.array("meta_i64", np.int64)
    L, top = int(meta[0]), int(meta[1])
    mf = setup.array("meta_f64", np.float64)
    k = float(mf[5])
    parts = setup.array("particles", np.float64).reshape(-1, 5)
    pos = parts[:, :3]
    q = parts[:, 3] + 1j * parts[:, 4] if charges_sorted is None else charges_sorted
    leaf_start = setup.array("leaf_start", np.uint64).astype(np.int64)

    lv = {}
    for l in range(top, L + 1):
        tr, nt, nphi = (int(v) for v in setup.array(f"L{l}.sampling", np.int64))
        codes = setup.array(f"L{l}.codes", np.uint64)
        lv[l] = dict(trunc=tr, nt=nt, np=nphi, S=nt * nphi, codes=codes,
                     centers=setup.array(f"L{l}.centers", np.float64).reshape(-1, 3),
                     dirs=directions(nt, nphi), quad=quadrature(nt, nphi),
                     child_off=setup.array(f"L{l}.child_off", np.uint64).astype(np.int64),
                     children=setup.array(f"L{l}.children", np.uint64).astype(np.int64),
                     far_off=setup.array(f"L{l}.far_off", np.uint64).astype(np.int64),
                     far=np.searchsorted(codes, setup.array(f"L{l}.far", np.uint64)))
    mp, loc = {}, {}

    # C2M (operators.cpp:15-26, traversal.cpp:306-320)
    d = lv[L]
    M = np.zeros((d["codes"].size, d["S"]), dtype=complex)
    for li in range(d["codes"].size):
        b, e = leaf_start[li], leaf_start[li + 1]
        rel = pos[b:e] - d["centers"][li]
        M[li] = np.exp(1j * k * (d["dirs"] @ rel.T)) @ q[b:e]
    mp[L] = M

    # M2M (traversal.cpp:322-429): interpolate, shift by c_child - c_parent, sum in child order
    for l in range(L - 1, top - 1, -1):
        P, C = lv[l], lv[l + 1]
        up = fft_interpolate(mp[l + 1].reshape(-1, C["nt"], C["np"]), P["nt"], P["np"]).reshape(-1, P["S"])
        acc = np.zeros((P["codes"].size, P["S"]), dtype=complex)
        for pi in range(P["codes"].size):
            for ci in C_children(P, pi):
                disp = C["centers"][ci] - P["centers"][pi]
                acc[pi] += up[ci] * np.exp(1j * k * (P["dirs"] @ disp))
        mp[l] = acc

    # M2L (operators.cpp:82-87, traversal.cpp:443-581)
    for l in range(top, L + 1):
        d = lv[l]
        side = float(setup.array("meta_f64", np.float64)[0]) / 2 ** (l - 1)
        cells = _cells(d["codes"], l)
        Lc = np.zeros((d["codes"].size, d["S"]), dtype=complex)
        cache = {}
        for o in range(d["codes"].size):
            for src in d["far"][d["far_off"][o]:d["far_off"][o + 1]]:
                off = tuple(cells[o] - cells[src])
                if off not in cache:
                    cache[off] = translation_operator(d["trunc"], d["dirs"], np.array(off, float) * side, k)
                Lc[o] += mp[l][src] * cache[off]
        loc[l] = Lc

    # L2L (traversal.cpp:583-707): shift by c_parent - c_child, x w_p, weighted-adjoint anterp, / w_c
    for l in range(top, L):
        P, C = lv[l], lv[l + 1]
        wp = np.repeat(P["quad"][0], P["np"]) * P["quad"][1]
        wc = np.repeat(C["quad"][0], C["np"]) * C["quad"][1]
        for pi in range(P["codes"].size):
            for ci in C_children(P, pi):
                disp = P["centers"][pi] - C["centers"][ci]
                z = loc[l][pi] * np.exp(1j * k * (P["dirs"] @ disp)) * wp
                down = fft_anterpolate(z.reshape(P["nt"], P["np"]), C["nt"], C["np"]).reshape(-1)
                down *= P["S"] / C["S"]
                loc[l + 1][ci] += down / wc

    # L2O + near field (operators.cpp:89-122, traversal.cpp:709-788)
    d = lv[L]
    w = np.repeat(d["quad"][0], d["np"]) * d["quad"][1]
    norm = -1j * k / (16.0 * np.pi ** 2)
    pot = np.zeros(pos.shape[0], dtype=complex)
    near_off = setup.array("near_off", np.uint64).astype(np.int64)
    near = np.searchsorted(d["codes"], setup.array("near", np.uint64))
    for li in range(d["codes"].size):
        b, e = leaf_start[li], leaf_start[li + 1]
        rel = pos[b:e] - d["centers"][li]
        pot[b:e] = norm * (np.exp(-1j * k * (rel @ d["dirs"].T)) @ (w * loc[L][li]))
        srcs = np.concatenate([np.arange(leaf_start[j], leaf_start[j + 1]) for j in near[near_off[li]:near_off[li + 1]]])
        dv = pos[b:e, None, :] - pos[None, srcs, :]
        r = np.sqrt((dv * dv).sum(-1))
        ok = r > 0
        g = np.where(ok, np.exp(-1j * k * r) / (4.0 * np.pi * np.where(ok, r, 1.0)), 0.0)
        pot[b:e] += g @ q[srcs]
    if return_expansions:
        return pot, mp, loc
    return pot


def C_children(P, pi):
    return P["children"][P["child_off"][pi]:P["child_off"][pi + 1]]


def direct(pos: np.ndarray, q: np.ndarray, obs_idx: np.ndarray, k: float) -> np.ndarray:
    """direct_potential, kernel.cpp:16-41 (self pair skipped)."""
    out = np.empty(obs_idx.size, dtype=complex)
    for i, m in enumerate(obs_idx):
        dv = pos[m] - pos
        r = np.sqrt((dv * dv).sum(-1))
        ok = r > 0
        out[i] = (np.exp(-1j * k * r[ok]) / (4.0 * np.pi * r[ok])) @ q[ok]
    return out
