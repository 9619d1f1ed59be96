"""Dense resampling matrices (what the device applies) reproduce the
reference's FFT resampling (sphere_grid.cpp:128-214)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2


def test_resample_matrix_vs_golden(native):
    import paper_2006_15367_b200 as hb
    z = np.load(os.path.join(GOLDEN, "resample.npz"))
    for key in z.files:
        if key.startswith("circ_") and key.endswith("_in"):
            _, ni, si, no, so, _ = key.split("_")
            M = hb.resample_matrix(int(ni), float(si), int(no), float(so))
            assert rel_l2(M @ z[key], z[key[:-3] + "_out"]) < 1e-14, key


def _interp_dense(x, nc, npar):
    """fft_interpolate via the dense phi / folded-theta matrices (device recipe)."""
    import paper_2006_15367_b200 as hb
    P = hb.resample_matrix(nc, 0.0, npar, 0.0)
    T = hb.resample_matrix(2 * nc, 0.5, 2 * npar, 0.5)
    W = x.reshape(nc, nc) @ P.T
    half = npar // 2
    F = np.concatenate([W[:, :half].T, W[::-1, half:].T], axis=1)  # (half, 2nc)
    G = F @ T.T                                                   # (half, 2npar)
    Y = np.empty((npar, npar), complex)
    Y[:, :half] = G[:, :npar].T
    Y[:, half:] = G[:, npar:].T[::-1, :]
    return Y.reshape(-1)


@pytest.mark.parametrize("nc,npar", [(18, 28), (26, 34)])
def test_dense_interpolation_equals_fft(nc, npar, native):
    z = np.load(os.path.join(GOLDEN, "resample.npz"))
    out = _interp_dense(z[f"interp_{nc}_{npar}_in"], nc, npar)
    assert rel_l2(out, z[f"interp_{nc}_{npar}_out"]) < 1e-14


@pytest.mark.parametrize("nc,npar", [(18, 28), (22, 30), (116, 210)])
def test_dense_interpolation_live(nc, npar, native, refo):
    rng = np.random.default_rng(nc)
    x = rng.standard_normal(nc * nc) + 1j * rng.standard_normal(nc * nc)
    want = refo.resample_grid(0, x, nc, nc, npar, npar)
    assert rel_l2(_interp_dense(x, nc, npar), want) < 1e-13


# ---------------------------------------------------------------------------
# The packed device operands (real + rank-1 matrices, even / odd theta passes with
# the fold / unfold baked into the phi matrices, csrc/interp.hpp) applied the way
# the kernels apply them (interp_rb.cuh, interp_fused.cuh) reproduce the dense maps.
def _m2m_packed(x, nc, npar):
    from paper_2006_15367_b200 import hfmm
    bphi, vphi, bth, vth, kh = hfmm.m2m_operands(nc, npar)
    half = npar // 2
    X = x.reshape(nc, nc)
    # phi pass: row [x ; i (v . x)] @ B -> column 2 p + h = part h of circle p
    A = np.zeros((nc, bphi.shape[0]), complex)
    A[:, :nc] = X
    A[:, nc] = 1j * (X @ vphi)
    W = A @ bphi                                  # (nc rows i, Np columns)
    Y = np.empty((npar, npar), complex)
    for p in range(half):
        xe, xo = W[:, 2 * p], W[:, 2 * p + 1]
        alpha = vth[:nc] @ xe + vth[kh:kh + nc] @ xo
        ae, ao = np.zeros(kh, complex), np.zeros(kh, complex)
        ae[:nc], ao[:nc] = xe, xo
        ae[nc] = ao[nc] = 1j * alpha
        ye, yo = ae @ bth[:kh], ao @ bth[kh:]
        Y[:, p] = (ye + yo)[:npar]                # front sample (theta row n, column p)
        Y[:, p + half] = (ye - yo)[:npar]         # back sample (column p + half)
    return Y.reshape(-1)


@pytest.mark.parametrize("nc,npar", [(18, 28), (28, 42), (26, 34), (42, 68)])
def test_packed_m2m_operands_equal_dense(nc, npar, native):
    rng = np.random.default_rng(nc + npar)
    x = rng.standard_normal(nc * nc) + 1j * rng.standard_normal(nc * nc)
    assert rel_l2(_m2m_packed(x, nc, npar), _interp_dense(x, nc, npar)) < 1e-13


def _anterp_dense(y, nc, npar, rs, cs):
    """theta map 2 np -> 2 nc (scaled) per folded circle, then phi map np -> nc per row."""
    import paper_2006_15367_b200 as hb
    T = rs[:, None] * hb.resample_matrix(2 * npar, 0.5, 2 * nc, 0.5) * cs[None, :]
    P = hb.resample_matrix(npar, 0.0, nc, 0.0)
    half = npar // 2
    Yg = y.reshape(npar, npar)
    F = np.concatenate([Yg[:, :half].T, Yg[::-1, half:].T], axis=1)  # (half, 2 np)
    G = F @ T.T                                                      # (half, 2 nc)
    N = np.empty((nc, npar), complex)                                # narrow rows
    N[:, :half] = G[:, :nc].T
    N[:, half:] = G[:, nc:].T[::-1, :]
    return (N @ P.T).reshape(-1)


def _anterp_packed(y, nc, npar, rs, cs):
    from paper_2006_15367_b200 import hfmm
    bth, vth, bphi, vphi, kh = hfmm.l2l_operands(nc, npar, rs, cs)
    half = npar // 2
    Yg = y.reshape(npar, npar)
    N = np.zeros((nc, bphi.shape[0]), complex)    # narrow rows of (Ye, Yo) pairs + rank-1 column
    for p in range(half):
        f, b = Yg[:, p], Yg[:, p + half]
        xe, xo = f + b, f - b
        alpha = vth[:npar] @ xe + vth[kh:kh + npar] @ xo
        ae, ao = np.zeros(kh, complex), np.zeros(kh, complex)
        ae[:npar], ao[:npar] = xe, xo
        ae[npar] = ao[npar] = 1j * alpha
        N[:, 2 * p] = (ae @ bth[:kh])[:nc]
        N[:, 2 * p + 1] = (ao @ bth[kh:])[:nc]
    N[:, npar] = 1j * (N[:, :npar] @ vphi)
    return (N @ bphi)[:, :nc].reshape(-1)


@pytest.mark.parametrize("nc,npar", [(18, 28), (28, 42), (26, 34)])
def test_packed_l2l_operands_equal_dense(nc, npar, native):
    rng = np.random.default_rng(7 * nc + npar)
    y = rng.standard_normal(npar * npar) + 1j * rng.standard_normal(npar * npar)
    # symmetric positive weights, as the theta quadrature weights are (w_i = w_{2n-1-i})
    wc, wp = rng.uniform(0.5, 1.5, nc), rng.uniform(0.5, 1.5, npar)
    rs, cs = np.concatenate([wc, wc[::-1]]), np.concatenate([wp, wp[::-1]])
    assert rel_l2(_anterp_packed(y, nc, npar, rs, cs), _anterp_dense(y, nc, npar, rs, cs)) < 1e-13


def test_operand_queries_reject_odd_grids(native):
    import paper_2006_15367_b200 as hb
    from paper_2006_15367_b200 import hfmm
    with pytest.raises(hb.InvalidArgument):
        hfmm.m2m_operands(17, 28)
