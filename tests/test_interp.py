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
