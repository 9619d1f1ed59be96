"""The oracle is pinned before it is trusted: known answers frozen in the
reference's own tests, the compiled reference, and the golden fixtures."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2
from oracle import hfmm_np

KA = json.load(open(os.path.join(GOLDEN, "known_answers.json")))


def test_known_answers_restatement():
    # green(k=1, (3,0,0)) -- proj/tests/test_kernel.cpp:29-34
    k, r = 1.0, 3.0
    g = np.exp(-1j * k * r) / (4 * np.pi * r)
    assert abs(g - complex(*KA["green_k1_r3"])) < 1e-15
    # translation operator, L_t = 0 -- proj/tests/test_operators.cpp:83-97
    T = hfmm_np.translation_operator(0, hfmm_np.directions(2, 2), np.array([2.5, 0, 0]), 1.0)
    assert np.all(np.abs(T - complex(*KA["T_Lt0_k1_D2.5"])) < 1e-13)
    # truncation order -- proj/tests/test_sphere_interp.cpp:64-67
    assert hfmm_np.truncation_order(1.0, 1.0, 3.0) == KA["trunc_d1_k1_dig3"]
    for key, want in KA["ref_trunc"].items():
        d, k2, dig = (float(v) for v in key.split("_"))
        assert hfmm_np.truncation_order(d, k2, dig) == want, key
    for nt, w in KA["ref_quad"].items():
        mine, pw = hfmm_np.quadrature(int(nt), int(nt))
        assert np.allclose(mine, w, rtol=0, atol=1e-15)
        assert abs(mine.sum() * pw * int(nt) - 4 * np.pi) < 1e-12  # weights sum to 4 pi


def test_known_answers_reference(refo):
    assert abs(refo.green(1.0, [3.0, 0, 0]) - complex(*KA["green_k1_r3"])) < 1e-15
    T = refo.translation_operator(0, 2, 2, [2.5, 0, 0], 1.0, 1.0)
    assert np.all(np.abs(T - complex(*KA["T_Lt0_k1_D2.5"])) < 1e-13)
    assert refo.truncation_order(1.0, 1.0, 3.0) == KA["trunc_d1_k1_dig3"]


def test_resample_golden():
    z = np.load(os.path.join(GOLDEN, "resample.npz"))
    for key in z.files:
        if key.startswith("circ_") and key.endswith("_in"):
            _, ni, si, no, so, _ = key.split("_")
            out = hfmm_np.resample_circle(z[key], int(no), float(si), float(so))
            assert rel_l2(out, z[key[:-3] + "_out"]) < 1e-13, key
    for nc, npar in [(18, 28), (26, 34)]:
        x = z[f"interp_{nc}_{npar}_in"].reshape(nc, nc)
        out = hfmm_np.fft_interpolate(x, npar, npar).reshape(-1)
        assert rel_l2(out, z[f"interp_{nc}_{npar}_out"]) < 1e-13
        y = z[f"anterp_{npar}_{nc}_in"].reshape(npar, npar)
        out = hfmm_np.fft_anterpolate(y, nc, nc).reshape(-1)
        assert rel_l2(out, z[f"anterp_{npar}_{nc}_out"]) < 1e-13


@pytest.mark.parametrize("case", ["case_cube3", "case_sphere4", "case_cube6"])
def test_restatement_vs_golden_potentials(case, native):
    import paper_2006_15367_b200 as hb
    z = np.load(os.path.join(GOLDEN, f"{case}.npz"))
    n, ext, seed, dig, _ = z["meta"]
    pos, q = hb.generate_inputs(str(z["shape"]), int(n), float(ext), int(seed))
    setup = hb.build_setup(pos, q, hb.RunConfig(digits=float(dig)))
    pot_sorted = hfmm_np.evaluate(setup)
    want = z["potentials"][setup.original_index]
    assert rel_l2(pot_sorted, want) < 1e-10
    # FMM accuracy against the direct sum is the reference's (not 10^-digits)
    k = 2 * np.pi
    d = hfmm_np.direct(pos, q, z["direct_obs"], k)
    assert rel_l2(d, z["direct"]) < 1e-13
    inv = np.empty_like(setup.original_index)
    inv[setup.original_index] = np.arange(int(n))
    err_np = rel_l2(pot_sorted[inv][z["direct_obs"]], d)
    err_ref = rel_l2(z["potentials"][z["direct_obs"]], z["direct"])
    assert abs(err_np - err_ref) < 1e-9


def test_restatement_vs_live_reference(refo):
    pos, q = refo.generate_inputs("cube", 4000, 2.5, 21)
    rs = refo.RefSetup(pos, q, refo.config(digits=3))
    pot, _, _ = rs.evaluate()
    mine = hfmm_np.evaluate(rs)
    orig = rs.array("original_index", np.uint64).astype(np.int64)
    assert rel_l2(mine, pot[orig]) < 1e-10
