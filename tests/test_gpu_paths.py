"""Kernel families that the small parity cases do not reach on their own.

The engine picks its M2M / L2L kernels per (child, parent) grid pair:
compile-time-shaped streaming pairs (interp_rb.cuh, the BASELINE leaf-side
pairs), runtime-shaped streaming kernels (`*_rbl`, B in shared memory) and,
for grids whose matrices do not fit shared memory, the two-stage large-grid
kernels (interp_big.cuh: k_m2m_big_*, k_l2l_big_*; config 5's top levels).
Leaf grids past n = 32 use the generic C2M / L2T kernels (k_c2m, k_l2t).

Here every family is compared phase by phase with the reference
(RankEngine::multipole / local_expansion after each phase, traversal.hpp:129-143)
at 1e-10, both through the test hooks that force a family on every level
(HFMM_NO_RB, HFMM_NO_RBL, HFMM_NO_QUAD, read when an engine is created) and on
geometries whose natural dispatch selects it.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def hb(native):
    import paper_2006_15367_b200 as hb
    return hb


def _phase_by_phase(hb, refo, pos, q2, cfg_kw, levels_check=True):
    q = q2[:, 0] + 1j * q2[:, 1]
    rs = refo.RefSetup(pos, q2, refo.config(**cfg_kw))
    kw = dict(cfg_kw)
    kw.pop("num_ranks", None)
    kw.pop("scheduler", None)
    setup = hb.build_setup(pos, q, hb.RunConfig(**kw))
    eng = hb.RankEngine(setup)
    L, top = setup.levels, setup.top_level
    eng.c2m_phase()
    assert rel_l2(eng.multipole(L), rs.expansions(1, 0, L)) < TOL
    eng.m2m_pass()
    if levels_check:
        for l in range(L - 1, top - 1, -1):
            assert rel_l2(eng.multipole(l), rs.expansions(2, 0, l)) < TOL, ("m2m", l)
    eng.m2l_pass()
    eng.l2l_pass()
    if levels_check:
        for l in range(top, L + 1):
            assert rel_l2(eng.local_expansion(l), rs.expansions(4, 1, l)) < TOL, ("l2l", l)
    pot_sorted = eng.l2o_near_phase()
    _, want = rs.expansions(5, 1, L, want_pot=True)
    assert rel_l2(pot_sorted, want) < TOL
    return setup


@pytest.mark.parametrize("hooks", [("HFMM_NO_RB",), ("HFMM_NO_RB", "HFMM_NO_RBL"), ("HFMM_NO_QUAD",)])
@pytest.mark.parametrize("case", [("cube", 20_000, 3.0, 31, 3.0), ("sphere", 30_000, 2.0, 32, 4.0)])
def test_forced_kernel_family(hooks, case, hb, refo, monkeypatch):
    """NO_RB: every pair on the runtime-shaped `*_rbl` kernels; NO_RB + NO_RBL:
    every pair on the two-stage large-grid kernels; NO_QUAD: generic C2M / L2T."""
    for h in hooks:
        monkeypatch.setenv(h, "1")
    shape, n, ext, seed, dig = case
    pos, q2 = refo.generate_inputs(shape, n, ext, seed)
    _phase_by_phase(hb, refo, pos, q2, dict(digits=dig))


def test_large_grid_kernels_natural_dispatch(hb, refo):
    """A 40-wavelength cube with 5-wavelength leaves: level 3 samples n = 256,
    whose theta matrices exceed shared memory, so M2M (level 4 -> 3) and L2L
    (3 -> 4) run k_m2m_big_* / k_l2l_big_* without any hook."""
    pos, q2 = refo.generate_inputs("cube", 3000, 40.0, 41)
    setup = _phase_by_phase(hb, refo, pos, q2, dict(digits=3.0, leaf_lambda=5.0))
    assert setup.sampling(3)[1] == 256 and setup.levels == 4


def test_generic_leaf_kernels_natural_dispatch(hb, refo):
    """Half-wavelength leaves at 6 digits give a leaf grid of n = 34 > 32:
    C2M / L2T run the generic kernels without any hook."""
    pos, q2 = refo.generate_inputs("cube", 6000, 4.0, 42)
    setup = _phase_by_phase(hb, refo, pos, q2, dict(digits=6.0, leaf_lambda=0.5))
    assert setup.sampling(setup.levels)[1] > 32


@pytest.mark.parametrize("hooks", [("HFMM_NO_RB", "HFMM_NO_RBL"), ("HFMM_NO_RB",)])
def test_forced_kernel_family_multirank(hooks, hb, refo, monkeypatch):
    """The same kernel families over held-node lists (distributed mode: the
    `clist` / `plist` paths), 3 ranks emulated on one GPU."""
    from test_gpu_multirank import _run_ranks
    for h in hooks:
        monkeypatch.setenv(h, "1")
    pos, q = hb.generate_inputs("sphere", 40_000, 2.0, 62)
    setup = hb.build_setup(pos, q, hb.RunConfig(digits=4.0, num_ranks=3))
    engs = [hb.RankEngine(setup, r, 0) for r in range(3)]
    pot_sorted = _run_ranks(hb, setup, q, engs)
    want, _, _ = refo.RefSetup(pos, np.stack([q.real, q.imag], -1),
                               refo.config(digits=4.0, num_ranks=os.cpu_count() or 1, scheduler=2)).evaluate()
    got = np.empty(q.size, complex)
    got[setup.original_index] = pot_sorted
    assert rel_l2(got, want) < TOL
