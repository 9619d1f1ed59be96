"""All logical ranks in one process (hfmm_world, the reference's run_world +
evaluate_with_setup): evaluate_with_setup for num_ranks > 1 and the phase
seam, against the reference at 1e-10.

The phase-by-phase check assembles every node's expansion from its users'
slices exactly as the reference's RankEngine::multipole / local_expansion
expose them (traversal.hpp:142-143; oracle ref_expansions): after M2M the
plural nodes' slices must hold the FULL multipole (the reference's sliced
aggregation, traversal.cpp:350-426), after L2L every slice the full local.
"""
import os

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.mark.parametrize("ranks,case", [
    (3, ("sphere", 30_000, 2.0, 32, 4.0)),
    (5, ("cube", 20_000, 3.0, 31, 3.0)),
    (8, ("cube", 60_000, 4.0, 64, 3.0)),
])
def test_world_phase_by_phase(ranks, case, native, refo):
    import paper_2006_15367_b200 as hb
    shape, n, ext, seed, dig = case
    pos, q2 = refo.generate_inputs(shape, n, ext, seed)
    q = q2[:, 0] + 1j * q2[:, 1]
    rs = refo.RefSetup(pos, q2, refo.config(digits=dig, num_ranks=ranks))
    setup = hb.build_setup(pos, q, hb.RunConfig(digits=dig, num_ranks=ranks))
    w = hb.World(setup)
    w.set_intensities(q)
    L, top = setup.levels, setup.top_level
    w.run_phase(hb.Phase.C2M)
    w.run_phase(hb.Phase.M2M)
    n_plural = 0
    for lvl in range(L - 1, top - 1, -1):
        n_plural += int(setup.array(f"L{lvl}.users", np.int64).reshape(-1, 3)[:, 2].sum())
        assert rel_l2(w.assembled(0, lvl), rs.expansions(2, 0, lvl)) < TOL, ("m2m", lvl)
    assert n_plural > 0
    w.run_phase(hb.Phase.M2L)
    w.run_phase(hb.Phase.L2L)
    for lvl in range(top, L + 1):
        assert rel_l2(w.assembled(1, lvl), rs.expansions(4, 1, lvl)) < TOL, ("l2l", lvl)
    w.run_phase(hb.Phase.L2T)
    want, _, _ = rs.evaluate()
    assert rel_l2(w.potentials(), want) < TOL


def test_evaluate_with_setup_multirank_matches_reference(native, refo):
    """evaluate_with_setup(num_ranks = 4) on one GPU: the reference's own
    semantics (all ranks in one process) -- same potentials as the reference
    at 4 ranks, and as the single-rank engine; a ledger row per rank."""
    import paper_2006_15367_b200 as hb
    pos, q2 = refo.generate_inputs("sphere", 40_000, 2.0, 62)
    q = q2[:, 0] + 1j * q2[:, 1]
    setup = hb.build_setup(pos, q, hb.RunConfig(digits=4.0, num_ranks=4))
    res = hb.evaluate_with_setup(setup)
    want, _, _ = refo.RefSetup(pos, q2, refo.config(digits=4.0, num_ranks=os.cpu_count() or 1,
                                                    scheduler=2)).evaluate()
    assert rel_l2(res.potentials, want) < TOL
    one = hb.evaluate_with_setup(hb.build_setup(pos, q, hb.RunConfig(digits=4.0))).potentials
    assert rel_l2(res.potentials, one) < 1e-12
    assert res.rank_ms.shape == (4, 7) and np.all(res.rank_ms >= 0) and res.rank_ms[:, 3].min() > 0
    # a second evaluation with new charges reuses the world's buffers
    w = hb.World(setup)
    r1 = w.evaluate(q).potentials
    r2 = w.evaluate(2.0 * q).potentials
    assert rel_l2(r2, 2.0 * r1) < 1e-13
