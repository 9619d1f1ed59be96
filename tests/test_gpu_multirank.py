"""Distributed-mode device code on ONE GPU: all P ranks' engines run in one
process, stage by stage through the same schedule as the NCCL driver (no
kernel ever waits on another rank): ghosts, plural multipole reduce-scatter,
sliced M2L halo (the reference CommPlan), plural local gather.  Potentials
must match the reference within 1e-10."""
import os

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _run_ranks(hb, setup, q, engs):
    """One evaluation of all P rank engines through the distributed schedule
    (paper_2006_15367_b200.distributed.run_emulated); returns the assembled
    sorted-order potentials."""
    from paper_2006_15367_b200.distributed import run_emulated
    for e in engs:
        e.set_intensities(q)
    run_emulated(engs, lambda n: torch.empty(int(n), dtype=torch.float64, device="cuda"))
    for e in engs:
        e.synchronize()
    pot = np.full(setup.n, np.nan, complex)
    dev = torch.full((setup.n, 2), float("nan"), dtype=torch.float64, device="cuda")
    for e in engs:
        b, en = e.particle_range()
        pot[b:en] = e.potentials_sorted()[b:en]
        e.store_potentials_device(dev.data_ptr())  # own range only, async on the engine stream
        e.synchronize()
    d = dev.cpu().numpy()
    assert np.array_equal(d[:, 0] + 1j * d[:, 1], pot)  # ranges tile [0, n) exactly
    return pot


@pytest.mark.parametrize("ranks,case,pw", [
    (2, ("cube", 30_000, 3.0, 61, 3.0), 0),
    (3, ("sphere", 40_000, 2.0, 62, 4.0), 0),
    (4, ("cube", 20_000, 2.5, 63, 6.0), 0),
    (4, ("sphere", 40_000, 2.0, 62, 4.0), 1),  # near-pair-weighted partition (opt-in)
    (8, ("cube", 60_000, 4.0, 64, 3.0), 0),
])
def test_ranks_emulated_on_one_gpu(ranks, case, pw, native, refo):
    import paper_2006_15367_b200 as hb
    shape, n, ext, seed, dig = case
    pos, q = hb.generate_inputs(shape, n, ext, seed)
    setup = hb.build_setup(pos, q, hb.RunConfig(digits=dig, num_ranks=ranks, partition_weight=pw))
    engs = [hb.RankEngine(setup, r, 0) for r in range(ranks)]
    l0 = [e.launch_count() for e in engs]
    pot_sorted = _run_ranks(hb, setup, q, engs)
    assert all(e.launch_count() - c >= 6 for e, c in zip(engs, l0))  # every phase launched kernels
    assert np.all(np.isfinite(pot_sorted))
    q2 = np.stack([q.real, q.imag], -1)
    want, _, _ = refo.RefSetup(pos, q2, refo.config(digits=dig, num_ranks=os.cpu_count() or 1,
                                                   scheduler=2)).evaluate()
    got = np.empty(n, complex)
    got[setup.original_index] = pot_sorted
    assert rel_l2(got, want) < 1e-10
    # a second evaluation on the same engines must not see stale halo data
    pot2 = _run_ranks(hb, setup, 2.0 * q, engs)
    assert rel_l2(pot2, 2.0 * pot_sorted) < 1e-13


def test_distributed_engine_rejects_one_shot_evaluate(native):
    import paper_2006_15367_b200 as hb
    pos, q = hb.generate_inputs("cube", 5000, 2.0, 64)
    setup = hb.build_setup(pos, q, hb.RunConfig(num_ranks=2))
    eng = hb.RankEngine(setup, 1, 0)
    with pytest.raises(hb.LogicError):
        eng.evaluate()
