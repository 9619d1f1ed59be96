"""Multi-rank path on CPU: world_size 2 and 3 over gloo.

Each process builds the global setup with num_ranks = world (bit-exact
partition), runs the rank-local CPU engine (tests/dist_np.py) through the SAME
driver the GPUs use (paper_2006_15367_b200/distributed.py: ghost exchange,
partial-multipole exchange), and the gathered potentials must equal the
single-rank evaluation.  Also checks that every rank's send plan is exactly
what its peer expects to receive.
"""
import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, case):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2006_15367_b200 as hb
    from paper_2006_15367_b200.distributed import DistributedEvaluator
    from dist_np import NumpyRankEngine
    shape, n, ext, seed, dig = case
    pos, q = hb.generate_inputs(shape, n, ext, seed)
    setup = hb.build_setup(pos, q, hb.RunConfig(digits=dig, num_ranks=world))
    eng = NumpyRankEngine(setup, rank)
    eng.set_charges_sorted(q[setup.original_index])
    ev = DistributedEvaluator(eng, rank, world, torch.device("cpu"))
    ev.step()
    pb, pot = eng.potentials_own()
    np.save(os.path.join(outdir, f"pot_{rank}.npy"), pot)
    np.save(os.path.join(outdir, f"pb_{rank}.npy"), np.array([pb]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, ("cube", 3000, 2.5, 51, 3.0)),
    (3, ("sphere", 4000, 1.5, 52, 4.0)),
])
def test_multirank_driver_matches_single_rank(world, case, native):
    import paper_2006_15367_b200 as hb
    sys.path.insert(0, ROOT)
    from oracle import hfmm_np
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, case), nprocs=world, join=True)
        shape, n, ext, seed, dig = case
        pos, q = hb.generate_inputs(shape, n, ext, seed)
        single = hb.build_setup(pos, q, hb.RunConfig(digits=dig))
        want = hfmm_np.evaluate(single)
        got = np.full(n, np.nan, complex)
        for r in range(world):
            pb = int(np.load(os.path.join(d, f"pb_{r}.npy"))[0])
            pot = np.load(os.path.join(d, f"pot_{r}.npy"))
            got[pb:pb + pot.size] = pot
    assert np.all(np.isfinite(got)), "a rank used data it was never sent"
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_exchange_plans_are_symmetric(ranks, native):
    """What r sends q is item for item what q expects from r; ghost plans too."""
    import paper_2006_15367_b200 as hb
    pos, q = hb.generate_inputs("cube", 100_000, 4.0, 0)
    s = hb.build_setup(pos, q, hb.RunConfig(num_ranks=ranks))
    for r in range(ranks):
        for p in range(ranks):
            if p == r:
                continue
            assert np.array_equal(s.array(f"R{r}.mp_send.{p}", np.int32), s.array(f"R{p}.mp_recv.{r}", np.int32))
    # every far source of a held observer is held or received
    for r in range(ranks):
        for l in range(s.top_level, s.levels + 1):
            held = set(s.array(f"R{r}.held.L{l}", np.int32).tolist())
            halo = set(s.array(f"R{r}.halo.L{l}", np.int32).tolist())
            assert not (held & halo)
            codes = s.array(f"L{l}.codes", np.uint64)
            fo = s.array(f"L{l}.far_off", np.uint64).astype(np.int64)
            far = np.searchsorted(codes, s.array(f"L{l}.far", np.uint64))
            for o in held:
                assert set(far[fo[o]:fo[o + 1]].tolist()) <= held | halo
