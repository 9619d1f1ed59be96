"""Multi-rank path on CPU: world_size 2 and 3 over gloo.

Each process builds the global setup with num_ranks = world (bit-exact
partition), runs the rank-local CPU engine (tests/dist_np.py) through the SAME
driver the GPUs use (paper_2006_15367_b200/distributed.py: ghosts, plural
multipole reduce-scatter, sliced M2L halo from the reference CommPlan in
buffer_limit chunks, plural local gather), and the gathered potentials must
equal the single-rank evaluation.  Also checks that every rank's send plan is
exactly what its peer expects to receive.
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


def _worker(rank, world, port, outdir, case, buffer_limit=2**64 - 1):
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
    setup = hb.build_setup(pos, q, hb.RunConfig(digits=dig, num_ranks=world, buffer_limit=buffer_limit))
    eng = NumpyRankEngine(setup, rank)
    eng.set_charges_sorted(q[setup.original_index])
    ev = DistributedEvaluator(eng, rank, world, torch.device("cpu"))
    ev.step()
    pb, pot = eng.potentials_own()
    np.save(os.path.join(outdir, f"pot_{rank}.npy"), pot)
    np.save(os.path.join(outdir, f"pb_{rank}.npy"), np.array([pb]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,case,buffer_limit", [
    (2, ("cube", 3000, 2.5, 51, 3.0), 2**64 - 1),
    (3, ("sphere", 4000, 1.5, 52, 4.0), 2**64 - 1),
    (4, ("cube", 3000, 2.5, 53, 3.0), 4096),  # M_S: the M2L halo goes in 4 KB chunks
])
def test_multirank_driver_matches_single_rank(world, case, buffer_limit, native):
    import paper_2006_15367_b200 as hb
    sys.path.insert(0, ROOT)
    from oracle import hfmm_np
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, case, buffer_limit), nprocs=world, join=True)
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
    """What r sends q is item for item what q expects from r (kinds 0, 2, 3);
    every held observer's slice rows of every far source are either in the
    rank's own slice of that source or received through the M2L plan."""
    import paper_2006_15367_b200 as hb
    pos, q = hb.generate_inputs("cube", 100_000, 4.0, 0)
    s = hb.build_setup(pos, q, hb.RunConfig(num_ranks=ranks))
    for r in range(ranks):
        for p in range(ranks):
            if p == r:
                continue
            for k in (0, 2, 3):
                assert np.array_equal(s.array(f"R{r}.send{k}.{p}", np.int64), s.array(f"R{p}.recv{k}.{r}", np.int64))
    n_plural = 0
    for r in range(ranks):
        recv0 = np.concatenate([s.array(f"R{r}.recv0.{p}", np.int64).reshape(-1, 4)
                                for p in range(ranks) if p != r] or [np.zeros((0, 4), np.int64)])
        for l in range(s.top_level, s.levels + 1):
            held = set(s.array(f"R{r}.held.L{l}", np.int32).tolist())
            codes = s.array(f"L{l}.codes", np.uint64)
            fo = s.array(f"L{l}.far_off", np.uint64).astype(np.int64)
            far = np.searchsorted(codes, s.array(f"L{l}.far", np.uint64))
            so = s.array(f"L{l}.slices_off", np.uint64).astype(np.int64)
            sl = s.array(f"L{l}.slices", np.int64).reshape(-1, 3)
            users = s.array(f"L{l}.users", np.int64).reshape(-1, 3)
            n_plural += int(users[:, 2].sum())

            def mine(n):
                for z in range(so[n], so[n + 1]):
                    if sl[z, 0] == r and sl[z, 2] > sl[z, 1]:
                        return int(sl[z, 1]), int(sl[z, 2])
                return 0, 0
            got = {}
            for lv_, n, b, e in recv0[recv0[:, 0] == l]:
                got.setdefault(int(n), []).append((int(b), int(e)))
            for o in held:
                b, e = mine(o)
                for src in far[fo[o]:fo[o + 1]]:
                    cover = np.zeros(e - b, bool)
                    if src in held:
                        sb, se = mine(src)
                        cover[max(sb, b) - b:max(min(se, e) - b, 0)] = True
                    for rb, re_ in got.get(int(src), []):
                        lo, hi = max(rb, b), min(re_, e)
                        if lo < hi:
                            cover[lo - b:hi - b] = True
                    assert cover.all(), (r, l, o, int(src))
    assert n_plural > 0  # the case exercises sliced plural nodes
