"""Opt-in partition by near-field work: RunConfig.partition_weight=1
weights each leaf by its near pairs (n_leaf x sum of near-leaf populations)
instead of its particle count (the reference's rule, traversal.cpp:128-131)."""
import numpy as np
import pytest


def _near_pairs_per_leaf(setup):
    ls = setup.array("leaf_start", np.uint64).astype(np.int64)
    sizes = np.diff(ls)
    near_off = setup.array("near_off", np.uint64).astype(np.int64)
    codes = setup.array(f"L{setup.levels}.codes", np.uint64)
    near = np.searchsorted(codes, setup.array("near", np.uint64))
    per = np.add.reduceat(sizes[near], near_off[:-1])
    return sizes * per


def _rank_loads(setup, w):
    rr = setup.array("rank_ranges", np.uint64).astype(np.int64).reshape(-1, 2)
    return np.array([w[b:e].sum() for b, e in rr], dtype=np.float64)


@pytest.mark.parametrize("shape,n,ext,seed", [("sphere", 60_000, 3.0, 71), ("cube", 40_000, 3.0, 72)])
def test_near_pair_partition_balances_p2p(shape, n, ext, seed, native):
    import paper_2006_15367_b200 as hb
    pos, q = hb.generate_inputs(shape, n, ext, seed)
    base = hb.build_setup(pos, q, hb.RunConfig(digits=3.0, num_ranks=4))
    wtd = hb.build_setup(pos, q, hb.RunConfig(digits=3.0, num_ranks=4, partition_weight=1))
    w = _near_pairs_per_leaf(base).astype(np.float64)
    assert np.array_equal(w, _near_pairs_per_leaf(wtd))  # the tree does not depend on the partition
    imb_base = _rank_loads(base, w).max() / w.sum() * 4
    imb_wtd = _rank_loads(wtd, w).max() / w.sum() * 4
    assert imb_wtd <= imb_base + 1e-12
    assert imb_wtd < 1.05
    # everything but the partition-derived arrays is unchanged
    for name in ("leaf_codes", "leaf_start", "near_off", "near", "original_index"):
        assert base.array(name).tobytes() == wtd.array(name).tobytes()


def test_partition_weight_validation(native):
    import paper_2006_15367_b200 as hb
    pos, q = hb.generate_inputs("cube", 5000, 2.0, 73)
    with pytest.raises(hb.InvalidArgument):
        hb.build_setup(pos, q, hb.RunConfig(partition_weight=2))
    # default: bit-exact with the particle-weighted (reference) partition
    a = hb.build_setup(pos, q, hb.RunConfig(num_ranks=3))
    b = hb.build_setup(pos, q, hb.RunConfig(num_ranks=3, partition_weight=0))
    assert a.array("rank_ranges").tobytes() == b.array("rank_ranges").tobytes()
