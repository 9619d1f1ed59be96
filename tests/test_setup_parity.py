"""Host setup (Morton keys, tree, partition, slices, lists, plans) is
bit-exact with the reference build_setup (traversal.cpp:66-238)."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, setup_array_names

CASES = [
    ("cube", 100_000, 4.0, 0, 3.0),
    ("sphere", 60_000, 2.0, 2, 3.0),
    ("cube", 20_000, 3.3, 5, 6.0),
    ("sphere", 30_000, 1.7, 9, 4.0),
]


def compare(ref_setup, mine):
    names = setup_array_names(ref_setup.levels, ref_setup.top_level)
    bad = [nm for nm in names if not np.array_equal(ref_setup.array(nm), mine.array(nm))]
    assert not bad, f"arrays differ: {bad[:8]}"


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("ranks", [1, 2, 3, 8])
@pytest.mark.parametrize("policy", [0, 1])
def test_setup_bit_exact(case, ranks, policy, refo, native):
    import paper_2006_15367_b200 as hb
    shape, n, ext, seed, dig = case
    pos, q = refo.generate_inputs(shape, n, ext, seed)
    rs = refo.RefSetup(pos, q, refo.config(digits=dig, num_ranks=ranks, policy=policy))
    mine = hb.build_setup(pos, q[:, 0] + 1j * q[:, 1],
                          hb.RunConfig(digits=dig, num_ranks=ranks, policy=hb.AlignPolicy(policy)))
    compare(rs, mine)


def test_setup_grid_and_top_level(refo, native):
    import paper_2006_15367_b200 as hb
    # 32x32 grid -> 6-level surface tree, d = 2 (proj/tests/test_traversal.cpp:42-62)
    pos, q = refo.generate_geometry("grid", 8.0, 0.25, seed=7)
    mine = hb.build_setup(pos, q, hb.RunConfig(one_particle_per_leaf=True))
    assert mine.levels == 6 and mine.d_class == 2 and mine.num_leaves == 1024
    compare(refo.RefSetup(pos, q, refo.config(one_particle_per_leaf=1)), mine)
    # aggregation to the root (top_level = 1), 8-leaf volume (test_traversal.cpp:111-130)
    pos, q = refo.generate_geometry("volume", 2.0, 1.0, seed=5)
    for ranks in (1, 2, 4):
        rs = refo.RefSetup(pos, q, refo.config(leaf_lambda=1.0, top_level=1, num_ranks=ranks))
        mine = hb.build_setup(pos, q, hb.RunConfig(leaf_lambda=1.0, top_level=1, num_ranks=ranks))
        assert mine.num_leaves == 8
        compare(rs, mine)
    # Fibonacci sphere, rank-ordered, 5 ranks
    pos, q = refo.generate_geometry("sphere", 3.0, 0.1, seed=3)
    for ranks in (1, 5):
        rs = refo.RefSetup(pos, q, refo.config(num_ranks=ranks, policy=0))
        compare(rs, hb.build_setup(pos, q, hb.RunConfig(num_ranks=ranks, policy=hb.AlignPolicy.RankOrdered)))


def test_setup_golden_hashes(native):
    """Bit-exactness pinned by fixtures (runs without the reference present)."""
    import paper_2006_15367_b200 as hb
    hashes = json.load(open(os.path.join(GOLDEN, "setup_hashes.json")))
    for name, ranks in (("cfg1_r1", 1), ("cfg1_r8", 8)):
        pos, q = hb.generate_inputs("cube", 100_000, 4.0, 0)
        mine = hb.build_setup(pos, q, hb.RunConfig(digits=3.0, num_ranks=ranks))
        for nm, h in hashes[name].items():
            assert hashlib.sha256(mine.array(nm).tobytes()).hexdigest() == h, (name, nm)


def test_setup_errors(native):
    import paper_2006_15367_b200 as hb
    with pytest.raises(hb.InvalidArgument):
        hb.build_setup(np.zeros((0, 3)), np.zeros(0, complex))
    with pytest.raises(hb.InvalidArgument):
        hb.build_setup(np.zeros((2, 3)), np.zeros(2, complex), hb.RunConfig(num_ranks=0))
    with pytest.raises(hb.InvalidArgument):
        hb.build_setup(np.array([[0.0, 0, 0], [np.nan, 0, 0]]), np.zeros(2, complex))
    # one_particle_per_leaf with two particles in one leaf (test_traversal.cpp:72-76)
    two = np.array([[0.1, 0.1, 0.1], [0.11, 0.1, 0.1]])
    with pytest.raises(hb.InvalidArgument):
        hb.build_setup(two, np.ones(2, complex), hb.RunConfig(one_particle_per_leaf=True))
    # more ranks than nonempty leaves (tree.cpp:25-27)
    with pytest.raises(hb.InvalidArgument):
        hb.build_setup(two, np.ones(2, complex), hb.RunConfig(num_ranks=2))
    with pytest.raises(hb.InvalidArgument):
        hb.RunConfig(buffer_limit=0).validate()
