"""Setup on the device: Morton keys + stable radix sort and the
far / near interaction lists built by CUDA kernels (RunConfig.setup_device=1)
are byte-identical to the host build, which test_setup_parity.py pins to the
reference's build_setup (traversal.cpp:66-238, interaction_lists.cpp:21-98)."""
import numpy as np
import pytest

from conftest import setup_array_names

CASES = [
    ("cube", 100_000, 4.0, 0, 3.0, 1),   # BASELINE config 1
    ("sphere", 200_000, 4.0, 2, 3.0, 1),  # sparse surface tree
    ("cube", 20_000, 3.3, 5, 6.0, 3),     # 3 ranks: partition / plans from the device lists
    ("sphere", 30_000, 1.7, 9, 4.0, 8),
]


def _arrays_equal(a, b, levels, top):
    names = setup_array_names(levels, top)
    return [nm for nm in names if not np.array_equal(a.array(nm), b.array(nm))]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_device_setup_bit_exact(case):
    import paper_2006_15367_b200 as hb
    shape, n, ext, seed, dig, ranks = case
    pos, q = hb.generate_inputs(shape, n, ext, seed)
    host = hb.build_setup(pos, q, hb.RunConfig(digits=dig, num_ranks=ranks))
    dev = hb.build_setup(pos, q, hb.RunConfig(digits=dig, num_ranks=ranks, setup_device=1))
    bad = _arrays_equal(host, dev, host.levels, host.top_level)
    assert not bad, f"arrays differ: {bad[:8]}"


@pytest.mark.gpu
def test_device_setup_top_level_one_and_errors():
    import paper_2006_15367_b200 as hb
    from paper_2006_15367_b200 import _native
    pos, q = hb.generate_inputs("cube", 5_000, 2.0, 4)
    for top in (1, 2):
        host = hb.build_setup(pos, q, hb.RunConfig(top_level=top, leaf_lambda=0.5))
        dev = hb.build_setup(pos, q, hb.RunConfig(top_level=top, leaf_lambda=0.5, setup_device=1))
        assert not _arrays_equal(host, dev, host.levels, host.top_level)
    with pytest.raises(_native.InvalidArgument):
        hb.build_setup(pos, q, hb.RunConfig(setup_device=2))


@pytest.mark.gpu
def test_device_setup_evaluates_like_host():
    import paper_2006_15367_b200 as hb
    pos, q = hb.generate_inputs("sphere", 50_000, 2.0, 11)
    a = hb.RankEngine(hb.build_setup(pos, q, hb.RunConfig(digits=4.0))).evaluate().potentials
    b = hb.RankEngine(hb.build_setup(pos, q, hb.RunConfig(digits=4.0, setup_device=1))).evaluate().potentials
    assert np.array_equal(a, b)


def test_device_setup_without_device_fails_loudly(native):
    """No silent host fallback: setup_device=1 without a CUDA device raises
    NoDeviceError (CPU-only check; on a GPU box the device build runs)."""
    import paper_2006_15367_b200 as hb
    from paper_2006_15367_b200 import _native
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except ImportError:
        pass
    pos, q = hb.generate_inputs("cube", 2_000, 2.0, 1)
    with pytest.raises(_native.NoDeviceError):
        hb.build_setup(pos, q, hb.RunConfig(setup_device=1))
