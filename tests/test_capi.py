"""The C-ABI library loads and exports every symbol include/hfmm_gpu.h declares."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hfmm_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hfmm_[a-z0-9_]+)\s*\(", src)))


def test_all_declared_symbols_exported(native):
    names = declared_symbols()
    assert len(names) >= 15
    for nm in names:
        assert hasattr(native, nm), nm
    from paper_2006_15367_b200 import _native
    assert set(_native.EXPORTED_SYMBOLS) == set(names)


def test_config_defaults(native):
    from paper_2006_15367_b200 import _native, RunConfig
    c = _native.RunConfigC()
    native.hfmm_run_config_default(ctypes.byref(c))
    d = RunConfig()
    assert (c.lambda_, c.digits, c.leaf_lambda, c.num_ranks, c.policy, c.top_level) == \
        (d.lambda_, d.digits, d.leaf_lambda, d.num_ranks, int(d.policy), d.top_level)
    assert c.buffer_limit == 2**64 - 1


def test_error_status_and_message(native):
    import paper_2006_15367_b200 as hb
    with pytest.raises(hb.InvalidArgument, match="no particles"):
        hb.build_setup(np.zeros((0, 3)), np.zeros(0, complex))
    setup = hb.build_setup(np.array([[0.1, 0.2, 0.3]]), np.ones(1, complex))
    with pytest.raises(hb.InvalidArgument, match="unknown array"):
        setup.array("no_such_array")


def test_no_cpu_fallback_without_device(native):
    """On a machine without a GPU the engine refuses loudly (no CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2006_15367_b200 as hb
    pos, q = hb.generate_inputs("cube", 1000, 1.0, 0)
    setup = hb.build_setup(pos, q)
    with pytest.raises(hb.NoDeviceError):
        hb.RankEngine(setup)
    with pytest.raises(hb.NoDeviceError):
        hb.direct_potential(pos, q, [0, 1])


def test_generator_matches_oracle(native, refo):
    import paper_2006_15367_b200 as hb
    for shape in ("cube", "sphere"):
        a = hb.generate_inputs(shape, 5000, 3.0, 17)
        b = refo.generate_inputs(shape, 5000, 3.0, 17)
        assert np.array_equal(a[0], b[0])
        assert np.array_equal(np.stack([a[1].real, a[1].imag], -1), b[1])
