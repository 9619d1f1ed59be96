"""hfmm_setup_import: the engine's setup taken from an EXISTING GlobalSetup
(traversal.hpp:93-118) instead of re-running build_setup.

The reference's own build_setup output (oracle/_ref, the flat arrays its
GlobalSetup flattens to) is imported through the C ABI; the imported setup
must equal hfmm_setup_build's byte for byte, for 1 and several ranks, and the
import must reject inconsistent arrays with the reference's exception types.
On the GPU the imported setup evaluates to the reference's potentials.
"""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import rel_l2, setup_array_names

CASES = [("cube", 20_000, 3.0, 31, 3.0, 1), ("sphere", 30_000, 2.0, 32, 4.0, 3), ("cube", 100_000, 4.0, 0, 3.0, 8)]


def _rank_names(levels, top, ranks):
    out = []
    for r in range(ranks):
        for l in range(top, levels + 1):
            out += [f"R{r}.held.L{l}", f"R{r}.halo.L{l}"]
        for p in range(ranks):
            if p != r:
                out += [f"R{r}.{d}{k}.{p}" for d in ("send", "recv") for k in (0, 2, 3)]
    return out


def _import(hb, arrays: dict, cfg):
    from paper_2006_15367_b200 import _native
    L = _native.lib()
    im = ctypes.c_void_p()
    c = cfg.to_c()
    _native.check(L.hfmm_setup_import_begin(ctypes.byref(c), ctypes.byref(im)))
    for name, a in arrays.items():
        a = np.ascontiguousarray(a)
        _native.check(L.hfmm_setup_import_put(im, name.encode(), a.ctypes.data if a.size else None, a.nbytes))
    h = ctypes.c_void_p()
    _native.check(L.hfmm_setup_import_end(im, ctypes.byref(h)))
    return hb.GlobalSetup(h, cfg, int(arrays["meta_i64"].view(np.int64)[3]))


@pytest.mark.parametrize("case", CASES)
def test_import_reference_setup_is_bit_exact(case, native, refo):
    import paper_2006_15367_b200 as hb
    shape, n, ext, seed, dig, ranks = case
    pos, q2 = refo.generate_inputs(shape, n, ext, seed)
    rs = refo.RefSetup(pos, q2, refo.config(digits=dig, num_ranks=ranks))
    names = setup_array_names(rs.levels, rs.top_level)
    cfg = hb.RunConfig(digits=dig, num_ranks=ranks)
    imported = _import(hb, {nm: rs.array(nm) for nm in names}, cfg)
    built = hb.build_setup(pos, q2[:, 0] + 1j * q2[:, 1], cfg)
    for nm in names + _rank_names(rs.levels, rs.top_level, ranks):
        assert np.array_equal(imported.array(nm), built.array(nm)), nm


def test_import_rejects_inconsistent_arrays(native):
    import paper_2006_15367_b200 as hb
    pos, q = hb.generate_inputs("cube", 5000, 2.0, 33)
    cfg = hb.RunConfig()
    s = hb.build_setup(pos, q, cfg)
    arrays = {nm: s.array(nm) for nm in setup_array_names(s.levels, s.top_level)}
    ok = _import(hb, arrays, cfg)
    assert ok.num_leaves == s.num_leaves
    bad = dict(arrays)
    del bad["near"]
    with pytest.raises(hb.InvalidArgument):
        _import(hb, bad, cfg)
    bad = dict(arrays)
    lo = bad["leaf_start"].view(np.uint64).copy()
    lo[-1] += 1
    bad["leaf_start"] = lo.view(np.uint8)
    with pytest.raises(hb.InvalidArgument):
        _import(hb, bad, cfg)
    bad = dict(arrays)
    far = bad[f"L{s.levels}.far"].view(np.uint64).copy()
    far[0] = np.uint64(2**40)
    bad[f"L{s.levels}.far"] = far.view(np.uint8)
    with pytest.raises(hb.OutOfRange):
        _import(hb, bad, cfg)
    with pytest.raises(hb.InvalidArgument):  # the partition's rank count must match the config
        _import(hb, arrays, hb.RunConfig(num_ranks=2))


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES[:2])
def test_imported_reference_setup_evaluates(case, native, refo):
    """Evaluation straight from the reference's GlobalSetup arrays (no
    build_setup on our side) matches evaluate_with_setup at 1e-10."""
    import paper_2006_15367_b200 as hb
    shape, n, ext, seed, dig, _ = case
    pos, q2 = refo.generate_inputs(shape, n, ext, seed)
    rs = refo.RefSetup(pos, q2, refo.config(digits=dig))
    setup = _import(hb, {nm: rs.array(nm) for nm in setup_array_names(rs.levels, rs.top_level)},
                    hb.RunConfig(digits=dig))
    want, _, _ = rs.evaluate()
    got = hb.evaluate_with_setup(setup).potentials
    assert rel_l2(got, want) < 1e-10
