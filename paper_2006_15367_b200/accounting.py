"""Algorithmic work per evaluation phase (SURVEY.md section 8(d) conventions).

Used by bench.py's roofline / per-phase table and by the ledger reporting in
paper_2006_15367_b200.io.  Flop conventions follow the reference's charges
(proj/include/hfmm/operators.hpp:16-20): 8 per (far pair x sample) for M2L,
12 per (particle x leaf sample) for C2M and L2T, 20 per near pair; M2M / L2L
use the dense separable count 8 (n_c^2 n_p + (n_p/2)(2 n_c)(2 n_p)) + 8 S_p
per child.  Bytes are each stage's inputs read once and outputs written once.
"""
from __future__ import annotations

import numpy as np


def m2l_accounting(setup):
    """Algorithmic flops / compulsory bytes of the M2L phase."""
    flops = 0.0
    nbytes = 0.0
    for lvl in range(setup.top_level, setup.levels + 1):
        _, nt, nphi = setup.sampling(lvl)
        S = nt * nphi
        far_off = setup.array(f"L{lvl}.far_off", np.uint64)
        nodes = far_off.size - 1
        pairs = float(far_off[-1])
        flops += 8.0 * pairs * S
        used = 316 if pairs > 0 else 0
        nbytes += nodes * S * 32.0 + used * S * 16.0
    return flops, nbytes


def phase_accounting(setup):
    """Algorithmic flops and compulsory bytes per phase.

    C2M / L2T: 12 flops per (particle, leaf sample) entry; M2M / L2L: the dense
    separable count 8 (n_c^2 n_p + (n_p/2)(2 n_c)(2 n_p)) + 8 S_p per child;
    M2L: 8 per (far pair, sample); P2P: 20 per near particle pair.  Bytes are
    each stage's inputs read once and outputs written once.
    """
    L, top = setup.levels, setup.top_level
    S = {l: setup.sampling(l)[1] * setup.sampling(l)[2] for l in range(top, L + 1)}
    n_t = {l: setup.sampling(l)[1] for l in range(top, L + 1)}
    nodes = {l: setup.array(f"L{l}.far_off", np.uint64).size - 1 for l in range(top, L + 1)}
    leaf_start = setup.array("leaf_start", np.uint64).astype(np.int64)
    n = float(leaf_start[-1])
    entries = n * S[L]
    acc = {"C2M": (12.0 * entries, n * 40.0 + nodes[L] * S[L] * 16.0),
           "L2T": (12.0 * entries, n * 56.0 + nodes[L] * S[L] * 16.0)}
    f_mm = b_m2m = b_l2l = 0.0
    for l in range(top, L):
        nc, np_ = n_t[l + 1], n_t[l]
        f_mm += nodes[l + 1] * (8.0 * (nc * nc * np_ + (np_ // 2) * 2 * nc * 2 * np_) + 8.0 * S[l])
        b_m2m += nodes[l + 1] * S[l + 1] * 16.0 + nodes[l] * S[l] * 16.0
        b_l2l += 2 * nodes[l + 1] * S[l + 1] * 16.0 + nodes[l] * S[l] * 16.0
    acc["M2M"] = (f_mm, b_m2m)
    acc["L2L"] = (f_mm, b_l2l)
    acc["M2L"] = m2l_accounting(setup)
    sizes = np.diff(leaf_start).astype(np.float64)
    near_off = setup.array("near_off", np.uint64).astype(np.int64)
    codes = setup.array(f"L{L}.codes", np.uint64)
    near = np.searchsorted(codes, setup.array("near", np.uint64))
    per_leaf = np.add.reduceat(sizes[near], near_off[:-1]) if near.size else np.zeros_like(sizes)
    per_leaf[np.diff(near_off) == 0] = 0.0
    pairs = float((sizes * per_leaf).sum())
    acc["Near"] = (20.0 * pairs, n * 56.0)
    return acc, pairs
