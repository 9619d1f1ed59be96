"""A/B of an engine switch read from the environment at engine creation (dev tool).

usage: python tools/ab_env.py cfg2 HFMM_LEAF_V1 [HFMM_P2P_V1 NAME=VALUE ...]
For "baseline" (none of the variables set) and each variable set alone:
builds an engine, runs sequential-phase evaluations (set_overlap off, so each
phase's events time its own kernels), prints the median per-phase ms of 3
and the relative L2 difference of the potentials against the baseline.
"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2006_15367_b200 as hb  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = sys.argv[1]
envs = sys.argv[2:]
shape, n, ext, seed, digits = CONFIGS[cfg]
pos, q = hb.generate_inputs(shape, n, ext, seed)
setup = hb.build_setup(pos, q, hb.RunConfig(digits=digits, setup_device=1))
ref = None
for var in [None] + envs:
    for e in envs:
        os.environ.pop(e.split("=")[0], None)
    if var:
        name, _, val = var.partition("=")
        os.environ[name] = val or "1"
    eng = hb.RankEngine(setup)
    eng.set_overlap(False)
    runs = []
    for _ in range(4):
        res = eng.evaluate()
        runs.append(res.phase_ms)
    pot = res.potentials
    if ref is None:
        ref = pot
    rel = np.linalg.norm(pot - ref) / np.linalg.norm(ref)
    med = {k: float(np.median([r[k] for r in runs[1:]])) for k in runs[0]}
    print(f"{cfg} {var or 'baseline':16s} rel {rel:.2e} " + " ".join(f"{k}={v:.3f}" for k, v in med.items()),
          flush=True)
    eng.close()
