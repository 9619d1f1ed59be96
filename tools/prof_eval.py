"""Runs `reps` device-resident evaluations of a BASELINE config (profiling driver)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2006_15367_b200 as hb
from bench import CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
shape, n, ext, seed, digits = CONFIGS[cfg]
pos, q = hb.generate_inputs(shape, n, ext, seed)
setup = hb.build_setup(pos, q, hb.RunConfig(digits=digits, setup_device=1))
eng = hb.RankEngine(setup)
for _ in range(reps):
    r = eng.evaluate()
    print({k: round(v, 3) for k, v in r.phase_ms.items()}, flush=True)
