"""A/B of an engine variant selected by an environment variable read at
launch time: sequential-phase device times (CUDA events) and the potentials'
relative difference, on one BASELINE config.  Dev tool.

usage: python tools/leaf_ab.py cfg4 HFMM_L2T_V2 [reps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2006_15367_b200 as hb  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg, var = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
shape, n, ext, seed, digits = CONFIGS[cfg]
pos, q = hb.generate_inputs(shape, n, ext, seed)
setup = hb.build_setup(pos, q, hb.RunConfig(digits=digits, setup_device=1))
eng = hb.RankEngine(setup)
eng.set_overlap(False)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
out = {}
for label, on in (("A", False), ("B", True), ("A2", False), ("B2", True)):
    if on:
        os.environ[var] = "1"
    else:
        os.environ.pop(var, None)
    acc = {}
    for i in range(reps + 1):
        flush.zero_()
        torch.cuda.synchronize()
        r = eng.evaluate()
        if i:
            for k, v in r.phase_ms.items():
                acc[k] = acc.get(k, 0.0) + v / reps
    out[label] = r.potentials
    print(label, f"{var}={'1' if on else 'unset'}", {k: round(v, 3) for k, v in acc.items()}, flush=True)
d = np.linalg.norm(out["A"] - out["B"]) / np.linalg.norm(out["A"])
print(f"rel diff A vs B: {d:.3e}")
