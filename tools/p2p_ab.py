"""A/B of the near-field kernels on one BASELINE config (dev tool).

usage: python tools/p2p_ab.py cfg3 [lib.so]
For the library (default: the in-tree one) and each P2P mode (HFMM_P2P_V1
set / unset) builds an engine, runs a full evaluation (potentials compared
with the first run), then times the near phase alone (wall clock around
run_phase(Near) + synchronize, median of 5).
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2006_15367_b200 as hb  # noqa: E402
from paper_2006_15367_b200 import _native  # noqa: E402
from paper_2006_15367_b200.hfmm import Phase  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
libs = sys.argv[2:3] or [None]
if libs[0] is not None:
    _native.LIB_PATH = os.path.abspath(libs[0])
shape, n, ext, seed, digits = CONFIGS[cfg]
pos, q = hb.generate_inputs(shape, n, ext, seed)
ref = None
for lib in libs:
    setup = hb.build_setup(pos, q, hb.RunConfig(digits=digits))
    for mode in ("v1", "v2"):
        if mode == "v1":
            os.environ["HFMM_P2P_V1"] = "1"
        else:
            os.environ.pop("HFMM_P2P_V1", None)
        eng = hb.RankEngine(setup)
        res = eng.evaluate()
        pot = res.potentials
        if ref is None:
            ref = pot
        rel = np.linalg.norm(pot - ref) / np.linalg.norm(ref)
        ts = []
        for _ in range(5):
            eng.synchronize()
            t0 = time.perf_counter()
            eng.run_phase(Phase.Near)
            eng.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"{cfg} lib={lib or 'in-tree'} {mode}: near {np.median(ts):8.3f} ms (min {min(ts):.3f})  "
              f"eval total {res.phase_ms.get('total', 0):.3f} ms  rel_vs_first {rel:.2e}", flush=True)
        eng.close()
