"""Potentials of an alternative build against the in-tree build on one BASELINE
config (relative L2), plus its sequential-phase times (dev tool).

usage: python tools/variant_check.py <lib.so> cfg3 [reps]
Runs the base build in a child process first (the native library is loaded once
per process) and compares through a .npy file under gpurun_out/.
"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, ".")
lib, cfg = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
out = f"gpurun_out/_pot_{cfg}_{os.path.basename(lib)}.npy"
if lib != "base" and not os.environ.get("_VC_CHILD"):
    base = f"gpurun_out/_pot_{cfg}_base.npy"
    if not os.path.exists(base):
        subprocess.run([sys.executable, __file__, "base", cfg, "1"], check=True, env={**os.environ, "_VC_CHILD": "1"})
from paper_2006_15367_b200 import _native  # noqa: E402

if lib != "base":
    _native.LIB_PATH = os.path.abspath(lib)
import torch  # noqa: E402

import paper_2006_15367_b200 as hb  # noqa: E402
from bench import CONFIGS  # noqa: E402

shape, n, ext, seed, digits = CONFIGS[cfg]
pos, q = hb.generate_inputs(shape, n, ext, seed)
setup = hb.build_setup(pos, q, hb.RunConfig(digits=digits, setup_device=1))
eng = hb.RankEngine(setup)
eng.set_overlap(False)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
acc = {}
for i in range(reps + 1):
    flush.zero_()
    torch.cuda.synchronize()
    r = eng.evaluate()
    if i:
        for k, v in r.phase_ms.items():
            acc[k] = acc.get(k, 0.0) + v / reps
pot = np.asarray(r.potentials)
msg = {k: round(v, 3) for k, v in acc.items()}
if lib == "base":
    np.save(out, pot)
else:
    ref = np.load(f"gpurun_out/_pot_{cfg}_base.npy")
    msg["rel_l2_vs_base"] = float(np.linalg.norm(pot - ref) / np.linalg.norm(ref))
print(lib, cfg, msg, flush=True)
