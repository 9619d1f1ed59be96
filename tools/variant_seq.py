"""Sequential-phase device times (CUDA events, L2 flushed) of one BASELINE
config with an alternative build of the native library (dev tool).

usage: python tools/variant_seq.py <lib.so | base> cfg4 [reps]
"""
import os
import sys

sys.path.insert(0, ".")
from paper_2006_15367_b200 import _native  # noqa: E402

if sys.argv[1] != "base":
    _native.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

import paper_2006_15367_b200 as hb  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
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
print({k: round(v, 3) for k, v in acc.items()}, flush=True)
