"""Host vs device setup wall time on BASELINE configs, and byte equality of
every setup array (dev tool).  usage: python tools/setup_time.py cfg2 cfg4"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2006_15367_b200 as hb  # noqa: E402
from bench import CONFIGS  # noqa: E402
from conftest import setup_array_names  # noqa: E402

for cfg in sys.argv[1:]:
    shape, n, ext, seed, digits = CONFIGS[cfg]
    pos, q = hb.generate_inputs(shape, n, ext, seed)
    out = {}
    for dev in (1, 0):
        t = time.perf_counter()
        out[dev] = hb.build_setup(pos, q, hb.RunConfig(digits=digits, setup_device=dev))
        print(f"{cfg} setup_device={dev}: {time.perf_counter() - t:.3f} s", flush=True)
    a, b = out[0], out[1]
    bad = [nm for nm in setup_array_names(a.levels, a.top_level) if not np.array_equal(a.array(nm), b.array(nm))]
    print(f"{cfg} arrays differing: {bad}", flush=True)
