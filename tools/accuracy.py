"""FMM-vs-direct accuracy and timing of one BASELINE config on the GPU (dev tool)."""
import sys
import time
import numpy as np
sys.path.insert(0, '.')
import paper_2006_15367_b200 as hb
from bench import CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
shape, n, ext, seed, digits = CONFIGS[cfg]
t0 = time.perf_counter()
pos, q = hb.generate_inputs(shape, n, ext, seed)
t1 = time.perf_counter()
setup = hb.build_setup(pos, q, hb.RunConfig(digits=digits))
t2 = time.perf_counter()
eng = hb.RankEngine(setup)
t3 = time.perf_counter()
res = eng.evaluate()
res = eng.evaluate()
obs = np.arange(1000) * (n // 1000)
d = hb.direct_potential(pos, q, obs)
err = np.linalg.norm(res.potentials[obs] - d) / np.linalg.norm(d)
print(f"{cfg}: N={n} levels={setup.levels} leaves={setup.num_leaves} gen {t1-t0:.1f}s setup {t2-t1:.1f}s "
      f"engine {t3-t2:.1f}s eval {res.phase_ms['total']:.2f} ms  rel err vs direct {err:.3e}", flush=True)
print({k: round(v, 3) for k, v in res.phase_ms.items()}, flush=True)
