"""Reference fixtures for the FULL BASELINE configurations 2-5.

Runs the UNMODIFIED reference (oracle/_ref/libhfmm_ref.so, built from
/root/reference by oracle/Makefile) on each whole configuration on the CPU
of the build container and commits what the GPU parity tests need, without
the reference at run time:

  full_cfgN.npz   sub_idx     -- fixed subsample of target indices (seeded)
                  sub_pot     -- reference potentials there (complex128)
                  direct_obs  -- direct-sum targets i*(N/1000), i < 1000
                  direct      -- direct_potential there (kernel.cpp:16-41)
  full_cfgN.json  sha256 of the full reference potential vector, the
                  reference's relative L2 error against the direct sum,
                  the reference wall time / per-phase seconds on this host
                  (core count stated), and sha256 of every setup array of
                  build_setup at 1 and 8 ranks (traversal.cpp:66-238).

The reference evaluation follows BASELINE.md §4: build_setup, then
evaluate_with_setup (traversal.cpp:790-817) with num_ranks = host cores and
the Threaded scheduler.

    python tests/golden/make_full_golden.py cfg2 [cfg3 cfg4 cfg5]
"""
from __future__ import annotations

import gc
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from oracle import ref  # noqa: E402
from make_golden import setup_array_names  # noqa: E402

# name: (shape, n, extent, seed, digits) -- BASELINE.json configs[1..4]
CONFIGS = {
    "cfg2": ("cube", 1_000_000, 16.0, 1, 6.0),
    "cfg3": ("sphere", 4_000_000, 8.0, 2, 3.0),
    "cfg4": ("cube", 16_000_000, 32.0, 3, 3.0),
    "cfg5": ("sphere", 64_000_000, 32.0, 4, 4.0),
}
SUBSAMPLE = 32768
HASH_RANKS = (1, 8)


def subsample_indices(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(1000 + seed)
    return np.sort(rng.choice(n, size=min(n, SUBSAMPLE), replace=False)).astype(np.int64)


def direct_indices(n: int) -> np.ndarray:
    return (np.arange(1000, dtype=np.int64) * (n // 1000)).astype(np.int64)


def rel_l2(a, b) -> float:
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run(name: str, eval_ranks: int) -> None:
    shape, n, ext, seed, dig = CONFIGS[name]
    t0 = time.time()
    pos, q = ref.generate_inputs(shape, n, ext, seed)
    out = {"config": name, "shape": shape, "n": n, "extent": ext, "seed": seed, "digits": dig,
           "host_cores": os.cpu_count(), "eval_ranks": eval_ranks, "scheduler": "Threaded",
           "fft_backend": "oracle/shim/fftw_shim.cpp (mixed-radix, FFTW3 absent)",
           "generated_by": "tests/golden/make_full_golden.py", "setup_sha256": {}}
    for ranks in HASH_RANKS:
        if ranks == eval_ranks:
            continue
        ts = time.time()
        rs = ref.RefSetup(pos, q, ref.config(digits=dig, num_ranks=ranks))
        out[f"setup_s_r{ranks}"] = time.time() - ts
        out["setup_sha256"][f"r{ranks}"] = {nm: hashlib.sha256(rs.array(nm).tobytes()).hexdigest()
                                             for nm in setup_array_names(rs.levels, rs.top_level)}
        del rs
        gc.collect()
    ts = time.time()
    rs = ref.RefSetup(pos, q, ref.config(digits=dig, num_ranks=eval_ranks, scheduler=2))
    out[f"setup_s_r{eval_ranks}"] = time.time() - ts
    out["levels"] = rs.levels
    out["num_leaves"] = rs.num_leaves
    if eval_ranks in HASH_RANKS:
        out["setup_sha256"][f"r{eval_ranks}"] = {nm: hashlib.sha256(rs.array(nm).tobytes()).hexdigest()
                                                 for nm in setup_array_names(rs.levels, rs.top_level)}
    print(f"[{name}] setup done, {time.time() - t0:.1f}s", flush=True)
    te = time.time()
    pot, sec, fl = rs.evaluate()
    out["eval_wall_s"] = time.time() - te
    out["phase_sec_max_rank"] = dict(zip(["setup", "c2m", "m2m", "m2l", "l2l", "l2o", "near"], sec.tolist()))
    out["phase_flops"] = fl.tolist()
    out["targets_per_s"] = n / out["eval_wall_s"]
    print(f"[{name}] evaluate {out['eval_wall_s']:.1f}s", flush=True)
    del rs
    gc.collect()
    pv = np.ascontiguousarray(np.stack([pot.real, pot.imag], -1))
    out["pot_sha256"] = hashlib.sha256(pv.tobytes()).hexdigest()
    out["pot_norm"] = float(np.linalg.norm(pot))
    sub = subsample_indices(n, seed)
    obs = direct_indices(n)
    td = time.time()
    d = ref.direct(pos, q, obs, nthreads=os.cpu_count() or 8)
    out["direct_s"] = time.time() - td
    out["ref_err_vs_direct"] = rel_l2(pot[obs], d)
    out["subsample"] = int(sub.size)
    np.savez_compressed(os.path.join(HERE, f"full_{name}.npz"), sub_idx=sub, sub_pot=pot[sub],
                        direct_obs=obs, direct=d)
    with open(os.path.join(HERE, f"full_{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(f"[{name}] done: ref err vs direct {out['ref_err_vs_direct']:.3e}, total {time.time() - t0:.1f}s",
          flush=True)


def main():
    names = sys.argv[1:] or list(CONFIGS)
    ranks = int(os.environ.get("REF_RANKS", os.cpu_count() or 8))
    for nm in names:
        run(nm, ranks)


if __name__ == "__main__":
    main()
