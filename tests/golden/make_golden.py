"""Generates the golden fixtures in this directory from the UNMODIFIED
reference (oracle/_ref/libhfmm_ref.so, built from /root/reference by
oracle/Makefile).  Run from the repo root in the build container:

    python tests/golden/make_golden.py

Fixtures (small, committed):
  known_answers.json  -- frozen scalars of the reference's own tests plus
                         reference outputs of green / truncation_order /
                         make_quadrature / translation_operator;
  resample.npz        -- resample_circle and fft_interpolate / fft_anterpolate
                         outputs on seeded inputs;
  case_*.npz          -- seeded small MLFMA runs: reference potentials in
                         input order (the inputs are regenerated from the seed
                         with the frozen generator);
  setup_hashes.json   -- sha256 of every flat setup array of the reference's
                         build_setup for config 1 at 1 and 8 ranks.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

CASES = {
    # name: (shape, n, extent, seed, digits)
    "case_cube3": ("cube", 2000, 2.0, 11, 3.0),
    "case_sphere4": ("sphere", 3000, 1.0, 12, 4.0),
    "case_cube6": ("cube", 1500, 2.0, 13, 6.0),
}
HASH_CASES = {"cfg1_r1": ("cube", 100_000, 4.0, 0, 3.0, 1), "cfg1_r8": ("cube", 100_000, 4.0, 0, 3.0, 8)}


def setup_array_names(levels: int, top: int):
    names = ["meta_i64", "meta_f64", "particles", "original_index", "leaf_codes", "leaf_start",
             "rank_ranges", "splitters", "near_off", "near", "m2l_plan", "near_plan"]
    for l in range(top, levels + 1):
        for f in ("sampling", "theta_weight", "phi_weight", "codes", "centers", "users", "slices_off",
                  "slices", "child_off", "children", "interp_off", "interp", "far_off", "far"):
            names.append(f"L{l}.{f}")
    return names


def main():
    ka = {
        # proj/tests/test_kernel.cpp:29-34 and test_operators.cpp:83-97 (frozen in the reference tests)
        "green_k1_r3": [-0.02626036657630788, -0.0037433244753159963],
        "T_Lt0_k1_D2.5": [0.23938885764158263, -0.3204574462187735],
        # proj/tests/test_sphere_interp.cpp:64-67
        "trunc_d1_k1_dig3": 5,
    }
    g = ref.green(1.0, [3.0, 0.0, 0.0])
    ka["ref_green_k1_r3"] = [g.real, g.imag]
    ka["ref_trunc"] = {f"{d}_{k}_{dig}": ref.truncation_order(d, k, dig)
                       for d in (0.25 * 3 ** 0.5, 0.5 * 3 ** 0.5, 4 * 3 ** 0.5, 1.0)
                       for k in (1.0, 2 * np.pi) for dig in (3.0, 4.0, 6.0)}
    ka["ref_quad"] = {str(nt): ref.quadrature(nt, nt)[0].tolist() for nt in (6, 18, 26, 34)}
    T = ref.translation_operator(0, 2, 2, [2.5, 0, 0], 1.0, 1.0)
    ka["ref_T_Lt0"] = [T[0].real, T[0].imag]
    with open(os.path.join(HERE, "known_answers.json"), "w") as f:
        json.dump(ka, f, indent=1)

    rng = np.random.default_rng(2024)
    res = {}
    for ni, si, no, so in [(26, 0.0, 34, 0.0), (52, 0.5, 68, 0.5), (68, 0.5, 52, 0.5), (34, 0.0, 26, 0.0),
                           (18, 0.0, 28, 0.0), (36, 0.5, 56, 0.5)]:
        x = rng.standard_normal(ni) + 1j * rng.standard_normal(ni)
        res[f"circ_{ni}_{si}_{no}_{so}_in"] = x
        res[f"circ_{ni}_{si}_{no}_{so}_out"] = ref.resample_circle(x, no, si, so)
    for nc, npar in [(18, 28), (26, 34)]:
        x = rng.standard_normal(nc * nc) + 1j * rng.standard_normal(nc * nc)
        res[f"interp_{nc}_{npar}_in"] = x
        res[f"interp_{nc}_{npar}_out"] = ref.resample_grid(0, x, nc, nc, npar, npar)
        y = rng.standard_normal(npar * npar) + 1j * rng.standard_normal(npar * npar)
        res[f"anterp_{npar}_{nc}_in"] = y
        res[f"anterp_{npar}_{nc}_out"] = ref.resample_grid(1, y, npar, npar, nc, nc)
    np.savez_compressed(os.path.join(HERE, "resample.npz"), **res)

    for name, (shape, n, ext, seed, dig) in CASES.items():
        pos, q = ref.generate_inputs(shape, n, ext, seed)
        rs = ref.RefSetup(pos, q, ref.config(digits=dig))
        pot, _, _ = rs.evaluate()
        obs = np.arange(0, n, max(1, n // 200))
        d = ref.direct(pos, q, obs, nthreads=8)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), potentials=pot, direct_obs=obs, direct=d,
                            meta=np.array([n, ext, seed, dig, rs.levels]), shape=np.array(shape))

    hashes = {}
    for name, (shape, n, ext, seed, dig, ranks) in HASH_CASES.items():
        pos, q = ref.generate_inputs(shape, n, ext, seed)
        rs = ref.RefSetup(pos, q, ref.config(digits=dig, num_ranks=ranks))
        hashes[name] = {nm: hashlib.sha256(rs.array(nm).tobytes()).hexdigest()
                        for nm in setup_array_names(rs.levels, rs.top_level)}
    with open(os.path.join(HERE, "setup_hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
