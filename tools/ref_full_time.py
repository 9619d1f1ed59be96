"""Times the reference (oracle/_ref, the unmodified reference sources) on a
WHOLE BASELINE configuration on this host: build_setup, then one
evaluate_with_setup (traversal.cpp:790-817) with num_ranks = host cores and
the Threaded scheduler.  Writes a JSON record.

    python tools/ref_full_time.py cfg4 gpurun_out/r02_ref_full_cfg4.json
"""
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS  # noqa: E402
from oracle import ref  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    cfg, out = sys.argv[1], sys.argv[2]
    shape, n, ext, seed, digits = CONFIGS[cfg]
    cores = os.cpu_count() or 1
    pos, q = ref.generate_inputs(shape, n, ext, seed)
    t0 = time.time()
    rs = ref.RefSetup(pos, q, ref.config(digits=digits, num_ranks=cores, scheduler=2))
    setup_s = time.time() - t0
    t0 = time.time()
    _, sec, _ = rs.evaluate()
    wall = time.time() - t0
    rec = {"config": cfg, "n": n, "host": "GPU box host CPU", "cpu_model": cpu_model(), "host_cores": cores,
           "eval_ranks": cores, "scheduler": "Threaded", "setup_s": setup_s, "eval_wall_s": wall,
           "targets_per_s": n / wall,
           "phase_sec_max_rank": dict(zip(["setup", "c2m", "m2m", "m2l", "l2l", "l2o", "near"], sec.tolist())),
           "fft_backend": "oracle/shim/fftw_shim.cpp (mixed-radix, FFTW3 absent)",
           "generated_by": "tools/ref_full_time.py"}
    json.dump(rec, open(out, "w"), indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
