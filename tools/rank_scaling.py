"""Per-rank device time of the distributed evaluation, ranks emulated one
after another on ONE GPU (dev tool; no kernel waits on another rank).

usage: python tools/rank_scaling.py cfg2 1 2 4 8

For each rank count P: builds the P-rank setup (bit-exact partition), runs
every rank's engine through the same phase sequence as the NCCL driver
(ghost exchange, C2M, M2M, multipole exchange, M2L, L2L, L2T, near) with the
exchanges done by device copies, and times each rank's phases with CUDA
events on its own stream.  Prints, per P, the max-over-ranks compute time
per evaluation and its phase split -- the compute part of a P-GPU strong-
scaling run (the NVLink transfer time of the exchanges is not included; the
exchanged bytes are printed).  This is a model input, not a bench value.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2006_15367_b200 as hb  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = sys.argv[1]
counts = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8]
shape, n, ext, seed, digits = CONFIGS[cfg]
pos, q = hb.generate_inputs(shape, n, ext, seed)
PH = [hb.Phase.C2M, hb.Phase.M2M, hb.Phase.M2L, hb.Phase.L2L, hb.Phase.L2T, hb.Phase.Near]
NAMES = ["C2M", "M2M", "M2L", "L2L", "L2T", "Near"]

for P in counts:
    setup = hb.build_setup(pos, q, hb.RunConfig(digits=digits, num_ranks=P, setup_device=1))
    engs = [hb.RankEngine(setup, r, 0) for r in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    for e, st in zip(engs, streams):
        e.set_stream(st.cuda_stream)
        e.set_intensities(q)
    xbytes = 0

    def exchange(kind):
        global xbytes
        if P == 1:
            return
        if kind == 0:
            for e in engs:
                e.exchange_begin(0)
        bufs = {}
        for r, e in enumerate(engs):
            for p in range(P):
                if p != r:
                    s, _ = e.exchange_sizes(kind, p)
                    if s:
                        bufs[r, p] = torch.empty(s, dtype=torch.float64, device="cuda")
                        e.pack(kind, p, bufs[r, p])
                        xbytes += 8 * s
            e.synchronize()
        for p, e in enumerate(engs):
            for r in range(P):
                if (r, p) in bufs:
                    e.unpack(kind, r, bufs[r, p])
            e.synchronize()

    per_rank = []
    for it in range(3):  # warm-up + 2 timed
        xbytes = 0
        times = [dict.fromkeys(NAMES, 0.0) for _ in range(P)]
        exchange(1)
        for r, (e, st) in enumerate(zip(engs, streams)):
            for ph, nm in zip(PH[:2], NAMES[:2]):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                e.run_phase(ph)
                b.record(st)
                b.synchronize()
                times[r][nm] += a.elapsed_time(b)
        exchange(0)
        for r, (e, st) in enumerate(zip(engs, streams)):
            for ph, nm in zip(PH[2:], NAMES[2:]):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                e.run_phase(ph)
                b.record(st)
                b.synchronize()
                times[r][nm] += a.elapsed_time(b)
        if it > 0:
            per_rank.append(times)
    tot = [np.mean([sum(t[r].values()) for t in per_rank]) for r in range(P)]
    worst = int(np.argmax(tot))
    split = {nm: round(float(np.mean([t[worst][nm] for t in per_rank])), 3) for nm in NAMES}
    print(f"{cfg} P={P}: max-over-ranks compute {max(tot):.3f} ms (rank {worst}; min {min(tot):.3f}) "
          f"phases {split} exchanged {xbytes / 1e9:.3f} GB/eval", flush=True)
    for e in engs:
        e.close()
    del engs
    torch.cuda.empty_cache()
