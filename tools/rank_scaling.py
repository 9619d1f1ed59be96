"""Per-rank device time of the distributed evaluation, ranks emulated one
after another on ONE GPU (dev tool; no kernel waits on another rank).

usage: python tools/rank_scaling.py cfg4 1 2 4 8

For each rank count P: builds the P-rank setup (bit-exact partition), runs
every rank's engine through the distributed schedule
(paper_2006_15367_b200.distributed.schedule: ghosts, C2M, M2M, plural
reduce-scatter, T build, per-level sliced M2L halo + M2L, per-level plural
gather + L2L, L2T, near) with the exchanges done by device copies, and times
each rank's compute stages with CUDA events on its own stream.  Prints, per P,
the max-over-ranks compute time per evaluation, its phase split and the bytes
each exchange kind moved -- the compute part of a P-GPU strong-scaling run
(NVLink transfer time is not included).  This is a model input, not a bench
value.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2006_15367_b200 as hb  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2006_15367_b200.distributed import schedule  # noqa: E402

cfg = sys.argv[1]
counts = [int(a) for a in sys.argv[2:] if not a.startswith("--")] or [1, 2, 4, 8]
shape, n, ext, seed, digits = CONFIGS[cfg]
pos, q = hb.generate_inputs(shape, n, ext, seed)
KN = {0: "halo", 1: "ghost", 2: "reduce", 3: "gather"}

for P in counts:
    setup = hb.build_setup(pos, q, hb.RunConfig(digits=digits, num_ranks=P, setup_device=1))
    engs = [hb.RankEngine(setup, r, 0) for r in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    for e, st in zip(engs, streams):
        e.set_stream(st.cuda_stream)
        e.set_intensities(q)
    # the near field runs inside the Near stage here (no side-stream launch),
    # so its time is charged to that stage of its own rank
    sched = [st for st in schedule(setup.top_level, setup.levels) if st[1] != hb.Phase.NearStart or st[0] != "run"]
    per_rank, xb = [], {}
    for it in range(3):  # warm-up + 2 timed
        xb = dict.fromkeys(KN.values(), 0)
        times = [{} for _ in range(P)]
        lvl_times = [{} for _ in range(P)]
        for what, a, lvl in sched:
            if what == "run":
                for r, (e, st) in enumerate(zip(engs, streams)):
                    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    ev0.record(st)
                    e.run_phase(a) if lvl < 0 else e.run_level(a, lvl)
                    ev1.record(st)
                    ev1.synchronize()
                    nm = hb.Phase(a).name
                    times[r][nm] = times[r].get(nm, 0.0) + ev0.elapsed_time(ev1)
                    if lvl >= 0:
                        lvl_times[r][f"{nm}@{lvl}"] = round(ev0.elapsed_time(ev1), 3)
            elif P > 1:
                bufs = {}
                for r, e in enumerate(engs):
                    for p in range(P):
                        if p != r:
                            s, _ = e.exchange_sizes(a, p, lvl)
                            if s:
                                bufs[r, p] = torch.empty(s, dtype=torch.float64, device="cuda")
                                e.pack(a, p, bufs[r, p], lvl)
                                xb[KN[a]] += 8 * s
                    e.synchronize()
                for p, e in enumerate(engs):
                    for r in range(P):
                        if (r, p) in bufs:
                            e.unpack(a, r, bufs[r, p], lvl)
                    e.synchronize()
        if it > 0:
            per_rank.append(times)
    tot = [np.mean([sum(t[r].values()) for t in per_rank]) for r in range(P)]
    worst = int(np.argmax(tot))
    split = {nm: round(float(np.mean([t[worst][nm] for t in per_rank])), 3) for nm in per_rank[0][worst]}
    print(f"{cfg} P={P}: max-over-ranks compute {max(tot):.3f} ms (rank {worst}; min {min(tot):.3f}) "
          f"phases {split} exchanged GB/eval {({k: round(v / 1e9, 4) for k, v in xb.items()})}", flush=True)
    if "--levels" in sys.argv:
        print(f"   per-level stages of rank {worst} (last pass): {lvl_times[worst]}", flush=True)
    for e in engs:
        e.close()
    del engs
    torch.cuda.empty_cache()
