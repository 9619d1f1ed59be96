"""Per-kernel table (per evaluation) from an ncu launch list of bench.py, plus
the per-phase DRAM traffic used by bench.py's roofline.traffic.

usage: python tools/summarize_launches.py gpurun_out/bench_launches.csv profiles/<name>.txt [cfgN]
"""
import collections
import csv
import json
import sys

src, out = sys.argv[1], sys.argv[2]
cfg = sys.argv[3] if len(sys.argv) > 3 else "cfg4"
rows = list(csv.reader(open(src)))
hdr, k = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        e = k.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0].replace("void ", ""), "grid": d["Grid Size"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
ks = list(k.values())
n_eval = sum(1 for x in ks if x["name"].split("::")[-1].startswith("k_c2m"))
agg = collections.OrderedDict()
for x in ks:
    a = agg.setdefault((x["name"], x["grid"]), [0, 0.0, 0.0])
    a[0] += 1
    a[1] += x["gpu__time_duration.sum"]
    a[2] += x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
tot = sum(v[1] for v in agg.values()) / n_eval
lines = ["# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none",
         f"#   python bench.py --config {cfg} --steps 2 --warmup 3 --no-cpu-baseline   ({len(ks)} launches = {n_eval} evaluations)",
         "# per-evaluation averages; ncu serialises launches (cold caches), so compare shares, not absolutes",
         f"{'kernel':34s} {'grid':16s} {'ms/eval':>8s} {'share':>6s} {'GB/eval':>8s} {'GB/s':>7s}"]
for (nm, gr), (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    te, be = t / n_eval / 1e6, b / n_eval / 1e9
    lines.append(f"{nm[:34]:34s} {gr:16s} {te:8.3f} {100 * te / (tot / 1e6):5.1f}% {be:8.3f} {be / max(te, 1e-9) * 1e3:7.0f}")
lines.append(f"total {tot / 1e6:.3f} ms per evaluation (serialised)")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:24]))
traffic = {}
for key, pre in (("M2L", "k_m2l"), ("M2M", "k_m2m"), ("L2L", "k_l2l")):
    traffic[key] = sum(b for (nm, gr), (c, t, b) in agg.items() if nm.split("::")[-1].startswith(pre)) / n_eval
traffic["_note"] = f"DRAM bytes (read+write) per evaluation summed over the phase's launches, {cfg}, from {out}"
try:
    allt = json.load(open("profiles/ncu_traffic.json"))
except (OSError, ValueError):
    allt = {}
allt[cfg] = traffic
json.dump(allt, open("profiles/ncu_traffic.json", "w"), indent=1)
