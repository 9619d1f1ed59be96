"""Per-launch table (ms, DRAM GB, FP64 / tensor pipe %) from an ncu --metrics CSV
(gpu__time_duration.sum, dram__bytes_{read,write}.sum, sm__pipe_{fp64,tensor}_cycles_active...).

usage: python tools/launch_list.py <launches.csv> [min_ms]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
min_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
hdr, k = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        e = k.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0].replace("void ", "").replace("hfmm_b200::", ""),
                                   "grid": d["Grid Size"], "block": d["Block Size"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
tot = 0.0
print(f"{'kernel':38s} {'grid':18s} {'block':14s} {'ms':>8s} {'GB':>7s} {'fp64%':>6s} {'tens%':>6s}")
for e in k.values():
    t = e["gpu__time_duration.sum"] / 1e6
    tot += t
    if t < min_ms:
        continue
    gb = (e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)) / 1e9
    print(f"{e['name'][:38]:38s} {e['grid']:18s} {e['block']:14s} {t:8.3f} {gb:7.2f} "
          f"{e.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0):6.1f} "
          f"{e.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):6.1f}")
print(f"total {tot:.3f} ms over {len(k)} launches (ncu serialises launches: compare shares, not absolutes)")
