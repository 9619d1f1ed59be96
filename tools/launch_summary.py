"""Per-launch table of an ncu --metrics CSV (dev tool): ms, DRAM GB, pipe %.
usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, k = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        e = k.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0].replace("void ", "").replace("hfmm_b200::", ""),
                                   "grid": d["Grid Size"]})
        try:
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            pass
tot = sum(x.get("gpu__time_duration.sum", 0) for x in k.values())
print(f"{'kernel':34s} {'grid':>14s} {'ms':>8s} {'share':>6s} {'GB':>7s} {'GB/s':>7s} {'fp64%':>6s} {'tens%':>6s}")
for x in k.values():
    t = x.get("gpu__time_duration.sum", 0)
    gb = (x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)) / 1e9
    print(f"{x['name'][:34]:34s} {x['grid']:>14s} {t / 1e6:8.3f} {100 * t / tot:5.1f}% {gb:7.3f} "
          f"{gb / (t / 1e9) if t else 0:7.0f} {x.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0):6.1f} "
          f"{x.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):6.1f}")
print(f"total {tot / 1e6:.3f} ms over {len(k)} launches")
