"""Per-launch table from an ncu --metrics gpu__time_duration.sum CSV (second half = last evaluation)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
half = data[int(len(data) * (1 - frac)):]
tot = sum(float(d["Metric Value"]) for d in half)
for d in half:
    v = float(d["Metric Value"])
    print(f"{d['Kernel Name'].split('(')[0]:22s} grid={d['Grid Size']:16s} {v / 1e6:8.3f} ms {100 * v / tot:5.1f}%")
print(f"total {tot / 1e6:.3f} ms over {len(half)} launches")
