"""Summarise an ncu source page (SASS) CSV: top stall-sampled instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
js = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) <= js:
        continue
    try:
        data.append((float(r[js]), r[0], r[1].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for v, a, s in sorted(data, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}%  {a[-5:]}  {s}")
# coarse split by instruction class
cls = {}
for v, a, s in data:
    op = s.split()[0] if s else "?"
    if op.startswith("@"):
        op = s.split()[1]
    op = op.split(".")[0]
    cls[op] = cls.get(op, 0) + v
print("by opcode:", {k: round(100 * v / tot, 1) for k, v in sorted(cls.items(), key=lambda x: -x[1])[:12]})
