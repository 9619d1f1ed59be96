"""SASS opcode counts per kernel of the built library (cuobjdump -sass).

usage: python tools/sass_summary.py [lib.so] > profiles/<name>.txt
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2006_15367_b200/_lib/libhfmm_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
dem = {}
kern, counts = None, collections.OrderedDict()
keep = ["DMMA", "DFMA", "DADD", "DMUL", "MUFU", "LDGSTS", "UBLKCP", "UBLKPF", "SYNCS", "UTMALDG", "LDS", "LDG", "STG", "SHFL", "BAR"]
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
    if m and kern:
        counts[kern]["_n"] += 1
        op = m.group(1)
        for k in keep:
            if op.startswith(k):
                counts[kern][k] += 1
                break
names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"# cuobjdump -sass {lib}: SASS opcodes per kernel (static counts)")
print("# DMMA = FP64 tensor (mma.sync m8n8k4 f64; B200 has no tcgen05 f64 kind); UBLKCP = cp.async.bulk global->shared with")
print("# mbarrier completion (bulk-copy / TMA engine), UBLKPF = cp.async.bulk.prefetch.L2, SYNCS = mbarrier ops, LDGSTS = cp.async")
rows = sorted(zip(names, counts.values()), key=lambda kv: -kv[1]["_n"])
for name, c in rows:
    if c["_n"] < 64:
        continue
    d = {k: c[k] for k in keep if c[k]}
    print(f"{name[:70]:70s} instr={c['_n']:6d} {d}")
