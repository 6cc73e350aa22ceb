"""Hot instruction footprint of a profiled kernel (ncu source page CSV +
nvdisasm -g listing): how many SASS instructions execute at least X times
per local_search iteration, attributed to source lines."""
import csv
import re
import sys

import numpy as np

sass, src_csv, fn, iters = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
lines = open(sass).read().split("\n")
start = [i for i, l in enumerate(lines) if (".text." + fn) in l and "section" in l][0]
cur = None
off2line = {}
for l in lines[start + 1:]:
    if ".section" in l and ".text." in l:
        break
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
hdr, data = rows[hi], rows[hi + 1:]
ie = hdr.index("Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
base = min(int(r[0], 16) for r in data)
ex = np.array([float(r[ie] or 0) for r in data])
print("instructions", len(ex), "executed", int((ex > 0).sum()))
for thr in [0.25, 0.5, 1, 2, 4]:
    sel = ex >= thr * iters
    print(f"  >= {thr}/iter: {sel.sum()} instr ({sel.sum() * 16 / 1024:.1f} KB) covering {ex[sel].sum() / ex.sum() * 100:.1f}%")
agg = {}
for r, e in zip(data, ex):
    if e < 0.5 * iters:
        continue
    k = off2line.get(int(r[0], 16) - base, ("?", 0))
    a = agg.setdefault(k, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += e
    a[2] += float(r[ws] or 0)
print("largest hot source lines (static instructions, executions per iteration):")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[5]) if len(sys.argv) > 5 else 25]:
    print(f"  {k[0]:12s} {k[1]:5d}  n={v[0]:4d}  exec/iter={v[1] / iters:8.1f}")
