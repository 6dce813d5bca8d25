#!/usr/bin/env python
"""Per-SASS-instruction stall reasons from an .ncu-rep (source page), grouped
by address range: python tools/ncu_stalls.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h, data = rows[hi], rows[hi + 1:]
si = h.index("Warp Stall Sampling (All Samples)")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
ri = [h.index(x) for x in reasons]
tot = {x: 0.0 for x in reasons}
for r in data:
    for x, i in zip(reasons, ri):
        tot[x] += float(r[i] or 0)
allv = sum(tot.values())
print("kernel-wide:", ", ".join(f"{k[6:]} {v / allv:.1%}" for k, v in
                                sorted(tot.items(), key=lambda kv: -kv[1]) if v / allv > 0.01))
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:top]:
    rs = sorted(((float(r[i] or 0), x[6:]) for x, i in zip(reasons, ri)), reverse=True)[:3]
    print(f"{r[0][-5:]} {r[1][:60]:60s} {r[si]:>7s}  " + " ".join(f"{n}:{v:.0f}" for v, n in rs if v))
