#!/usr/bin/env python
"""Design evidence, not product: per-role warp-stall breakdown of one kernel
from an ncu --set full --import-source capture.
  python tools/role_stalls.py <report.ncu-rep> <cubin from the .so> <kernel substring> \
         role=first_line-last_line [role=...]
Line ranges refer to the kernel's .cu file (the outermost inlined-at line of
that file decides the role)."""
import csv
import io
import re
import subprocess
import sys
from collections import Counter, defaultdict

rep, cubin, kname = sys.argv[1:4]
roles = []
for a in sys.argv[4:]:
    name, rng = a.split("=")
    lo, hi = map(int, rng.split("-"))
    roles.append((name, lo, hi))
src_file = None
lines = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
m, cur, insec = {}, [], False
for l in lines.splitlines():
    if l.startswith("\t.section") or l.startswith("//----"):
        insec = kname in l
        continue
    if not insec:
        continue
    if "//## File" in l:
        cur = [int(x) for x in re.findall(r'_kernel\.cu", line (\d+)', l)]
        continue
    mo = re.search(r"/\*([0-9a-f]{4,5})\*/", l)
    if mo:
        m[int(mo.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
base = int(data[0][0], 16)
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def role(ls):
    for L in reversed(ls):  # outermost first
        for name, lo, hi in roles:
            if lo <= L <= hi:
                return name
    return "other"


agg, tot, inst = defaultdict(Counter), Counter(), Counter()
for r in data:
    ro = role(m.get(int(r[0], 16) - base, []))
    tot[ro] += int(r[ix["Warp Stall Sampling (All Samples)"]])
    inst[ro] += int(r[ix["Instructions Executed"]] or 0)
    for h in cols:
        agg[ro][h[6:]] += int(r[ix[h]] or 0)
print(f"mapped {len(m)} SASS offsets")
for ro in sorted(tot, key=lambda k: -tot[k]):
    top = ", ".join(f"{k} {v}" for k, v in agg[ro].most_common(6))
    print(f"{ro:10s} samples {tot[ro]:7d} warp-inst {inst[ro]:11d} | {top}")
