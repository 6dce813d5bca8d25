#!/usr/bin/env python
"""Turn one round's gpurun_out/ evidence into committed profiles/ files:
   python tools/summarize_profiles.py <tag> [member/kernel key of the top kernel]
reads  gpurun_out/<tag>_bench.json, <tag>_launches.csv, <tag>_top.ncu-rep
writes profiles/<tag>_bench.json, <tag>_launches.csv (kernel-time rows only),
       <tag>_launch_shares.json, <tag>_top_ncu.json, and updates
       profiles/roofline_traffic.json (dram bytes per launch of the top kernel)."""
import csv
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO / "tools"))
from ncu_summary import summarise  # noqa: E402

tag = sys.argv[1]
key = sys.argv[2] if len(sys.argv) > 2 else None
src, dst = REPO / "gpurun_out", REPO / "profiles"
bench = json.loads((src / f"{tag}_bench.json").read_text())
(dst / f"{tag}_bench.json").write_text(json.dumps(bench) + "\n")

# launch list: keep csv rows, compute per-kernel shares of the profiled steps
rows = [l for l in (src / f"{tag}_launches.csv").read_text().splitlines() if l.startswith('"')]
(dst / f"{tag}_launches.csv").write_text("\n".join(rows) + "\n")
recs = list(csv.DictReader(rows))
t = defaultdict(float)
n = defaultdict(int)
for r in recs:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    t[name] += float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
    n[name] += 1
# the last (steps) x (launches per step) launches are the profiled steps; report all kernels
tot = sum(v for k, v in t.items() if "features" not in k and "dense_layer" not in k)
shares = {k: {"launches": n[k], "total_us": round(v, 1),
              "share_of_member_and_combine_time": round(v / tot, 4) if tot else None}
          for k, v in sorted(t.items(), key=lambda kv: -kv[1])}
(dst / f"{tag}_launch_shares.json").write_text(json.dumps(shares, indent=1) + "\n")

top = summarise(src / f"{tag}_top.ncu-rep")
(dst / f"{tag}_top_ncu.json").write_text(json.dumps(top, indent=1) + "\n")
if key and top:
    d = top[0]

    def gb(v):
        x, u = v.split()
        return float(x) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}[u]
    traffic = gb(d["dram_read"]) + gb(d["dram_write"])
    p = dst / "roofline_traffic.json"
    db = json.loads(p.read_text()) if p.exists() else {}
    db = {k: v for k, v in db.items() if "/" in k}  # drop pre-r1d keys (member name only)
    db[key] = traffic
    p.write_text(json.dumps(db, indent=1) + "\n")
    print("traffic", key, traffic)
print(json.dumps(shares, indent=1)[:1500])
