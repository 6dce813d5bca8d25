"""Summarise `ncu --set full` reports into a small JSON list (one entry per
profiled launch) for profiles/.

    python tools/ncu_summary.py OUT.json REP.ncu-rep [REP2.ncu-rep ...] \
        [--algo-bytes B] [--algo-flop F]

--algo-bytes / --algo-flop: the launch's algorithmic bytes / FLOP (DESIGN.md
§5), to report achieved GB/s / TFLOP/s and DRAM traffic over algorithmic.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

KEYS = {
    "time": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "sm_hz": "sm__cycles_elapsed.avg.per_second",
    "smem_dyn": "launch__shared_mem_per_block_dynamic",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}


def to_si(value: str, unit: str) -> float | None:
    try:
        v = float(value.replace(",", ""))
    except ValueError:
        return None
    return v * SCALE.get(unit, 1.0)


def summarise(rep: Path) -> list[dict]:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        col = dict(zip(head, r))
        unit = dict(zip(head, units))
        e = {"file": rep.name, "kernel": col.get("Kernel Name", "")[:120]}
        for k, m in KEYS.items():
            if m in col:
                e[k] = f"{col[m]} {unit[m]}".strip()
        t = to_si(col.get(KEYS["time"], ""), unit.get(KEYS["time"], ""))
        rd = to_si(col.get(KEYS["dram_read"], ""), unit.get(KEYS["dram_read"], ""))
        wr = to_si(col.get(KEYS["dram_write"], ""), unit.get(KEYS["dram_write"], ""))
        e["time_s"] = t
        e["dram_bytes"] = (rd or 0) + (wr or 0)
        out.append(e)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--algo-bytes", type=float, default=None)
    ap.add_argument("--algo-flop", type=float, default=None)
    args = ap.parse_args()
    res = []
    for rep in args.reps:
        for e in summarise(Path(rep)):
            if args.algo_bytes and e.get("time_s"):
                e["algorithmic_bytes"] = args.algo_bytes
                e["achieved_gbs"] = round(args.algo_bytes / e["time_s"] / 1e9, 1)
                e["dram_over_algorithmic"] = round(e["dram_bytes"] / args.algo_bytes, 3)
            if args.algo_flop and e.get("time_s"):
                e["algorithmic_flop"] = args.algo_flop
                e["achieved_tflops"] = round(args.algo_flop / e["time_s"] / 1e12, 1)
            res.append(e)
    Path(args.out).write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
