#!/usr/bin/env python
"""Key metrics of .ncu-rep files as one JSON object per kernel launch
(read here, without a GPU):  python tools/ncu_summary.py gpurun_out/ncu_*.ncu-rep"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_elapsed": "tensor_inst_pct",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed": "tc_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
    "launch__shared_mem_per_block_dynamic": "smem_dyn",
}


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return []
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"file": path.split("/")[-1], "kernel": r[head.index("Kernel Name")][:60]}
        for k, short in KEYS.items():
            if k in head:
                i = head.index(k)
                d[short] = f"{r[i]} {units[i]}".strip()
        # all tensor-pipe metrics present, for reference
        for i, h in enumerate(head):
            if "pipe_tensor" in h and "pct_of_peak_sustained_active" in h and "avg" in h:
                d[h] = r[i]
        out.append(d)
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in summarize(p):
            print(json.dumps(d))
