#!/usr/bin/env python
"""e2e (run_host) throughput of the cfg2 ensemble vs the share of chunks the
host converts to bf16 (PoolOptions::e2e_convert_eighths) and the chunk size.
Design evidence for the default; not part of the bench contract."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2208_14049_b200 as es  # noqa: E402

cfg = bench.CONFIGS["cfg2"]
cluster = bench.make_cluster(es, cfg)
A = es.AllocationMatrix.from_array([[128, 128, 128, 128]])
nb = 1 << 20
Xh = torch.empty((nb, 784), dtype=torch.float32, pin_memory=True).numpy()
Xh[:] = np.random.default_rng(0).random((nb, 784), dtype=np.float32)
Yh = torch.empty((nb, 10), dtype=torch.float32, pin_memory=True).numpy()
Lh = torch.empty((nb,), dtype=torch.int32, pin_memory=True).numpy()
for chunk in (65536, 131072):
    for k8 in (0, 4, 5, 6, 7, 8):
        s = es.InferenceSystem(A, cluster, es.CombinationRule.averaging(softmax=True),
                               device_map=[0], copy_outputs=False, e2e_chunk_rows=chunk,
                               e2e_host_convert=k8 > 0, e2e_convert_eighths=k8)
        s.run_host(Xh, Yh, Lh)
        ts = [s.run_host(Xh, Yh, Lh) for _ in range(4)]
        h2d, _ = s.last_transfer()
        s.close()
        print(f"chunk {chunk:6d} convert {k8}/8: {nb / np.median(ts):.3e} samples/s  "
              f"h2d {h2d / nb:.0f} B/sample", flush=True)
