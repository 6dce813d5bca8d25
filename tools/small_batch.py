"""Fixed cost of a small run: wall time of run_host / resident run for nb rows
of the cfg2 ensemble (what a deploy-mode flush pays per chunk)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2208_14049_b200 as es  # noqa: E402

cluster = bench.make_cluster(es, bench.CONFIGS["cfg2"])
A = es.AllocationMatrix.from_array([[128, 128, 128, 128]])
rng = np.random.default_rng(0)
with es.InferenceSystem(A, cluster) as s:
    for nb in [128, 1024, 4096, 16384, 65536]:
        X = rng.random((nb, 784), dtype=np.float32)
        Y = np.zeros((nb, 10), np.float32)
        lab = np.zeros(nb, np.int32)
        st = es.SampleStore(X)
        for _ in range(3):
            s.run_host(X, Y, lab)
            s.run(st)
        t = []
        for _ in range(20):
            t.append(s.run_host(X, Y, lab))
        dev = []
        wall = []
        for _ in range(20):
            t0 = time.perf_counter()
            out = s.run(st)
            wall.append(time.perf_counter() - t0)
            dev.append(out.stats.elapsed_s)
        km, cm = s.timing()
        print(f"nb={nb:6d} run_host {np.median(t)*1e3:7.3f} ms  run wall {np.median(wall)*1e3:7.3f} "
              f"ms  device {np.median(dev)*1e3:7.3f} ms  members {['%.3f' % k for k in km]} "
              f"combine {cm:.3f}", flush=True)
