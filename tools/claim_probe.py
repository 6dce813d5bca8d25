"""Device FIFO diagnostics: who claims what under different layouts."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2208_14049_b200 as es  # noqa: E402

ROSTER = [("mlp256", "mlp", [784, 256, 10], 11), ("mlp512x2", "mlp", [784, 512, 512, 10], 12),
          ("mlp1024", "mlp", [784, 1024, 10], 13), ("cnn-s", "cnn", [28, 4, 64, 32, 128, 10], 14)]
RULE = es.CombinationRule.averaging(softmax=True)


def run(cells, nb, **opts):
    D = len(cells)
    c = bench.make_cluster(es, {"roster": ROSTER, "devices": D, "device_mib": 183359.0})
    A = es.AllocationMatrix.from_array(cells)
    X = es.SampleStore(synthetic_seed=71, nb=nb, width=784, device=0)
    with es.InferenceSystem(A, c, RULE, device_map=[0] * D, **opts) as s:
        s.run(X, copy=False)
        t0 = time.perf_counter()
        out = s.run(X, copy=False)
        wall = time.perf_counter() - t0
        res = {}
        for m in s.claim_models():
            o = s.claims(m)
            res[m] = {int(k): int(v) for k, v in zip(*np.unique(o, return_counts=True))}
        print(f"{opts}: device {out.stats.elapsed_s * 1e3:.2f} ms, wall {wall * 1e3:.2f} ms, "
              f"launches {s.launches_last_run()}, claims {res}, member ms "
              f"{[round(x, 3) for x in s.timing()[0]]}", flush=True)


if __name__ == "__main__":
    nb = 128 * 4096 + 31
    A3 = [[0, 0, 8, 0], [128, 64, 128, 32], [0, 0, 128, 0]]
    A1 = [[0, 0, 128, 0], [0, 0, 128, 0], [0, 0, 128, 0]]
    for cells in (A3,):
        print("matrix", cells)
        run(cells, nb, row_nodes=True, dp_claim=True)
        run(cells, nb, row_nodes=True, sms_per_worker=48, claim_chunk=64, dp_claim=True)
        run(cells, nb, row_nodes=True, dp_claim=False)
        run(cells, nb, row_nodes=True, sms_per_worker=48, dp_claim=False)
        run(cells, nb, row_nodes=False, dp_claim=True)
