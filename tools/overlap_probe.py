"""Design evidence: cfg2 step time with co-located members time-sharing one
stream (default) vs one stream per worker (overlap_colocated).  Every member
kernel is a persistent grid over all SMs, so concurrency buys nothing
(measured 30.1 ms vs 30.3-30.7 ms per 4M-sample step)."""
import sys
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[1]))
import numpy as np, bench, paper_2208_14049_b200 as es
c = bench.make_cluster(es, bench.CONFIGS["cfg2"])
A = es.AllocationMatrix.from_array([[128, 128, 128, 128]])
X = es.SampleStore(synthetic_seed=1, nb=1 << 22, width=784, device=0)
for ov in (False, True, False, True):
    with es.InferenceSystem(A, c, es.CombinationRule.averaging(softmax=True), copy_outputs=False,
                            overlap_colocated=ov) as s:
        for _ in range(3):
            s.run(X, copy=False)
        t = [s.run(X, copy=False).stats.elapsed_s for _ in range(10)]
        print("overlap" if ov else "serial ", round(np.median(t) * 1e3, 3), "ms", flush=True)
