#!/usr/bin/env python
"""Per-member device time (CUDA events, InferenceSystem.timing) for single
members, for kernel tuning.  Not part of the bench contract.

  python tools/time_members.py cnn mlp:784,256,10 --nb 1048576 --batch 128
"""
from __future__ import annotations

import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2208_14049_b200 as es  # noqa: E402


def member(spec: str, seed: int) -> es.ModelSpec:
    kind, _, rest = spec.partition(":")
    if kind == "cnn":
        w = [int(v) for v in rest.split(",")] if rest else [28, 4, 64, 32, 128, 10]
        return es.cnn_model(0, spec, seed, S=w[0], P=w[1], c1=w[2], c2=w[3], hidden=w[4],
                            classes=w[5])
    return es.mlp_model(0, spec, [int(v) for v in rest.split(",")], seed)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("members", nargs="+")
    ap.add_argument("--nb", type=int, default=1 << 20)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    for i, spec in enumerate(a.members):
        m = member(spec, 100 + i)
        c = es.ClusterSpec([es.DeviceSpec(0, es.GPU, 183359.0, 1e15, 0.0)], [m], [a.batch], 128)
        A = es.AllocationMatrix.from_array([[a.batch]])
        width = m.arch.input_width()
        X = es.SampleStore(synthetic_seed=1, nb=a.nb, width=width, device=0)
        sysm = es.InferenceSystem(A, c, es.CombinationRule.averaging(softmax=True),
                                  device_map=[0], copy_outputs=False)
        for _ in range(3):
            sysm.run(X, copy=False)
        ms = []
        for _ in range(a.steps):
            sysm.run(X, copy=False)
            ms.append(sysm.timing()[0][0])
        sysm.close()
        t = statistics.median(ms)
        f = m.arch.flops_per_sample() * a.nb
        print(f"{spec:28s} b={a.batch:4d} nb={a.nb}: {t:.4f} ms  {a.nb / (t * 1e-3):.3e} samples/s  "
              f"{f / t / 1e9:.1f} TFLOP/s  X {a.nb * width * 2 / t / 1e6:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
