"""Label-identity probe (GPU): every BASELINE roster member and ensemble on the
device vs the oracle CPU member, over all rows of seeded inputs.

For each case prints the row count, the number of argmax mismatches, the max
|dz|/s (logits) or |dP| (ensembles), and for every mismatching row the
reference's top-2 gap — so a mismatch can be checked to be a sub-tolerance
tie.  Writes gpurun_out/label_probe.json.

    python tools/label_probe.py [--rows 4096]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import paper_2208_14049_b200 as es  # noqa: E402
from oracle import refcpu, restate  # noqa: E402

import bench  # noqa: E402


def gap2(P):
    s = np.sort(P, axis=1)
    return s[:, -1] - s[:, -2]


def member_case(model, X, b):
    got = es.Member(model, b).predict(X)
    cpu = refcpu.cpu_member(model.arch)
    want = cpu.forward(X)
    s = cpu.logit_scale(X)
    err = np.abs(got - want) / np.maximum(s, 1e-6)
    mis = np.nonzero(np.argmax(got, 1) != np.argmax(want, 1))[0]
    g = gap2(want)
    d = np.abs(got - want)
    normwise = d.max(axis=1) / np.maximum(np.abs(want).max(axis=1), 1e-6)
    return {"member": model.name, "rows": len(X), "b": b, "mismatches": int(len(mis)),
            "max_rel_err": float(err.max()), "max_abs_dz": float(d.max()),
            "max_normwise_rel": float(normwise.max()),
            "p999_rel_err": float(np.quantile(err.max(axis=1), 0.999)),
            "median_abs_z": float(np.median(np.abs(want))),
            "min_ref_gap": float(g.min()),
            "mismatch_ref_gaps": [float(g[i]) for i in mis[:20]]}, got, want


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--seed", type=int, default=2024)
    args = ap.parse_args()
    X = refcpu.features(args.seed, args.rows, 784)
    out = {"members": [], "ensembles": []}
    rosters = {"cfg1": bench.CONFIGS["cfg1"]["roster"], "cfg2": bench.ROSTER,
               "dozen": bench.DOZEN, "cfg4": bench.CONFIGS["cfg4"]["roster"]}
    for name, roster in rosters.items():
        models = bench.roster_models(es, roster)
        probs, mprobs = [], []
        for m in models:
            r, got, want = member_case(m, X, 128)
            r["roster"] = name
            out["members"].append(r)
            print(json.dumps(r), flush=True)
            probs.append(refcpu.softmax_rows(want))
            mprobs.append(refcpu.softmax_rows(got))
        # ensemble through the product system vs the oracle fold
        cfg = {"roster": roster, "devices": 1, "device_mib": 183359.0}
        cluster = bench.make_cluster(es, cfg)
        A = es.AllocationMatrix.from_array([[128] * len(models)])
        res = es.run_inference(es.SampleStore(X), A, cluster,
                               es.CombinationRule.averaging(softmax=True), device_map=[0])
        want, labels = restate.fold("avg", probs)
        g = gap2(want)
        mis = np.nonzero(res.winners != labels)[0]
        e = {"roster": name, "M": len(models), "rows": len(X), "mismatches": int(len(mis)),
             "max_abs_dP": float(np.abs(res.combined - want).max()),
             "min_ref_gap": float(g.min()),
             "rows_gap_below_1e-4": int((g < 1e-4).sum()),
             "rows_gap_below_1e-3": int((g < 1e-3).sum()),
             "mismatch_ref_gaps": [float(g[i]) for i in mis[:20]]}
        out["ensembles"].append(e)
        print(json.dumps(e), flush=True)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/label_probe.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
