"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE compiled
by oracle/Makefile (oracle/_ref/libenserve_ref.so).  Run here (the container
that has /root/reference):  python tests/golden/make_golden.py

  synthetic_prediction.json  synthetic_prediction(m, i, c) read back through the
                             reference's own run_inference + SyntheticBackend
                             (src/runtime/backend.cpp:21-29) with M = 1.
  weights.json               frozen values of the synthetic weight generator
                              from oracle/cpu_member.c.
  placement.json             worst_fit_decreasing matrices, analytic scores and
                             greedy trajectories of seeded random clusters
                             (tests/test_fixtures.hpp:67-94 instances), from the
                             reference library.
  spec_io.json               spec / matrix documents, cache keys, digests and
                             spec error messages printed by the reference's own
                             spec_io.cpp + cache.cpp (oracle/spec_golden.cpp,
                             built by `make -C oracle spec_golden` against the
                             nlohmann::json 3.11.3 header of this image).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE.parent))

from conftest import fast_cluster, random_cluster  # noqa: E402
from oracle import refcpu, restate  # noqa: E402


def synthetic_cases():
    # M = 1 averaging folds y = 0 + b * 1.0f exactly, so the combined output of a
    # one-model synthetic run IS synthetic_prediction(0, i, c).
    cases = []
    y, _, _, _ = refcpu.ref_run_synthetic(fast_cluster(1, 1, output_width=5), np.array([[16]]), 300)
    for i in (0, 1, 127, 128, 299):
        for cl in range(5):
            cases.append([0, i, cl, float(y[i, cl])])
    return cases


def weight_cases():
    cases = []
    for seed, layer, fi, fo in [(1, 0, 784, 256), (1, 1, 256, 10), (99, 0, 784, 512)]:
        for idx in (0, 1, 783, 784, 1000, fi * fo - 1):
            v = refcpu.orc().orc_weight(seed, layer, idx, fi, fo)
            cases.append({"seed": seed, "layer": layer, "idx": idx, "fan_in": fi, "fan_out": fo,
                          "value": float(np.float32(v))})
    return cases


def placement_cases():
    out = []
    rng = restate.MT19937_64(777)
    while len(out) < 30:
        c = random_cluster(rng)
        try:
            A = refcpu.ref_wfd(c, c.batch_menu[0])
        except refcpu.RefError:
            continue
        seed = rng()
        g = refcpu.ref_greedy(c, A, 10, 7, seed)
        out.append({
            "devices": [[d.kind, d.memory_mib, d.compute_rate, d.batch_overhead_s] for d in c.devices],
            "models": [[m.name, m.weight_mib, m.act_mib_per_sample, m.cost_per_sample] for m in c.models],
            "menu": c.batch_menu,
            "wfd": A.tolist(),
            "wfd_score": refcpu.ref_throughput(c, A),
            "greedy_seed": seed,
            "greedy_matrix": g["matrix"].tolist(),
            "greedy_final": g["final"],
            "greedy_neighbors": g["neighbors"],
            "greedy_stop": g["stop"],
        })
    return out


def spec_io_cases():
    import subprocess
    root = HERE.parent.parent
    subprocess.run(["make", "-C", str(root / "oracle"), "spec_golden"], check=True,
                   capture_output=True)
    out = subprocess.run([str(root / "oracle" / "_ref" / "spec_golden")], check=True,
                         capture_output=True, text=True).stdout
    return json.loads(out)


def main():
    (HERE / "synthetic_prediction.json").write_text(json.dumps({"cases": synthetic_cases()}))
    (HERE / "weights.json").write_text(json.dumps({"cases": weight_cases()}))
    (HERE / "placement.json").write_text(json.dumps({"cases": placement_cases()}, indent=0))
    (HERE / "spec_io.json").write_text(json.dumps(spec_io_cases(), indent=1) + "\n")
    print("golden fixtures written")


if __name__ == "__main__":
    main()
