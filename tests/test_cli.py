"""Operator commands: `python -m paper_2208_14049_b200.cli`
in analytic bench mode (no GPU) against the reports the reference's own
src/cli/commands.cpp prints for the same spec (tests/golden/spec_io.json),
plus the matrix-cache round trip of `optimize` (commands.cpp:96-143)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = json.loads((Path(__file__).parent / "golden" / "spec_io.json").read_text())
CASES = sorted(GOLDEN["clusters"])


def cli(*args, cwd=None):
    r = subprocess.run([sys.executable, "-m", "paper_2208_14049_b200.cli", *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    return r.returncode, r.stdout, r.stderr


def spec_file(tmp_path, name):
    p = tmp_path / f"{name}.json"
    p.write_text(GOLDEN["clusters"][name]["spec_indent2"])
    return p


def strip(report):
    report = dict(report)
    report.pop("wall_time_s", None)
    return report


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("seed", [0, 31337])
def test_optimize_and_baseline_reports_match_the_reference(tmp_path, name, seed):
    spec = spec_file(tmp_path, name)
    want = GOLDEN["clusters"][name]["commands"]
    for cmd in ("optimize", "baseline"):
        rc, out, err = cli("--cluster", str(spec), "--bench-mode", "analytic", "--seed", str(seed),
                           "--json", cmd)
        assert rc == 0, err
        assert strip(json.loads(out)) == want[f"{cmd}_seed{seed}"]


@pytest.mark.parametrize("name", CASES)
def test_count_and_bench_reports_match_the_reference(tmp_path, name):
    spec = spec_file(tmp_path, name)
    want = GOLDEN["clusters"][name]["commands"]
    rc, out, err = cli("--cluster", str(spec), "--json", "count")
    assert rc == 0, err
    assert strip(json.loads(out)) == want["count"]
    m = tmp_path / "m.json"
    m.write_text(GOLDEN["clusters"][name]["matrix_indent2"])
    rc, out, err = cli("--cluster", str(spec), "--bench-mode", "analytic", "--json", "bench",
                       "--matrix", str(m))
    assert rc == 0, err
    assert strip(json.loads(out)) == want["bench_wfd"]


def test_optimize_caches_then_hits_with_zero_bench_calls(tmp_path):
    spec = spec_file(tmp_path, "dozen")
    cache = tmp_path / "cache"
    args = ("--cluster", str(spec), "--bench-mode", "analytic", "--cache-dir", str(cache), "--json",
            "optimize")
    rc, out, err = cli(*args)
    assert rc == 0, err
    first = json.loads(out)
    assert first["cache"] == "miss" and first["cache_stored"] is True and first["bench_calls"] > 0
    rc, out, err = cli(*args)
    second = json.loads(out)
    assert second["cache"] == "hit" and second["bench_calls"] == 0
    assert second["best_matrix"] == first["best_matrix"] and second["score"] == first["score"]
    assert second["inputs_digest"] == first["inputs_digest"] == \
        GOLDEN["clusters"]["dozen"]["commands"]["optimize_seed0"]["inputs_digest"]


def test_text_report_and_error_exit_codes(tmp_path):
    spec = spec_file(tmp_path, "tiny")
    rc, out, _ = cli("--cluster", str(spec), "count")
    assert rc == 0 and "neighbor_formula.all_allowed: 12" in out
    rc, _, err = cli("--cluster", str(tmp_path / "missing.json"), "count")
    assert rc == 1 and "cannot open" in err
    rc, _, err = cli("--cluster", str(spec), "--bench-mode", "guess", "optimize")
    assert rc == 1 and "bench mode must be" in err
    # A spec whose models fit no device: AllocationError -> exit 2 (enserve_cli.cpp:128-130).
    doc = json.loads(GOLDEN["clusters"]["tiny"]["spec_compact"])
    doc["devices"][0]["memory_mib"] = 1.0
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps(doc))
    rc, _, err = cli("--cluster", str(bad), "--bench-mode", "analytic", "optimize")
    assert rc == 2 and "enserve:" in err


@pytest.mark.gpu
def test_measured_optimize_and_bench_on_the_b200_backend(tmp_path):
    """`optimize` / `bench` with --bench-mode measured run the device-timed
    bench (es_bench) as the greedy's ScoreFn (commands.cpp:132-150) on the
    members the spec's "arch" objects describe."""
    sys.path.insert(0, str(ROOT))
    import paper_2208_14049_b200 as es
    c = es.ClusterSpec([es.DeviceSpec(0, es.GPU, 160000.0, 1e9, 0.0)],
                       [es.mlp_model(0, "a", [784, 256, 10], 5), es.mlp_model(1, "b", [784, 128, 10], 6)],
                       [8, 32, 128], 128)
    spec = tmp_path / "cluster.json"
    spec.write_text(es.cluster_to_json(c, with_arch=True))
    rc, out, err = cli("--cluster", str(spec), "--bench-mode", "measured", "--backend", "b200",
                       "--calib-samples", "8192", "--input-width", "784", "--max-iter", "3",
                       "--json", "optimize")
    assert rc == 0, err
    rep = json.loads(out)
    assert rep["bench_calls"] > 1 and rep["score"] > 0
    best = rep["best_matrix"]
    rc, out, err = cli("--cluster", str(spec), "--bench-mode", "measured", "--backend", "b200",
                       "--calib-samples", "8192", "--input-width", "784", "--json", "bench",
                       "--matrix", str(_write_matrix(tmp_path, best)))
    assert rc == 0, err
    assert json.loads(out)["throughput"] > 0


def _write_matrix(tmp_path, best):
    p = tmp_path / "matrix.json"
    p.write_text(json.dumps(best) if isinstance(best, dict) else json.dumps({"entries": best}))
    return p
