"""B200-calibrated analytic cost model: the least-squares
fit of 1/throughput = c_m + o/b on synthetic measurements (host), and the
calibration against the device bench (GPU)."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2208_14049_b200 as es
from conftest import gpu

ROOT = Path(__file__).resolve().parents[1]
MENU = [8, 16, 32, 64, 128]


def exact(costs, o):
    return [(m, b, b / (b * c + o)) for m, c in enumerate(costs) for b in MENU]


def test_fit_recovers_exact_parameters():
    costs, o = [2.5e-9, 1.1e-8, 4e-7], 3.5e-6
    f = es.fit_cost_model(exact(costs, o), 3)
    np.testing.assert_allclose(f.cost_per_sample, costs, rtol=1e-9)
    assert f.batch_overhead_s == pytest.approx(o, rel=1e-9)
    assert f.rms_rel_error < 1e-9


def test_fit_is_robust_to_noise_and_clamps_negative_overhead():
    rng = np.random.default_rng(3)
    costs, o = [1e-8, 2e-8], 1e-6
    noisy = [(m, b, t * (1 + 0.02 * rng.standard_normal())) for m, b, t in exact(costs, o)]
    f = es.fit_cost_model(noisy, 2)
    np.testing.assert_allclose(f.cost_per_sample, costs, rtol=0.05)
    assert f.rms_rel_error < 0.05
    # Throughput falling with batch would need o < 0: pinned to 0 instead.
    falling = [(0, b, 1e8 * (1 + 1.0 / b)) for b in MENU]
    g = es.fit_cost_model(falling, 1)
    assert g.batch_overhead_s == 0.0 and g.cost_per_sample[0] > 0


def test_fit_needs_a_sample_per_model():
    with pytest.raises(es.SpecError, match="model 1 has no"):
        es.fit_cost_model([(0, 8, 1e6)], 2)


def test_calibrated_spec_drives_the_reference_analytic_score():
    costs, o = [1e-8, 3e-8], 2e-6
    c = es.ClusterSpec([es.DeviceSpec(0, es.GPU, 1e6, 1e15, 0.0)],
                       [es.mlp_model(0, "a", [784, 256, 10], 1), es.mlp_model(1, "b", [784, 512, 10], 2)],
                       MENU, 128)
    cal = es.apply_cost_fit(c, es.CostFit(costs, o, 0.0))
    A = es.AllocationMatrix.from_array([[128, 64]])
    # cost_model.cpp: min over models of b / (b*c*n/R + o), n = 2 co-located, R = 1.
    want = min(128 / (128 * costs[0] * 2 + o), 64 / (64 * costs[1] * 2 + o))
    assert es.predict_ensemble_throughput(A, cal) == pytest.approx(want, rel=1e-12)


@pytest.mark.gpu
def test_calibration_against_the_device_bench(tmp_path):
    c = es.ClusterSpec([gpu(0, 183359.0, 1e15, 0.0)],
                       [es.mlp_model(0, "mlp256", [784, 256, 10], 11),
                        es.mlp_model(1, "mlp1024", [784, 1024, 10], 13)], MENU, 128)
    f = es.calibrate_cost_model(c, 0, calib_nb=1 << 16, repeats=3)
    assert all(x > 0 for x in f.cost_per_sample) and f.batch_overhead_s >= 0
    assert len(f.measured) == 2 * len(MENU)
    # The wider member costs more per sample; larger batches are faster.
    assert f.cost_per_sample[1] > f.cost_per_sample[0]
    m0 = [t for m, b, t in f.measured if m == 0]
    assert m0[-1] > m0[0]
    # One overhead per device (the reference's model) cannot follow per-member
    # tile costs (a b-row tile costs about what a 128-row one does): measured
    # misfit ~0.7 on B200 -- recorded, bounded, not hidden.
    assert f.rms_rel_error < 1.0
    spec = tmp_path / "spec.json"
    spec.write_text(es.cluster_to_json(c, 2, with_arch=True))
    out = tmp_path / "cal.json"
    r = subprocess.run([sys.executable, "-m", "paper_2208_14049_b200.cli", "--cluster", str(spec),
                        "--calib-samples", "65536", "--json", "calibrate", "--out", str(out)],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert set(rep["models"]) == {"mlp256", "mlp1024"} and rep["spec_written"] == str(out)
    cal = es.load_spec(str(out))
    assert cal.models[1].arch == c.models[1].arch and cal.devices[0].compute_rate == 1.0
