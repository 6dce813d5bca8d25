"""Heterogeneous members beyond the 2-layer MLP: deeper MLPs (tcgen05 dense
layers chained into the fused head) against the oracle CPU member, same
tolerance contract as tests/test_gpu_parity.py."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2208_14049_b200 as es
from conftest import gpu
from oracle import refcpu, restate
from test_gpu_parity import RTOL_BF16, assert_logits_close

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("widths", [[784, 512, 512, 10], [784, 256, 384, 128, 10],
                                    [784, 128, 256, 10]])
@pytest.mark.parametrize("b", [32, 128])
def test_deep_mlp_member_matches_cpu_oracle(widths, b):
    X = refcpu.features(41, 700, 784)
    model = es.mlp_model(0, "deep", widths, 4242)
    got = es.Member(model, b).predict(X)
    cpu = refcpu.CpuMlp(widths, 4242)
    want = cpu.forward(X)
    # Every bf16-rounded activation layer brings its own rounding-flip budget
    # (DESIGN.md §Tolerances): rtol scales with the number of hidden layers.
    assert_logits_close(got, want, cpu.logit_scale(X), rtol=RTOL_BF16 * (len(widths) - 2))
    np.testing.assert_array_equal(np.argmax(got, 1), np.argmax(want, 1))


def test_heterogeneous_depths_in_one_ensemble_match_reference_pipeline():
    if not refcpu.ref_available():
        pytest.skip("oracle/_ref not built")
    models = [es.mlp_model(0, "a", [784, 512, 512, 10], 7),
              es.mlp_model(1, "b", [784, 1024 // 2, 10], 8),
              es.mlp_model(2, "c", [784, 256, 128, 10], 9)]
    c = es.ClusterSpec([gpu(0, 180000.0, 1e15, 0.0), gpu(1, 180000.0, 1e15, 0.0)], models,
                       [8, 16, 32, 64, 128], 128)
    A = es.AllocationMatrix.from_array([[128, 64, 0], [128, 0, 32]])  # model 0 data-parallel
    X = refcpu.features(77, 128 * 9 + 40, 784)
    out = es.run_inference(es.SampleStore(X), A, c, es.CombinationRule.averaging(softmax=True))
    Yr, _, _ = refcpu.ref_run_ensemble(c, A.cells, X, rule=0, softmax=True)
    np.testing.assert_allclose(out.combined, Yr, rtol=0, atol=1e-3)
    # Winners agree wherever the reference's top two probabilities are further
    # apart than the two tolerances; inside that band either may win, but the
    # winner must still be one of the reference's top two.
    top = np.argsort(Yr, axis=1)[:, -2:]
    gap = np.take_along_axis(Yr, top[:, 1:], 1)[:, 0] - np.take_along_axis(Yr, top[:, :1], 1)[:, 0]
    clear = gap > 2e-3
    np.testing.assert_array_equal(out.winners[clear], top[clear, 1])
    assert np.all((out.winners == top[:, 1]) | (out.winners == top[:, 0]))
