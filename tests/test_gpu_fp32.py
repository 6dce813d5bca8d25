"""The fp32-accurate member mode (PoolOptions.fp32; north_star: logits and
averaged probabilities within 1e-5 for fp32, predicted classes identical).

Every BASELINE roster member in fp32 (X, weights, activations, accumulation)
against the oracle member with quantize_bf16 = 0 (oracle/cpu_member.c), and
the cfg2 ensemble against the reference's own InferenceSystem (oracle/_ref,
pipeline.cpp) running those fp32 oracle members.  The two sides accumulate
in different orders, so a logit is held to 1e-5 of its conditioning s (the
dot product's scale); averaged probabilities to 1e-5 absolute.
"""
from __future__ import annotations

import numpy as np
import pytest

import bench
import paper_2208_14049_b200 as es
from oracle import refcpu
from test_gpu_parity import assert_labels_identical_or_tied

pytestmark = pytest.mark.gpu
need_ref = pytest.mark.skipif(not refcpu.ref_available(), reason="oracle/_ref not built")
RTOL_FP32 = 1e-5
TOL_P_FP32 = 1e-5

MEMBERS = bench.ROSTER + [r[:4] for r in bench.DOZEN if r[0] in ("mlp2048", "mlp384x2", "cnn-w")]


def cpu_fp32(model):
    a = model.arch
    if a.kind == "cnn":
        return refcpu.CpuCnn(a.widths, a.weight_seed, quantize_bf16=False)
    return refcpu.CpuMlp(a.widths, a.weight_seed, quantize_bf16=False)


def member_logits(model, X, **pool):
    """One member alone, averaging without softmax: the fold multiplies by
    1.0f, so `combined` is the member's logits exactly."""
    c = es.ClusterSpec([es.DeviceSpec(0, es.GPU, 183359.0, 1e15, 0.0)], [model],
                       [8, 16, 32, 64, 128], 128)
    return es.run_inference(es.SampleStore(X), es.AllocationMatrix.from_array([[128]]), c,
                            es.CombinationRule.averaging(), fp32=True, **pool).combined


@pytest.mark.parametrize("idx", range(len(MEMBERS)), ids=[m[0] for m in MEMBERS])
def test_fp32_member_matches_fp32_oracle(idx):
    model = bench.roster_models(es, [MEMBERS[idx]])[0]
    X = refcpu.features(300 + idx, 777, model.arch.input_width())
    got = member_logits(model, X)
    cpu = cpu_fp32(model)
    want = cpu.forward(X)
    s = cpu.logit_scale(X)
    err = np.abs(got.astype(np.float64) - want) / np.maximum(s, 1e-6)
    print(f"{model.name}: max |dz|/s = {err.max():.2e}")
    assert np.all(np.isfinite(got)) and err.max() <= RTOL_FP32
    assert_labels_identical_or_tied(np.argmax(got, 1), want, RTOL_FP32 * s, model.name)


@need_ref
def test_fp32_cfg2_ensemble_matches_reference_pipeline():
    c = bench.make_cluster(es, {"roster": bench.ROSTER, "devices": 1, "device_mib": 183359.0})
    A = es.AllocationMatrix.from_array([[128, 64, 128, 32]])
    X = refcpu.features(310, 128 * 9 + 41, 784)
    out = es.run_inference(es.SampleStore(X), A, c, es.CombinationRule.averaging(softmax=True),
                           fp32=True)
    Yr, _, _ = refcpu.ref_run_ensemble(c, A.cells, X, rule=0, quantize=False, softmax=True)
    dY = float(np.abs(out.combined - Yr).max())
    print(f"fp32 cfg2 ensemble: max |dP| = {dY:.2e}")
    assert dY <= TOL_P_FP32
    assert_labels_identical_or_tied(out.winners, Yr, TOL_P_FP32, "fp32 cfg2")


def test_fp32_paths_agree_bit_for_bit():
    """run_host (fp32 rows over PCIe, no conversion) and a data-parallel
    layout popping the device queue give the resident run's bits."""
    c1 = bench.make_cluster(es, {"roster": bench.ROSTER, "devices": 1, "device_mib": 183359.0})
    c2 = bench.make_cluster(es, {"roster": bench.ROSTER, "devices": 2, "device_mib": 183359.0})
    nb = 128 * 11 + 3
    X = refcpu.features(311, nb, 784)
    rule = es.CombinationRule.averaging(softmax=True)
    ref = es.run_inference(es.SampleStore(X), es.AllocationMatrix.from_array([[128, 64, 128, 32]]),
                           c1, rule, fp32=True)
    with es.InferenceSystem(es.AllocationMatrix.from_array([[128, 64, 128, 32]]), c1, rule,
                            fp32=True, e2e_chunk_rows=512) as s:
        Y = np.zeros((nb, 10), np.float32)
        L = np.zeros(nb, np.int32)
        s.run_host(X, Y, L)
        h2d, _ = s.last_transfer()
    assert h2d == nb * 784 * 4
    np.testing.assert_array_equal(Y, ref.combined)
    np.testing.assert_array_equal(L, ref.winners)
    A = es.AllocationMatrix.from_array([[128, 64, 128, 32], [64, 128, 32, 128]])
    with es.InferenceSystem(A, c2, rule, fp32=True, device_map=[0, 0], row_nodes=True,
                            dp_claim=True, claim_chunk=2) as s:
        out = s.run(es.SampleStore(X))
        assert s.claim_models() == [0, 1, 2, 3]
    np.testing.assert_array_equal(out.combined, ref.combined)
