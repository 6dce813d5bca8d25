"""Pin the oracle before trusting it: the restatement (oracle/restate.py) and the
CPU member (oracle/cpu_member.c) against the reference's own known-answer tests
and against the reference library compiled from its sources (oracle/_ref)."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from conftest import (fast_cluster, imagenet4_cluster, imagenet4_matrix, random_cluster,
                      tiny_cluster, gpu, model)
from oracle import refcpu, restate

GOLDEN = Path(__file__).resolve().parent / "golden"
need_ref = pytest.mark.skipif(not refcpu.ref_available(), reason="oracle/_ref not built")


def golden(name):
    return json.loads((GOLDEN / name).read_text())


# ------------------------------------------------ reference KATs (restatement)
def test_rng_stream_matches_std_mt19937_64():
    # std::mt19937_64 default-seeded: the 10000th output is 9981545732273789042
    # (C++ standard [rand.predef]).
    g = restate.MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


def test_kat_combine_average_and_identity():
    # test_runtime.cpp:110-122
    y, _ = restate.fold("avg", [[[0, 1], [1, 0]], [[1, 0], [1, 0]]])
    assert y.ravel().tolist() == [0.5, 0.5, 1.0, 0.0]
    y, _ = restate.fold("avg", [[[0.25, 1], [1, 0.75]]])
    assert y.ravel().tolist() == [0.25, 1.0, 1.0, 0.75]


def test_kat_vote_and_tie():
    # test_runtime.cpp:168-185
    y, w = restate.fold("vote", [[[0, 9, 0], [9, 0, 0]], [[0, 5, 1], [0, 0, 7]],
                                 [[1, 0, 8], [0, 0, 2]]])
    assert y.ravel().tolist() == [0, 2, 1, 1, 0, 2]
    assert w.tolist() == [1, 2]
    _, w = restate.fold("vote", [[[9, 0]], [[0, 9]]])
    assert w.tolist() == [0]


def test_kat_weighted():
    # test_runtime.cpp:187-196
    y, _ = restate.fold("wavg", [[[1, 0]], [[0, 1]]], [0.75, 0.25])
    assert y.ravel().tolist() == [0.75, 0.25]


def test_kat_segments():
    # test_core.cpp:422-448
    assert restate.segment_bounds(2, 128, 300) == (256, 300)
    assert restate.segment_bounds(0, 128, 50) == (0, 50)
    assert restate.num_segments(300, 128) == 3 and restate.num_segments(0, 128) == 0
    with pytest.raises(IndexError):
        restate.segment_bounds(3, 128, 300)


def test_kat_costs():
    # test_cost.cpp:27-53: 0.018 s, 0.026 s, 444.44/s, 927.54/s
    c = tiny_cluster([8, 16, 32, 64, 128])
    c.devices = [gpu(0, 100000.0, 1000.0, 0.01)]
    c.models = [model(0, "m0", 100.0, 0.0, 1.0)]
    assert restate.service_time(0, 0, 8, 1, c) == pytest.approx(0.018)
    assert restate.service_time(0, 0, 8, 2, c) == pytest.approx(0.026)
    assert restate.worker_throughput(0, 0, 8, 1, c) == pytest.approx(444.4444444)
    assert restate.worker_throughput(0, 0, 128, 1, c) == pytest.approx(927.5362319)


def test_kat_combinatorics():
    # test_optimizer.cpp:101-113
    assert restate.count_total_matrices(5, 5, 8) == 13353748160923658642730712890625
    assert restate.count_total_neighs(5, 5, 8, 8) == 232
    assert restate.count_total_neighs(5, 5, 8, 0) == 240


def test_kat_wfd_examples():
    # test_optimizer.cpp:33-55, :363-373
    c = tiny_cluster([8], 2, 3)
    c.devices = [gpu(0, 16000.0), gpu(1, 16000.0)]
    c.models = [model(0, "big", 8000.0), model(1, "mid", 6000.0), model(2, "small", 4000.0)]
    A = restate.worst_fit_decreasing(c, 8)
    assert A[0, 0] == 8 and A[1, 1] == 8 and A[1, 2] == 8
    c = tiny_cluster([8], 4, 4)
    c.devices = [gpu(d, 16000.0) for d in range(4)]
    c.models = [model(m, f"m{m}", 1000.0 - m) for m in range(4)]
    A = restate.worst_fit_decreasing(c, 8)
    assert all(np.count_nonzero(A[d]) == 1 for d in range(4)) and A[0, 0] == 8 and A[3, 3] == 8


def test_synthetic_prediction_golden():
    g = golden("synthetic_prediction.json")
    for m, i, c, v in g["cases"]:
        assert float(restate.synthetic_prediction(m, i, c)) == v


# ------------------------------------------------ restatement == compiled reference
@need_ref
def test_restated_wfd_and_costs_match_reference_50_instances():
    rng = restate.MT19937_64(5150)  # test_optimizer.cpp:329-361 seed
    done = 0
    while done < 50:
        c = random_cluster(rng)
        try:
            want = refcpu.ref_wfd(c, c.batch_menu[0])
        except refcpu.RefError as e:
            assert e.code == 2
            with pytest.raises(LookupError):
                restate.worst_fit_decreasing(c, c.batch_menu[0])
            continue
        got = restate.worst_fit_decreasing(c, c.batch_menu[0])
        np.testing.assert_array_equal(got, want)
        assert restate.predict_ensemble_throughput(got, c) == refcpu.ref_throughput(c, want)
        assert restate.fit_mem(got, c)[0] == refcpu.ref_fit_mem(c, want)[0]
        done += 1


@need_ref
def test_restated_neighborhood_and_rng_match_reference():
    c = imagenet4_cluster()
    A = imagenet4_matrix().cells
    ref_n = refcpu.ref_neighborhood(c, A)
    mine = restate.neighborhood(A, c)
    assert len(mine) == len(ref_n)
    for x, y in zip(mine, ref_n):
        np.testing.assert_array_equal(x, y)
    for seed, n, k in [(0, 100, 10), (7, 228, 100), (1234, 468, 100), (3, 5, 10)]:
        assert restate.sample_indices(restate.MT19937_64(seed), n, k) == \
            refcpu.ref_sample_indices(seed, n, k)


@need_ref
def test_restated_greedy_matches_reference_trajectory():
    rng = restate.MT19937_64(2024)  # test_optimizer.cpp:251-273 seed
    done = 0
    while done < 12:
        c = random_cluster(rng)
        try:
            A0 = refcpu.ref_wfd(c, c.batch_menu[0])
        except refcpu.RefError:
            continue
        seed = rng()
        want = refcpu.ref_greedy(c, A0, 10, 100, seed)
        got = restate.bounded_greedy(A0, c, lambda A: restate.predict_ensemble_throughput(A, c),
                                     10, 100, seed)
        np.testing.assert_array_equal(got["matrix"], want["matrix"])
        assert got["final"] == want["final"] and got["start"] == want["start"]
        assert got["neighbors"] == want["neighbors"] and got["best"] == want["best"]
        assert got["stop"] == want["stop"] and got["calls"] == want["calls"]
        done += 1


@need_ref
def test_restated_fold_matches_reference_accumulator_shuffled():
    # test_runtime.cpp:123-154: 300 samples, C=3, M=4, shuffled arrival
    nb, C, M, N = 300, 3, 4, 128
    outs = [restate.synthetic_block(m, nb, C) for m in range(M)]
    order = [(s, m) for s in range(3) for m in range(M)]
    rng = restate.MT19937_64(11)
    for i in range(len(order), 1, -1):
        j = restate.uniform_index(rng, i)
        order[i - 1], order[j] = order[j], order[i - 1]
    for rule, name, w in [(0, "avg", None), (1, "vote", None), (2, "wavg", [0.4, 0.3, 0.2, 0.1])]:
        y_ref, win_ref = refcpu.ref_accumulate(nb, N, rule, outs, order, w)
        y, win = restate.fold(name, outs, w)
        np.testing.assert_array_equal(y, y_ref)
        if rule == 1:
            np.testing.assert_array_equal(win, win_ref)
        yc, _ = refcpu.fold(rule, outs, w)  # the C restatement too
        np.testing.assert_array_equal(yc, y_ref)


@need_ref
def test_reference_synthetic_pipeline_is_layout_invariant():
    # test_runtime.cpp:253-280 run through the compiled reference itself
    A1 = np.array([[32, 8]])
    y1, _, segs, msgs = refcpu.ref_run_synthetic(fast_cluster(1, 2), A1, 500)
    A2 = np.array([[16, 0], [64, 8], [0, 128]])
    y2, _, _, _ = refcpu.ref_run_synthetic(fast_cluster(3, 2), A2, 500)
    np.testing.assert_array_equal(y1, y2)
    assert segs == 4 and msgs == 8
    want, _ = restate.fold("avg", [restate.synthetic_block(m, 500, 4) for m in range(2)])
    np.testing.assert_array_equal(y1, want)


# ------------------------------------------------ CPU member oracle
def test_cpu_member_weights_follow_the_documented_generator():
    g = golden("weights.json")
    for case in g["cases"]:
        v = refcpu.orc().orc_weight(case["seed"], case["layer"], case["idx"], case["fan_in"],
                                   case["fan_out"])
        assert v == np.float32(case["value"])


def test_cpu_member_matches_float64_reference_within_bf16_tolerance():
    """The C member (bf16 quantisation, fp32 accumulation) against a float64
    numpy forward on the same quantised operands: only accumulation-order
    differences remain (rel. 1e-5 of the row scale)."""
    X = refcpu.features(3, 64, 784)
    mlp = refcpu.CpuMlp([784, 256, 10], seed=11)
    W1, b1 = mlp.layer(0)
    W2, b2 = mlp.layer(1)
    q = np.vectorize(lambda v: refcpu.orc().orc_round_bf16(float(v)), otypes=[np.float32])
    Xq = q(X).astype(np.float64)
    h = np.maximum(Xq @ W1.T.astype(np.float64) + b1, 0.0)
    hq = q(h.astype(np.float32)).astype(np.float64)
    z = hq @ W2.T.astype(np.float64) + b2
    got = mlp.forward(X)
    scale = np.abs(z).max(axis=1, keepdims=True)
    assert np.max(np.abs(got - z) / scale) < 2e-3  # bf16 hidden re-rounding dominates
    assert (np.argmax(got, 1) == np.argmax(z, 1)).mean() > 0.98


def _cnn_numpy(cnn, x):
    """The CNN member's definition (cpu_member.h) written directly in numpy:
    patch convolution, zero-padded 3x3 convolution over HWC activations, HWC
    flatten, two dense layers; bf16 rounding of X, weights and activations."""
    S, P, c1, c2, hidden, _ = cnn.widths
    G = S // P
    w0, b0 = cnn.layer(0)
    w1, b1 = cnn.layer(1)
    w2, b2 = cnn.layer(2)
    w3, b3 = cnn.layer(3)
    q = refcpu.round_bf16
    img = q(x.reshape(S, S).astype(np.float32)).astype(np.float64)
    patches = img.reshape(G, P, G, P).transpose(0, 2, 1, 3).reshape(G, G, P * P)
    a1 = q(np.maximum(patches @ w0.T + b0, 0).astype(np.float32)).astype(np.float64)
    pad = np.zeros((G + 2, G + 2, c1))
    pad[1:G + 1, 1:G + 1] = a1
    cols = np.concatenate([pad[dh:dh + G, dw:dw + G] for dh in range(3) for dw in range(3)], axis=2)
    a2 = q(np.maximum(cols @ w1.T + b1, 0).astype(np.float32)).astype(np.float64)
    h = q(np.maximum(a2.reshape(-1) @ w2.T + b2, 0).astype(np.float32)).astype(np.float64)
    return h @ w3.T + b3


@pytest.mark.parametrize("widths", [(28, 4, 64, 32, 128, 10), (16, 4, 32, 64, 64, 7)])
def test_cpu_cnn_member_matches_numpy_definition(widths):
    cnn = refcpu.CpuCnn(widths, seed=5)
    X = refcpu.features(3, 6, widths[0] * widths[0])
    got = cnn.forward(X)
    want = np.stack([_cnn_numpy(cnn, x) for x in X])
    # Same quantisation points; fp32-vs-float64 accumulation can still flip a
    # bf16 activation rounding, so the bound is the MLP test's (2e-3 of the row).
    scale = np.abs(want).max(axis=1, keepdims=True)
    assert np.max(np.abs(got - want) / scale) < 2e-3
    np.testing.assert_array_equal(np.argmax(got, 1), np.argmax(want, 1))


def test_cpu_cnn_weights_use_the_shared_generator():
    cnn = refcpu.CpuCnn((28, 4, 64, 32, 128, 10), seed=9)
    for layer, (fi, fo) in enumerate(cnn.dims):
        w, b = cnn.layer(layer)
        for idx in (0, 7, fi * fo - 1):
            v = refcpu.round_bf16(np.float32(refcpu.orc().orc_weight(9, layer, idx, fi, fo)))
            assert w.reshape(-1)[idx] == v
        assert b[0] == np.float32(refcpu.orc().orc_bias(9, layer, 0))
