"""The device FIFO: a data-parallel model's
workers pop chunks of segments off one device counter, the reference's shared
per-model queue (/root/reference/proj/src/runtime/pipeline.cpp:44-51,
:103-104).  Ported checks: every segment is predicted exactly once
(tests/test_runtime.cpp:282-313) and the layout never changes the result
(:253-280) -- here also under skewed worker rates, where a faster worker must
take more of the queue."""
from __future__ import annotations

import numpy as np
import pytest

import bench
import paper_2208_14049_b200 as es
from conftest import fast_cluster
from oracle import refcpu, restate

pytestmark = pytest.mark.gpu

RULE = es.CombinationRule.averaging(softmax=True)
ROSTER = [("mlp256", "mlp", [784, 256, 10], 11), ("mlp512x2", "mlp", [784, 512, 512, 10], 12),
          ("mlp1024", "mlp", [784, 1024, 10], 13), ("cnn-s", "cnn", [28, 4, 64, 32, 128, 10], 14)]


def cluster(devices):
    return bench.make_cluster(es, {"roster": ROSTER, "devices": devices, "device_mib": 183359.0})


def workers_of(A, m):
    idx = [(d, mm) for d in range(A.device_count()) for mm in range(A.model_count()) if A.at(d, mm)]
    return [i for i, (d, mm) in enumerate(idx) if mm == m]


def assert_exactly_once(owner, workers, segments):
    assert owner is not None and len(owner) == segments
    assert np.all(owner >= 0), "a segment was never claimed"
    assert set(np.unique(owner).tolist()) <= set(workers)


def test_synthetic_members_every_segment_exactly_once():
    """test_runtime.cpp:282-313 with the queue on the device: synthetic
    members (output keyed on the absolute sample index), both models
    data-parallel over four rows on their own streams."""
    c = fast_cluster(4, 2, output_width=3)
    A = es.AllocationMatrix.from_array([[8, 16], [32, 0], [0, 64], [128, 8]])
    nb = 128 * 40 + 17
    X = es.SampleStore(np.zeros((nb, 4), np.float32))
    with es.InferenceSystem(A, c, es.CombinationRule.averaging(), device_map=[0] * 4,
                            row_nodes=True, claim_chunk=3, dp_claim=True) as s:
        assert s.claim_models() == [0, 1]
        out = s.run(X)
        for m in (0, 1):
            assert_exactly_once(s.claims(m), workers_of(A, m), 41)
    want = restate.fold("avg", [restate.synthetic_block(m, nb, 3) for m in (0, 1)])[0]
    np.testing.assert_array_equal(out.combined, want)


def test_claims_under_skewed_rates_are_exactly_once_and_favour_the_fast_workers():
    """mlp1024 data-parallel over three rows, each row its own node on a
    disjoint third of the SMs (48 each: three GPUs in one), so the workers
    really run side by side: one at b = 8 (an 8-row tile costs about a 128-row
    tile: ~16x slower per segment), two at b = 128.  The queue is drained
    exactly once; the slow worker takes less than half of what the fast ones
    take together; the result is bit-identical to the static split and to one
    worker.  (Without the SM partition, persistent grids time-share the GPU
    and whichever stream the dispatcher favours drains the queue -- still
    exactly once.)  The auto mode keeps workers sharing a GPU on the probed
    split (no queue) and queues only workers on distinct GPUs."""
    c = cluster(3)
    A = es.AllocationMatrix.from_array([[0, 0, 8, 0], [128, 64, 128, 32], [0, 0, 128, 0]])
    nb = 128 * 4096 + 31
    X = es.SampleStore(synthetic_seed=71, nb=nb, width=784, device=0)
    with es.InferenceSystem(A, c, RULE, device_map=[0] * 3, row_nodes=True, sms_per_worker=48,
                            claim_chunk=64, dp_claim=True) as s:
        assert 2 in s.claim_models()
        s.run(X)  # first run: lazy module loads serialise the streams
        out = s.run(X)
        owner = s.claims(2)
    w = workers_of(A, 2)
    assert_exactly_once(owner, w, 4097)
    counts = {i: int((owner == i).sum()) for i in w}
    print(f"segments claimed per mlp1024 worker (b=8, b=128, b=128): {counts}")
    assert 2 * counts[w[0]] < counts[w[1]] + counts[w[2]]
    with es.InferenceSystem(A, c, RULE, device_map=[0] * 3, row_nodes=True,
                            dp_claim=False) as s:
        assert s.claim_models() == []
        static = s.run(X)
    single = es.run_inference(X, es.AllocationMatrix.from_array([[128, 64, 128, 32]]), cluster(1),
                              RULE)
    with es.InferenceSystem(A, c, RULE, device_map=[0] * 3, row_nodes=True) as s:
        assert s.claim_models() == []  # auto: every worker on GPU 0
    np.testing.assert_array_equal(out.combined, static.combined)
    np.testing.assert_array_equal(out.combined, single.combined)
    np.testing.assert_array_equal(out.winners, single.winners)


@pytest.mark.parametrize("cells", [[[128, 64, 128, 32], [64, 128, 0, 128]],
                                   [[128, 0, 0, 32], [128, 64, 128, 128], [0, 64, 128, 0]]])
def test_every_member_family_follows_its_claims(cells):
    """Every member kernel family (TMEM head, SM-pair head, SM-pair dense
    layer + pair head, conv stack + head) data-parallel through the queue,
    rows sharing one stream (first worker drains it) and on their own streams
    (racing): bit-identical to the one-worker layout."""
    D = len(cells)
    A = es.AllocationMatrix.from_array(cells)
    nb = 128 * 97 + 5
    X = es.SampleStore(refcpu.features(72, nb, 784))
    single = es.run_inference(X, es.AllocationMatrix.from_array([[128, 64, 128, 32]]), cluster(1),
                              RULE)
    for row_nodes in (False, True):
        with es.InferenceSystem(A, cluster(D), RULE, device_map=[0] * D, row_nodes=row_nodes,
                                claim_chunk=5, dp_claim=True) as s:
            out = s.run(X)
            out2 = s.run(X)  # queues reset between runs
            for m in range(4):
                if len(workers_of(A, m)) > 1:
                    assert m in s.claim_models()
                    assert_exactly_once(s.claims(m), workers_of(A, m), 98)
        np.testing.assert_array_equal(out.combined, single.combined)
        np.testing.assert_array_equal(out2.combined, single.combined)
        np.testing.assert_array_equal(out.winners, single.winners)


@pytest.mark.skipif(es.device_count() < 2, reason="needs two visible GPUs")
def test_auto_queue_across_two_physical_gpus():
    """The deployment case: data-parallel workers on distinct GPUs pop one
    queue on the combining GPU through NVLink peer atomics (auto mode)."""
    A = es.AllocationMatrix.from_array([[128, 64, 128, 32], [128, 64, 128, 32]])
    nb = 128 * 301 + 9
    X = es.SampleStore(refcpu.features(73, nb, 784))
    with es.InferenceSystem(A, cluster(2), RULE, device_map=[0, 1]) as s:
        assert s.claim_models() == [0, 1, 2, 3]
        out = s.run(X)
        for m in range(4):
            assert_exactly_once(s.claims(m), workers_of(A, m), 302)
    single = es.run_inference(X, es.AllocationMatrix.from_array([[128, 64, 128, 32]]), cluster(1),
                              RULE)
    np.testing.assert_array_equal(out.combined, single.combined)


@pytest.mark.parametrize("nb", [0, 1, 127, 129])
def test_tiny_and_empty_stores_through_every_new_path(nb):
    """Edge sizes the reference handles (an empty store Deploys to nothing,
    test_runtime.cpp): claims, row nodes with peer-store and staged routes,
    run_host lanes and fp32 all agree with the one-node bf16 layout."""
    A = es.AllocationMatrix.from_array([[128, 64, 0, 32], [64, 128, 128, 128]])
    c = cluster(2)
    X = refcpu.features(74, nb, 784) if nb else np.zeros((0, 784), np.float32)
    rule = RULE
    ref = es.run_inference(es.SampleStore(X), A, c, rule, device_map=[0, 0])
    for opts in ({"row_nodes": True, "dp_claim": True, "claim_chunk": 1},
                 {"row_nodes": True, "peer_stores": False},
                 {"dp_claim": False}):
        with es.InferenceSystem(A, c, rule, device_map=[0, 0], **opts) as s:
            out = s.run(es.SampleStore(X))
            Y = np.zeros((nb, 10), np.float32)
            L = np.zeros(nb, np.int32)
            s.run_host(X, Y, L)
        np.testing.assert_array_equal(out.combined, ref.combined)
        np.testing.assert_array_equal(Y, ref.combined)
        np.testing.assert_array_equal(L, ref.winners)
    fp = es.run_inference(es.SampleStore(X), A, c, rule, device_map=[0, 0], fp32=True)
    assert fp.combined.shape == (nb, 10)
    if nb:
        assert np.abs(fp.combined - ref.combined).max() < 2e-3  # bf16 vs fp32 members


@pytest.mark.parametrize("single", [False, True], ids=["dense_pair", "dense_single"])
def test_wide_member_dense_head_follows_claims(single, monkeypatch):
    """The dense schedules -- a hidden layer too wide for a fused head
    (784 -> 4096 -> 10: dense hidden layer + dense logits layer), on SM pairs
    or, with ES_DENSE_KERNEL=single, one SM -- also follow a claimed run:
    data-parallel over two rows they give the one-worker bits."""
    if single:
        monkeypatch.setenv("ES_DENSE_KERNEL", "single")
    roster = [("wide", "mlp", [784, 4096, 10], 91), ("mlp256", "mlp", [784, 256, 10], 92)]
    c1 = bench.make_cluster(es, {"roster": roster, "devices": 1, "device_mib": 183359.0})
    c2 = bench.make_cluster(es, {"roster": roster, "devices": 2, "device_mib": 183359.0})
    X = es.SampleStore(refcpu.features(75, 128 * 37 + 9, 784))
    single_out = es.run_inference(X, es.AllocationMatrix.from_array([[128, 128]]), c1, RULE)
    A = es.AllocationMatrix.from_array([[128, 128], [64, 32]])
    with es.InferenceSystem(A, c2, RULE, device_map=[0, 0], row_nodes=True, dp_claim=True,
                            claim_chunk=3) as s:
        out = s.run(X)
        assert s.claim_models() == [0, 1]
        assert_exactly_once(s.claims(0), workers_of(A, 0), 38)
    np.testing.assert_array_equal(out.combined, single_out.combined)
    cpu = refcpu.CpuMlp([784, 4096, 10], 91)
    Xh = refcpu.features(75, 128 * 37 + 9, 784)
    z = es.run_inference(es.SampleStore(Xh), es.AllocationMatrix.from_array([[128]]),
                         bench.make_cluster(es, {"roster": roster[:1], "devices": 1,
                                                 "device_mib": 183359.0}),
                         es.CombinationRule.averaging()).combined
    want = cpu.forward(Xh)
    s_ = cpu.logit_scale(Xh)
    assert (np.abs(z - want) / np.maximum(s_, 1e-6)).max() <= 1e-3
