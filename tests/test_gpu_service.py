"""Deploy-mode service on the GPU, ported from the
reference's tests/test_server.cpp without the HTTP layer: POST /v1/predict is
`submit`/`result`, GET /v1/stats is `stats`, a 400 is InvalidArgument, a 503 is
NotReadyError.  Results must be bit-identical to an offline `run_inference` over
the same rows (test_server.cpp:176-220, 313-350)."""
from __future__ import annotations

import threading
import time

import numpy as np
import pytest

import paper_2208_14049_b200 as es
from conftest import fast_cluster

pytestmark = pytest.mark.gpu


def serve_cluster():
    """test_server.cpp:31-39: two synthetic members, 3 classes, segment 128."""
    return fast_cluster(1, 2, output_width=3)


def serve_matrix():
    return es.AllocationMatrix.from_array([[32, 16]])


def mlp_cluster():
    models = [es.mlp_model(0, "a", [784, 256, 10], 301), es.mlp_model(1, "b", [784, 128, 10], 302)]
    return es.ClusterSpec([es.DeviceSpec(0, es.GPU, 160000.0, 1e9, 0.0)], models,
                          [8, 16, 32, 64, 128], 128)


def sample_rows(rows, width, offset=0.0):
    """test_server.cpp:sample_rows: deterministic features."""
    return (offset + np.arange(rows * width, dtype=np.float32).reshape(rows, width) * 0.01)


def offline(X, A, c):
    return es.run_inference(es.SampleStore(np.ascontiguousarray(X)), A, c)


@pytest.mark.parametrize("kind", ["synthetic", "mlp"])
def test_predictions_identical_to_offline_runtime(kind):
    c, A = (serve_cluster(), serve_matrix()) if kind == "synthetic" else (
        mlp_cluster(), es.AllocationMatrix.from_array([[64, 32]]))
    width = 4 if kind == "synthetic" else 784
    X = sample_rows(5, width)
    if kind == "mlp":
        X = np.random.default_rng(3).random((5, width), dtype=np.float32)
    with es.PredictionService(c, A, flush_timeout_ms=10, input_width=width) as svc:
        assert svc.wait_ready(30.0)
        Y, W = svc.predict(X)
        ref = offline(X, A, c)
        np.testing.assert_array_equal(Y, ref.combined)  # bit-identical
        np.testing.assert_array_equal(W, ref.winners)
        st = svc.stats()
        assert st.ready and st.samples_served >= 5 and st.requests_served >= 1
        assert st.pending_requests == 0 and st.flushes >= 1 and st.uptime_s > 0
        assert st.matrix == A.cells.tolist()  # test_server.cpp:210-217


def test_full_segment_flushes_immediately_single_sample_waits_timer():
    # test_server.cpp:223-253
    with es.PredictionService(serve_cluster(), serve_matrix(), flush_timeout_ms=200,
                              input_width=4) as svc:
        assert svc.wait_ready(30.0)
        t0 = time.perf_counter()
        Y, _ = svc.predict(sample_rows(128, 4))
        assert Y.shape == (128, 3)
        assert time.perf_counter() - t0 < 0.19  # did not sit out the 200 ms timer
        t0 = time.perf_counter()
        Y, _ = svc.predict(sample_rows(1, 4))
        waited = time.perf_counter() - t0
        assert Y.shape == (1, 3)
        assert 0.19 <= waited < 5.0  # flushed by the timer


def test_bad_requests_rejected_empty_request_answered():
    # test_server.cpp:286-311
    with es.PredictionService(serve_cluster(), serve_matrix(), flush_timeout_ms=10,
                              input_width=4) as svc:
        assert svc.wait_ready(30.0)
        with pytest.raises(es.InvalidArgument):
            svc.submit(sample_rows(2, 3))
        Y, W = svc.predict(np.zeros((0, 4), np.float32))
        assert Y.shape == (0, 3) and W.shape == (0,)


def test_concatenated_buffered_requests_equal_one_offline_pass():
    # test_server.cpp:313-350: both requests land in one flush
    c, A = serve_cluster(), serve_matrix()
    first, second = sample_rows(3, 4, 0.0), sample_rows(2, 4, 100.0)
    out = {}
    with es.PredictionService(c, A, flush_timeout_ms=120, input_width=4) as svc:
        assert svc.wait_ready(30.0)

        def post(key, x):
            out[key] = svc.predict(x)

        t1 = threading.Thread(target=post, args=("a", first))
        t1.start()
        time.sleep(0.02)
        t2 = threading.Thread(target=post, args=("b", second))
        t2.start()
        t1.join()
        t2.join()
        assert svc.stats().flushes == 1
    ref = offline(np.concatenate([first, second]), A, c)
    np.testing.assert_array_equal(np.concatenate([out["a"][0], out["b"][0]]), ref.combined)


def test_many_concurrent_clients_get_their_own_rows():
    c, A = mlp_cluster(), es.AllocationMatrix.from_array([[64, 32]])
    rng = np.random.default_rng(7)
    reqs = [rng.random((int(n), 784), dtype=np.float32) for n in rng.integers(1, 300, 24)]
    with es.PredictionService(c, A, flush_timeout_ms=5, input_width=784) as svc:
        assert svc.wait_ready(30.0)
        pending = [svc.submit(x) for x in reqs]
        got = [p.result() for p in pending]
        st = svc.stats()
        assert st.requests_served == len(reqs)
        assert st.samples_served == sum(len(x) for x in reqs)
        assert st.last_flush_throughput > 0
    ref = offline(np.concatenate(reqs), A, c)
    np.testing.assert_array_equal(np.concatenate([g[1] for g in got]), ref.winners)
    # Member outputs do not depend on which flush a row landed in.
    np.testing.assert_array_equal(np.concatenate([g[0] for g in got]), ref.combined)


def test_stop_fails_buffered_requests_and_refuses_new_ones():
    svc = es.PredictionService(serve_cluster(), serve_matrix(), flush_timeout_ms=60000,
                               input_width=4)
    assert svc.wait_ready(30.0)
    p = svc.submit(sample_rows(1, 4))  # waits for a timer that never fires
    assert svc.stats().pending_requests == 1
    handle = svc._h
    es.lib().es_service_destroy(handle)  # stop + release, p still outstanding
    svc._h = None
    with pytest.raises(es.NotReadyError, match="shutting down"):
        p.result()


def test_invalid_matrix_is_a_spec_error():
    with pytest.raises(es.SpecError):
        es.PredictionService(serve_cluster(), es.AllocationMatrix.from_array([[0, 16]]),
                             input_width=4)


def test_startup_oom_reported_by_wait_ready():
    # server.cpp:37-52: a failed pool load leaves the service not ready with the error kept
    c = fast_cluster(1, 2)
    c.models[0].weight_mib = c.models[1].weight_mib = 9000.0
    c.devices[0].memory_mib = 16000.0
    with es.PredictionService(c, es.AllocationMatrix.from_array([[8, 8]]), input_width=4) as svc:
        assert not svc.wait_ready(30.0)
        assert svc.startup_error
        assert not svc.stats().ready
        with pytest.raises(es.NotReadyError):
            svc.submit(np.zeros((1, 4), np.float32))


@pytest.mark.parametrize("arena_rows", [0, 256, 131072])
def test_arena_sizes_give_identical_answers(arena_rows):
    """Requests staged in the page-locked arenas, spilled to private buffers
    (arena full or too small), or mixed in one flush answer identically."""
    c, A = mlp_cluster(), es.AllocationMatrix.from_array([[64, 32]])
    rng = np.random.default_rng(11)
    reqs = [rng.random((int(n), 784), dtype=np.float32) for n in rng.integers(1, 400, 40)]
    with es.PredictionService(c, A, flush_timeout_ms=3, input_width=784,
                              arena_rows=arena_rows) as svc:
        assert svc.wait_ready(30.0)
        got = [p.result() for p in [svc.submit(x) for x in reqs]]
    ref = offline(np.concatenate(reqs), A, c)
    np.testing.assert_array_equal(np.concatenate([g[0] for g in got]), ref.combined)
    np.testing.assert_array_equal(np.concatenate([g[1] for g in got]), ref.winners)


def test_service_matches_the_reference_pipeline_with_mlp_and_cnn_members():
    """The reference's fidelity test (test_server.cpp:176-221) compares served
    predictions with offline inference; here the offline side is the
    reference's own InferenceSystem (oracle/_ref, pipeline.cpp) running the
    oracle CPU members of the cfg2 roster (MLPs + CNN), and the requests
    arrive from four concurrent clients with ragged sizes."""
    import bench
    from oracle import refcpu
    from test_gpu_parity import TOL_P, assert_labels_identical_or_tied
    if not refcpu.ref_available():
        pytest.skip("oracle/_ref not built")
    c = bench.make_cluster(es, {"roster": bench.ROSTER, "devices": 1, "device_mib": 183359.0})
    A = es.AllocationMatrix.from_array([[128, 64, 128, 32]])
    rule = es.CombinationRule.averaging(softmax=True)
    X = refcpu.features(501, 1300, 784)
    sizes = [1, 37, 128, 200, 3, 331, 100, 500]
    cuts = np.cumsum([0] + sizes)
    Yr, _, _ = refcpu.ref_run_ensemble(c, A.cells, X, rule=0, softmax=True)
    got = [None] * len(sizes)
    with es.PredictionService(c, A, rule, flush_timeout_ms=5) as svc:
        assert svc.wait_ready(60.0)

        def client(k):
            for i in range(k, len(sizes), 4):
                got[i] = svc.predict(X[cuts[i]:cuts[i + 1]])

        threads = [threading.Thread(target=client, args=(k,)) for k in range(4)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    Y = np.concatenate([g[0] for g in got])
    W = np.concatenate([g[1] for g in got])
    assert np.abs(Y - Yr).max() <= TOL_P
    assert_labels_identical_or_tied(W, Yr, TOL_P, "service vs reference pipeline")
