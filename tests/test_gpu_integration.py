"""The drop-in, end to end: the REFERENCE's own InferenceSystem
(src/runtime/pipeline.cpp, compiled from /root/reference) driving B200 members
through the INTEGRATION.md adapter (integration/enserve_b200_backend.cpp ->
es_member_create / es_member_predict), against the native device system and
the oracle."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import paper_2208_14049_b200 as es
from paper_2208_14049_b200 import api
from conftest import gpu
from oracle import refcpu, restate

pytestmark = pytest.mark.gpu
SO = refcpu.HERE / "_ref" / "libenserve_ref_b200.so"


@pytest.fixture(scope="module")
def reflib():
    if not SO.exists():
        pytest.skip("oracle/_ref/libenserve_ref_b200.so not built")
    lib = C.CDLL(str(SO))
    lib.ref_b200_run.restype = C.c_int
    lib.ref_b200_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_size_t,
                                 C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.ref_b200_greedy.restype = C.c_int
    lib.ref_b200_greedy.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_uint64,
                                    C.c_void_p, C.c_size_t, C.c_size_t, C.c_int, C.c_void_p,
                                    C.POINTER(C.c_double), C.POINTER(C.c_int)]
    return lib


def cluster2():
    models = [es.mlp_model(0, "a", [784, 256, 10], 301), es.mlp_model(1, "b", [784, 128, 10], 302)]
    return es.ClusterSpec([gpu(0, 180000.0, 1e15, 0.0), gpu(1, 180000.0, 1e15, 0.0)], models,
                          [8, 16, 32, 64, 128], 128)


def test_reference_pipeline_with_b200_backend_matches_native_system(reflib):
    c = cluster2()
    A = es.AllocationMatrix.from_array([[32, 64], [16, 0]])  # model 0 data-parallel
    nb = 700
    X = refcpu.features(12, nb, 784)
    Y = np.zeros((nb, 10), np.float32)
    W = np.zeros(nb, np.int32)
    with api._Desc(c) as d:
        rc = reflib.ref_b200_run(C.addressof(d.desc), A.cells.ctypes.data, 0,
                                 X.ctypes.data, nb, 784, Y.ctypes.data, W.ctypes.data, None)
    assert rc == 0
    native = es.run_inference(es.SampleStore(X), A, c, es.CombinationRule.averaging())
    # same member kernels, batched differently (per-batch compat vs persistent):
    # the member arithmetic does not depend on the tile, so bit-identical
    np.testing.assert_array_equal(Y, native.combined)
    want, _ = restate.fold("avg", [refcpu.CpuMlp([784, 256, 10], 301).forward(X),
                                   refcpu.CpuMlp([784, 128, 10], 302).forward(X)])
    np.testing.assert_array_equal(np.argmax(Y, 1), np.argmax(want, 1))


def test_reference_pipeline_reports_b200_oom_as_startup_error(reflib):
    c = cluster2()
    c.devices[0].memory_mib = 0.5  # the declared budget refuses the worker
    A = es.AllocationMatrix.from_array([[32, 64], [0, 0]])
    X = refcpu.features(1, 10, 784)
    Y = np.zeros((10, 10), np.float32)
    with api._Desc(c) as d:
        rc = reflib.ref_b200_run(C.addressof(d.desc), A.cells.ctypes.data, 0, X.ctypes.data, 10,
                                 784, Y.ctypes.data, None, None)
    assert rc == 3  # StartupError from the reference's Ready gate


def test_reference_greedy_with_the_b200_score(reflib):
    """The second half of the boundary: the reference's own
    bounded_greedy (optimizer.cpp:178-227, as cmd_optimize drives it,
    commands.cpp:76-94) scoring every candidate with make_b200_score -- the
    device-timed bench behind the C ABI.  It must walk a valid trajectory to a
    matrix at least as good as its start, with one bench call per matrix
    scored."""
    c = cluster2()
    A0 = es.worst_fit_decreasing(c, 8)
    X = refcpu.features(14, 4096, 784)
    out = np.zeros(A0.cells.size, np.int32)
    score, calls = C.c_double(), C.c_int()
    with api._Desc(c) as d:
        rc = reflib.ref_b200_greedy(C.addressof(d.desc), A0.cells.ctypes.data, 3, 6, 0,
                                    X.ctypes.data, 4096, 784, 1, out.ctypes.data,
                                    C.byref(score), C.byref(calls))
    assert rc == 0
    A = es.AllocationMatrix.from_array(out.reshape(A0.cells.shape).tolist())
    assert es.validate_matrix(A, c).ok
    start = es.bench(A0, es.SampleStore(X), c, 1).throughput
    assert score.value > 0 and score.value >= 0.8 * start
    assert 1 <= calls.value <= 1 + 3 * 6


def test_reference_pipeline_seam_throughput_at_cfg1(reflib):
    """Measured, not assumed: the reference's thread pipeline driving B200
    members one batch at a time through es_member_predict (H2D + member + D2H
    per batch of 32 on the predictor thread) at the cfg1 shape, next to the
    native persistent-kernel system on the same rows.  Printed for the record
    (profiles/r2*_seam.txt); asserted only to be positive and identical."""
    import time
    models = [es.mlp_model(0, "a", [784, 256, 10], 1), es.mlp_model(1, "b", [784, 256, 10], 2)]
    c = es.ClusterSpec([gpu(0, 180000.0, 1e15, 0.0)], models, [8, 16, 32, 64, 128], 128)
    A = es.AllocationMatrix.from_array([[32, 32]])
    nb = 1 << 16
    X = refcpu.features(15, nb, 784)
    Y = np.zeros((nb, 10), np.float32)
    el = C.c_double()
    with api._Desc(c) as d:
        t0 = time.perf_counter()
        rc = reflib.ref_b200_run(C.addressof(d.desc), A.cells.ctypes.data, 0, X.ctypes.data, nb,
                                 784, Y.ctypes.data, None, C.byref(el))
        wall = time.perf_counter() - t0
    assert rc == 0 and el.value > 0
    with es.InferenceSystem(A, c, es.CombinationRule.averaging()) as s:
        s.run(es.SampleStore(X))
        out = s.run(es.SampleStore(X))
        Yh = np.zeros((nb, 10), np.float32)
        e2e = s.run_host(X, Yh, None)
    np.testing.assert_array_equal(Y, out.combined)
    np.testing.assert_array_equal(Yh, out.combined)
    print(f"seam cfg1 nb={nb}: reference pipeline + b200 backend {nb / el.value:.4g} samples/s "
          f"(its window; {nb / wall:.4g} incl. startup), native run_host {nb / e2e:.4g}, "
          f"native resident {nb / out.stats.elapsed_s:.4g}")
