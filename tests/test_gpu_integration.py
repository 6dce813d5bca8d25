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
                                 C.c_size_t, C.c_void_p, C.c_void_p]
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
                                 X.ctypes.data, nb, 784, Y.ctypes.data, W.ctypes.data)
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
                                 784, Y.ctypes.data, None)
    assert rc == 3  # StartupError from the reference's Ready gate
