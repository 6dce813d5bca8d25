"""The multi-GPU data path.

The reference funnels every worker's predictions into one accumulator
(/root/reference/proj/src/runtime/pipeline.cpp:210-211, :258-279) and a
layout change never changes a result (tests/test_runtime.cpp:253-280).  Here:

* `row_nodes` lays an N-device matrix out on one GPU with the cross-device
  machinery intact -- every row its own stream, remote rows storing their
  logits into the combining node's buffers (route 1, the NVLink peer-store
  path) or through staging + cudaMemcpyPeerAsync (route 2), run_host with
  one lane per node -- and must be bit-identical to the one-node layout;
* the NCCL prediction gather (one process per GPU) is exercised with a
  one-rank communicator (the root's own rows) here, and over real ranks by
  `bench.py --gpus N`;
* with two or more visible GPUs, the same matrices over physical GPUs 0 and 1
  (peer access enabled, direct peer stores and staged copies) must be
  bit-identical to the one-GPU layout -- skipped on one-GPU boxes.
"""
from __future__ import annotations

import numpy as np
import pytest

import bench
import paper_2208_14049_b200 as es
from oracle import refcpu

pytestmark = pytest.mark.gpu

RULE = es.CombinationRule.averaging(softmax=True)
SMALL = [("mlp256", "mlp", [784, 256, 10], 11), ("mlp512x2", "mlp", [784, 512, 512, 10], 12),
         ("mlp128", "mlp", [784, 128, 10], 13), ("cnn-s", "cnn", [28, 4, 64, 32, 128, 10], 14)]


def cluster(devices, roster=SMALL, mib=183359.0):
    return bench.make_cluster(es, {"roster": roster, "devices": devices, "device_mib": mib})


# (name, cells): pure member placement over 3 rows, and data-parallel columns
LAYOUTS = [
    ("placed", [[128, 0, 0, 64], [0, 32, 0, 0], [0, 0, 128, 0]]),
    ("dp", [[128, 64, 0, 32], [64, 0, 128, 128], [0, 128, 32, 0]]),
]


def one_node(X, cells):
    A = es.AllocationMatrix.from_array(cells)
    return es.run_inference(X, A, cluster(len(cells)), RULE, device_map=[0] * len(cells))


@pytest.mark.parametrize("name,cells", LAYOUTS, ids=[n for n, _ in LAYOUTS])
@pytest.mark.parametrize("peer_stores", [True, False], ids=["direct", "staged"])
def test_row_nodes_bit_identical_to_one_node(name, cells, peer_stores):
    X = es.SampleStore(refcpu.features(61, 128 * 19 + 45, 784))
    ref = one_node(X, cells)
    A = es.AllocationMatrix.from_array(cells)
    with es.InferenceSystem(A, cluster(len(cells)), RULE, device_map=[0] * len(cells),
                            row_nodes=True, peer_stores=peer_stores, dp_equal_split=True) as s:
        routes, peers = s.routes()
        rows = [d for d in range(A.device_count()) for m in range(A.model_count()) if A.at(d, m)]
        want = [0 if r == rows[0] else (1 if peer_stores else 2) for r in rows]
        assert routes == want and peers == []
        out = s.run(X)
    np.testing.assert_array_equal(out.combined, ref.combined)
    np.testing.assert_array_equal(out.winners, ref.winners)


@pytest.mark.parametrize("name,cells", LAYOUTS, ids=[n for n, _ in LAYOUTS])
@pytest.mark.parametrize("peer_stores", [True, False], ids=["direct", "staged"])
def test_run_host_lanes_bit_identical_to_device_run(name, cells, peer_stores):
    """run_host over one lane per node (each lane receives only the rows its
    workers predict), 3 chunks of a ragged store, vs the resident run."""
    nb = 128 * 29 + 5
    Xh = refcpu.features(62, nb, 784)
    ref = one_node(es.SampleStore(Xh), cells)
    A = es.AllocationMatrix.from_array(cells)
    with es.InferenceSystem(A, cluster(len(cells)), RULE, device_map=[0] * len(cells),
                            row_nodes=True, peer_stores=peer_stores, dp_equal_split=True,
                            e2e_chunk_rows=1280) as s:
        Y = np.zeros((nb, 10), np.float32)
        L = np.zeros(nb, np.int32)
        s.run_host(Xh, Y, L)
        h2d, d2h = s.last_transfer()
    np.testing.assert_array_equal(Y, ref.combined)
    np.testing.assert_array_equal(L, ref.winners)
    assert d2h == nb * 44
    if name == "placed":  # every node hosts whole members: each lane receives every row
        assert h2d == 3 * nb * 784 * 2
    else:  # data-parallel runs: a lane receives only its workers' rows
        assert nb * 784 * 2 < h2d < 3 * nb * 784 * 2


def test_service_on_row_nodes_matches_offline():
    """The deploy-mode service flushes a multi-node pool through the run_host
    lanes (pinned arenas are portable across GPUs)."""
    cells = LAYOUTS[1][1]
    A = es.AllocationMatrix.from_array(cells)
    c = cluster(len(cells))
    X = refcpu.features(63, 700, 784)
    ref = one_node(es.SampleStore(X), cells)
    with es.PredictionService(c, A, RULE, flush_timeout_ms=5, device_map=[0] * len(cells),
                              row_nodes=True, dp_equal_split=True) as svc:
        assert svc.wait_ready(120.0)
        got = [svc.submit(X[a:a + 100]) for a in range(0, 700, 100)]
        Y = np.concatenate([g.result()[0] for g in got])
    np.testing.assert_array_equal(Y, ref.combined)


def test_nccl_gather_single_rank_returns_every_row():
    """set_gather with a one-rank communicator: the root's own rows are copied
    into the gathered result on the run's stream, inside the window."""
    cells = [[128, 64, 128, 32]]
    X = es.SampleStore(refcpu.features(64, 1000, 784))
    ref = one_node(X, cells)
    comm = es.Comm(es.nccl_unique_id(), 1, 0, 0)
    assert es.nccl_version() >= 22000
    with es.InferenceSystem(es.AllocationMatrix.from_array(cells), cluster(1), RULE,
                            device_map=[0]) as s:
        s.set_gather(comm, 0, [0], [1000])
        out = s.run(X)
        np.testing.assert_array_equal(out.combined, ref.combined)
        np.testing.assert_array_equal(out.winners, ref.winners)
        with pytest.raises(es.SpecError):  # the plan must match the store
            s.run(es.SampleStore(refcpu.features(65, 999, 784)))
        s.set_gather(None)
        out = s.run(X)
        np.testing.assert_array_equal(out.combined, ref.combined)
    comm.close()


def test_gather_plan_must_tile_exactly_once():
    comm = es.Comm(es.nccl_unique_id(), 1, 0, 0)
    with es.InferenceSystem(es.AllocationMatrix.from_array([[128, 64, 128, 32]]), cluster(1), RULE,
                            device_map=[0]) as s:
        with pytest.raises(es.SpecError):
            s.set_gather(comm, 0, [5], [100])  # does not start at row 0
        with pytest.raises(es.SpecError):
            s.set_gather(comm, 1, [0], [100])  # root out of range
    comm.close()


two_gpus = pytest.mark.skipif(es.device_count() < 2, reason="needs two visible GPUs")


@two_gpus
@pytest.mark.parametrize("name,cells", LAYOUTS, ids=[n for n, _ in LAYOUTS])
@pytest.mark.parametrize("peer_stores", [True, False], ids=["direct", "staged"])
def test_two_physical_gpus_bit_identical_to_one(name, cells, peer_stores):
    X = es.SampleStore(refcpu.features(66, 128 * 17 + 3, 784))
    ref = one_node(X, cells)
    A = es.AllocationMatrix.from_array(cells)
    dmap = [d % 2 for d in range(len(cells))]
    with es.InferenceSystem(A, cluster(len(cells)), RULE, device_map=dmap,
                            peer_stores=peer_stores, dp_equal_split=True) as s:
        routes, peers = s.routes()
        assert peers == [1]  # NVLink peer access enabled both ways
        out = s.run(X)
        nb = 128 * 17 + 3
        Y = np.zeros((nb, 10), np.float32)
        L = np.zeros(nb, np.int32)
        s.run_host(refcpu.features(66, nb, 784), Y, L)
    assert (1 if peer_stores else 2) in routes
    np.testing.assert_array_equal(out.combined, ref.combined)
    np.testing.assert_array_equal(out.winners, ref.winners)
    np.testing.assert_array_equal(Y, ref.combined)
    np.testing.assert_array_equal(L, ref.winners)
