"""Host core of the product (C++ behind the C ABI) against the reference:
ports of /root/reference/proj/tests/test_{core,memory,cost,optimizer}.cpp plus
bit-exact comparisons with the compiled reference (oracle/_ref) and the frozen
golden placements (tests/golden/placement.json)."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2208_14049_b200 as es
from conftest import (cpu, gpu, imagenet4_cluster, imagenet4_matrix, model, random_cluster,
                      tiny_cluster)
from oracle import refcpu, restate

need_ref = pytest.mark.skipif(not refcpu.ref_available(), reason="oracle/_ref not built")
GOLDEN = Path(__file__).resolve().parent / "golden"


def analytic(c):
    return lambda A: es.predict_ensemble_throughput(A, c)


# ------------------------------------------------------------- test_core.cpp
def test_validate_matrix_worked_allocation():
    v = es.validate_matrix(imagenet4_matrix(), imagenet4_cluster())
    assert v.ok and not v.violations and imagenet4_matrix().worker_count() == 5


def test_validate_matrix_flags_empty_columns_and_menu():
    v = es.validate_matrix(es.AllocationMatrix(5, 4), imagenet4_cluster())
    assert not v.ok and sum(x.kind == "EmptyColumn" for x in v.violations) == 4
    A = imagenet4_matrix()
    A.set(1, 0, 12)
    v = es.validate_matrix(A, imagenet4_cluster())
    assert not v.ok and len(v.violations) == 1
    x = v.violations[0]
    assert (x.kind, x.device, x.model, x.value) == ("EntryNotInMenu", 1, 0, 12)
    with pytest.raises(es.SpecError):
        es.validate_matrix(es.AllocationMatrix(2, 4), imagenet4_cluster())


def test_segments():
    assert es.segment_bounds(2, 128, 300) == (256, 300)
    assert es.segment_bounds(0, 128, 50) == (0, 50)
    assert es.segment_bounds(1, 128, 300) == (128, 256)
    with pytest.raises(es.InvalidArgument):
        es.segment_bounds(3, 128, 300)
    assert es.num_segments(300, 128) == 3 and es.num_segments(0, 128) == 0
    for nb in (1, 7, 127, 128, 129, 300, 1000):
        for N in (1, 8, 128):
            cursor = 0
            for s in range(es.num_segments(nb, N)):
                a, b = es.segment_bounds(s, N, nb)
                assert a == cursor and b > a and b - a <= N
                cursor = b
            assert cursor == nb


def test_row_and_column_counts():
    A = imagenet4_matrix()
    assert A.is_colocated(1) and not A.is_colocated(3)
    assert A.is_data_parallel(1) and not A.is_data_parallel(0)
    assert A.row_worker_count(0) == 0 and A.column_worker_count(1) == 2


def test_cluster_validation():
    c = imagenet4_cluster()
    assert c.validate() == []
    c.batch_menu = [8, 8]
    with pytest.raises(es.SpecError):
        c.validate()
    c = imagenet4_cluster()
    c.devices[1].memory_mib = 0
    with pytest.raises(es.SpecError):
        c.validate()
    c = imagenet4_cluster()
    c.segment_size = 64
    assert len(c.validate()) == 1


def test_cnn_member_spec_and_footprint():
    m = es.cnn_model(0, "cnn-s", 4)
    # conv 4x4/4 (16->64) and 3x3 (576->32) applied at 49 pixels, dense 1568->128->10.
    assert m.arch.layer_dims() == [(16, 64), (576, 32), (1568, 128), (128, 10)]
    assert m.arch.input_width() == 784
    assert m.cost_per_sample == 2 * (49 * 16 * 64 + 49 * 576 * 32 + 1568 * 128 + 128 * 10)
    assert m.arch.parameter_count() == 16 * 64 + 64 + 576 * 32 + 32 + 1568 * 128 + 128 + 1290
    c = es.ClusterSpec([es.DeviceSpec(0, es.GPU, 1000.0, 1.0, 0.0)], [m], [8, 16], 128)
    assert c.validate() == []
    bad = es.cnn_model(0, "cnn-bad", 4, S=30)  # patch 4 does not divide 30
    with pytest.raises(es.SpecError):
        es.ClusterSpec([es.DeviceSpec(0, es.GPU, 1000.0, 1.0, 0.0)], [bad], [8], 128).validate()
    wrong_c = es.cnn_model(0, "cnn-c", 4)
    wrong_c.output_width = 7
    with pytest.raises(es.SpecError):
        es.ClusterSpec([es.DeviceSpec(0, es.GPU, 1000.0, 1.0, 0.0)], [wrong_c], [8], 128).validate()


# ------------------------------------------------------------- test_memory.cpp
def test_memory_model():
    c = es.ClusterSpec([gpu(0, 16000.0)], [model(0, "a", 1000.0, 10.0), model(1, "b", 500.0, 2.0)],
                       [8, 128])
    A = es.AllocationMatrix(1, 2)
    assert es.fit_mem(A, c).used_mib == [0.0]
    A.set(0, 0, 8)
    assert es.fit_mem(A, c).used_mib == [pytest.approx(1080.0)]
    A.set(0, 1, 128)
    r = es.fit_mem(A, c)
    assert r.fits and r.used_mib == [pytest.approx(1836.0)]
    c.devices[0].memory_mib = 1000.0
    assert not es.fit_mem(A, c).fits


def test_more_remaining_memory():
    c = es.ClusterSpec([gpu(0, 32000.0), gpu(1, 16000.0)], [model(0, "a", 1000.0)], [8])
    A = es.AllocationMatrix(2, 1)
    assert es.more_remaining_memory(A, es.GPU, c) == 0
    c.devices[0].memory_mib = 16000.0
    assert es.more_remaining_memory(A, es.GPU, c) == 0  # tie -> lower id
    assert es.more_remaining_memory(A, es.CPU, c) is None
    c.devices[0].memory_mib = 32000.0
    A.set(0, 0, 8)
    assert es.more_remaining_memory(A, es.GPU, c) == 0
    c.devices[1].memory_mib = 31500.0
    assert es.more_remaining_memory(A, es.GPU, c) == 1


# ------------------------------------------------------------- test_cost.cpp
def test_cost_model():
    def rate1000(n):
        return es.ClusterSpec([gpu(d, 100000.0, 1000.0, 0.01) for d in range(n)],
                              [model(0, "m0", 100.0, 0.0, 1.0)], [8, 16, 32, 64, 128])
    c = rate1000(2)
    single = es.AllocationMatrix(2, 1)
    single.set(0, 0, 32)
    both = single.copy()
    both.set(1, 0, 32)
    assert es.predict_ensemble_throughput(both, c) == pytest.approx(
        2 * es.predict_ensemble_throughput(single, c))
    c = es.ClusterSpec([gpu(0, 1e5, 1000.0, 0.0), gpu(1, 1e5, 1000.0, 0.0)],
                       [model(0, "fast", 100.0, 0.0, 2.5), model(1, "slow", 100.0, 0.0, 10.0)],
                       [8, 16, 32, 64, 128])
    A = es.AllocationMatrix(2, 2)
    A.set(0, 0, 8)
    A.set(1, 1, 8)
    assert es.predict_ensemble_throughput(A, c) == pytest.approx(100.0)
    c = rate1000(1)
    c.devices[0].memory_mib = 50.0
    A = es.AllocationMatrix(1, 1)
    A.set(0, 0, 8)
    assert es.predict_ensemble_throughput(A, c) == 0.0


# ------------------------------------------------------------- test_optimizer.cpp
def test_wfd_examples():
    c = es.ClusterSpec([gpu(0, 16000.0)], [model(0, "m0", 1000.0, 10.0)], [8, 16, 32, 64, 128])
    A = es.worst_fit_decreasing(c, 8)
    assert A.at(0, 0) == 8 and A.worker_count() == 1
    c = es.ClusterSpec([cpu(0, 64000.0), gpu(1, 5000.0)],
                       [model(0, "fills-gpu", 4000.0), model(1, "spills", 2000.0)], [8])
    A = es.worst_fit_decreasing(c, 8)
    assert A.at(1, 0) == 8 and A.at(0, 1) == 8


def test_neighborhood_and_counts():
    c = tiny_cluster([8, 16], 1, 1)
    A = es.AllocationMatrix(1, 1)
    A.set(0, 0, 8)
    n = es.neighborhood(A, c)
    assert len(n) == 1 and n[0].at(0, 0) == 16
    c = tiny_cluster([8], 2, 1)
    A = es.AllocationMatrix(2, 1)
    A.set(0, 0, 8)
    n = es.neighborhood(A, c)
    assert len(n) == 1 and n[0].at(1, 0) == 8
    for B in es.neighborhood(imagenet4_matrix(), imagenet4_cluster()):
        assert es.validate_matrix(B, imagenet4_cluster()).ok
    assert es.count_total_matrices(5, 5, 8) == 13353748160923658642730712890625
    assert es.count_total_matrices(5, 1, 1) == 5 and es.count_total_matrices(1, 2, 1) == 3
    assert es.count_total_neighs(5, 5, 8, 8) == 232 and es.count_total_neighs(5, 5, 8, 0) == 240
    assert es.effective_max_iter(17, 1, 10) == 16 and es.effective_max_iter(5, 8, 10) == 10
    # cfg5 needs ~248 bits: (6^8 - 1)^12
    assert es.count_total_matrices(5, 8, 12) == (6 ** 8 - 1) ** 12


def test_enumeration():
    c = tiny_cluster([8], 2, 1)
    seen = {(A.at(0, 0), A.at(1, 0)) for A in es.enumerate_all_matrices(c, 100)}
    assert seen == {(0, 8), (8, 0), (8, 8)}
    for B in (1, 2):
        for D in (1, 2, 3):
            for M in (1, 2):
                c = tiny_cluster([8, 16][:B], D, M)
                all_ = es.enumerate_all_matrices(c, 100000)
                assert len(all_) == es.count_total_matrices(B, D, M)
                assert len({A.cells.tobytes() for A in all_}) == len(all_)
    c = imagenet4_cluster()
    c.models += [model(4 + i, f"x{i}", 100.0) for i in range(4)]
    with pytest.raises(es.CapExceededError):
        es.enumerate_all_matrices(c, 1000000)


def test_greedy_brute_force_optimum_and_plateau():
    c = tiny_cluster([8], 1, 1)
    A = es.AllocationMatrix(1, 1)
    A.set(0, 0, 8)
    r = es.bounded_greedy(A, c, "analytic", es.GreedyConfig(10, 100, 1))
    assert r.matrix == A and r.trace.stop_reason == "local_optimum"
    assert len(r.trace.iterations) == 1 and not r.trace.iterations[0].accepted
    c = tiny_cluster([8, 128], 2, 1)
    for d in c.devices:
        d.compute_rate, d.batch_overhead_s = 1000.0, 0.01
    best = max(es.enumerate_all_matrices(c, 100), key=lambda A: es.predict_ensemble_throughput(A, c))
    r = es.bounded_greedy(es.worst_fit_decreasing(c, 8), c, "analytic", es.GreedyConfig(10, 100, 42))
    assert r.matrix == best and best.at(0, 0) == 128 and best.at(1, 0) == 128


def test_greedy_budget_and_callback_bench():
    c = imagenet4_cluster()
    c.models += [model(4 + i, f"x{i}", 120.0, 4.0, 1.0 + i) for i in range(4)]
    calls = []

    def counted(A):
        calls.append(1)
        return es.predict_ensemble_throughput(A, c)
    r = es.bounded_greedy(es.worst_fit_decreasing(c, 8), c, counted, es.GreedyConfig(10, 100, 3))
    assert all(it.neighbors_evaluated <= 100 for it in r.trace.iterations)
    assert len(calls) <= 1001 and len(calls) == r.trace.bench_calls() == r.trace.calls


def test_bbs():
    c = es.ClusterSpec([gpu(0, 16000.0)], [model(0, "m0", 1000.0, 2.0, 1.0)], [8, 16, 32, 64, 128])
    r = es.bbs_baseline(c)
    assert r.bench_calls == 5 and r.matrix.at(0, 0) == 128
    c = imagenet4_cluster()
    c.devices = c.devices[1:]
    for i, d in enumerate(c.devices):
        d.id = i
    r = es.bbs_baseline(c)
    assert r.bench_calls == 20 and r.matrix.worker_count() == 4 and r.matrix.at(0, 3) > 0


def test_dozen_on_four_gpus_is_colocated():
    # acceptance.cpp:217-232 (SURVEY cfg3 packing)
    c = es.ClusterSpec([gpu(d, 16000.0) for d in range(4)],
                       [model(m, f"m{m}", 4600.0 - 100.0 * m, 10.0, 1.0 + m * 0.25)
                        for m in range(12)], [8, 16, 32, 64, 128])
    A = es.worst_fit_decreasing(c, 8)
    assert es.validate_matrix(A, c).ok and es.fit_mem(A, c).fits and A.worker_count() == 12
    assert all(A.is_colocated(d) for d in range(4))


# ------------------------------------------------------------- bit-exact vs reference
@need_ref
@pytest.mark.parametrize("seed", [5150, 31337, 777, 2024])
def test_wfd_greedy_scores_bit_identical_to_reference(seed):
    rng = restate.MT19937_64(seed)
    done = tries = 0
    while done < 40 and tries < 400:
        tries += 1
        c = random_cluster(rng)
        try:
            want = refcpu.ref_wfd(c, c.batch_menu[0])
        except refcpu.RefError as e:
            assert e.code == 2
            with pytest.raises(es.AllocationError):
                es.worst_fit_decreasing(c, c.batch_menu[0])
            continue
        got = es.worst_fit_decreasing(c, c.batch_menu[0])
        np.testing.assert_array_equal(got.cells, want)
        assert es.predict_ensemble_throughput(got, c) == refcpu.ref_throughput(c, want)
        assert es.fit_mem(got, c).used_mib == refcpu.ref_fit_mem(c, want)[0]
        n_mine = es.neighborhood(got, c)
        n_ref = refcpu.ref_neighborhood(c, want)
        assert [x.cells.tolist() for x in n_mine] == n_ref.tolist()
        gseed = rng()
        g_ref = refcpu.ref_greedy(c, want, 10, 5, gseed)  # small max_neighs: exercises sampling
        g = es.bounded_greedy(got, c, "analytic", es.GreedyConfig(10, 5, gseed))
        np.testing.assert_array_equal(g.matrix.cells, g_ref["matrix"])
        assert g.trace.final_score == g_ref["final"] and g.trace.start_score == g_ref["start"]
        assert [it.neighbors_evaluated for it in g.trace.iterations] == g_ref["neighbors"]
        assert [it.best_score for it in g.trace.iterations] == g_ref["best"]
        assert g.trace.stop_reason == g_ref["stop"] and g.trace.calls == g_ref["calls"]
        done += 1
    assert done >= 20


def test_placement_golden_fixtures():
    """The same bit-exactness against frozen reference outputs (no _ref needed)."""
    cases = json.loads((GOLDEN / "placement.json").read_text())["cases"]
    for case in cases:
        c = es.ClusterSpec(
            [es.DeviceSpec(i, k, mem, r, o) for i, (k, mem, r, o) in enumerate(case["devices"])],
            [es.ModelSpec(i, n, w, a, cst, 4) for i, (n, w, a, cst) in enumerate(case["models"])],
            case["menu"], 128)
        A = es.worst_fit_decreasing(c, c.batch_menu[0])
        assert A.cells.tolist() == case["wfd"]
        assert es.predict_ensemble_throughput(A, c) == case["wfd_score"]
        g = es.bounded_greedy(A, c, "analytic", es.GreedyConfig(10, 7, case["greedy_seed"]))
        assert g.matrix.cells.tolist() == case["greedy_matrix"]
        assert g.trace.final_score == case["greedy_final"]
        assert [it.neighbors_evaluated for it in g.trace.iterations] == case["greedy_neighbors"]
        assert g.trace.stop_reason == case["greedy_stop"]


@need_ref
def test_sample_indices_stream_matches_reference():
    for seed, n, k in [(0, 100, 10), (7, 228, 100), (1234, 468, 100), (3, 5, 10), (9, 1, 1)]:
        assert es.sample_indices(seed, n, k) == refcpu.ref_sample_indices(seed, n, k)


@need_ref
def test_bbs_matches_reference():
    c = imagenet4_cluster()
    c.devices = c.devices[1:]
    for i, d in enumerate(c.devices):
        d.id = i
    want = refcpu.ref_bbs(c)
    got = es.bbs_baseline(c)
    np.testing.assert_array_equal(got.matrix.cells, want["matrix"])
    assert got.chosen_batches == want["chosen"] and got.bench_calls == want["calls"]


def test_batcher_splits_segments_into_full_batches_plus_remainder():
    """test_runtime.cpp:315-332: 300 rows (segments 128, 128, 44) at b = 32 ->
    nine batches of 32 and one of 12; es.batch_rows is the tile space the
    fused-head kernels run (csrc/cuda/batching.cuh)."""
    import collections
    tiles = es.batch_rows(300, 128, 32)
    assert collections.Counter(r for _, r in tiles) == {32: 9, 12: 1}
    # every row once, in order, no tile crossing a segment boundary
    covered = [r0 + i for r0, r in tiles for i in range(r)]
    assert covered == list(range(300))
    for r0, r in tiles:
        assert r0 // 128 == (r0 + r - 1) // 128
    # a share of segments, odd batch and segment sizes, against a plain restatement
    rng = np.random.default_rng(4)
    for _ in range(50):
        seg = int(rng.integers(1, 300))
        nb = int(rng.integers(1, 5000))
        b = int(rng.integers(1, 129))
        S = (nb + seg - 1) // seg
        s0 = int(rng.integers(0, S))
        s1 = int(rng.integers(s0, S + 1))
        want = []
        for s in range(s0, s1):
            lo, hi = s * seg, min((s + 1) * seg, nb)
            want += [(r, min(b, hi - r)) for r in range(lo, hi, b)]
        assert es.batch_rows(nb, seg, b, s0, s1) == want
