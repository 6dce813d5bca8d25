"""N > 1 plumbing on CPU (gloo, world_size 2): each rank derives its segment
shard from the library's partition (es.segment_shares), the shards cover every
segment exactly once, and the timing reduction is the max over ranks — the
same code bench.py runs under torchrun with NCCL."""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

REPO = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, str(REPO))
    import bench
    import paper_2208_14049_b200 as es
    dist = bench.Dist(backend="gloo")
    try:
        nb_per_gpu = 1000 + 37  # ragged: not a multiple of the segment size
        r0, r1, shares = bench.rank_shard(es, world, rank, [64, 64, 128, 128], nb_per_gpu)
        rows = dist.gather([r0, r1])
        t = dist.max(float(rank + 1) * 0.5)
        # bench.py: rank 0's optimized matrix reaches every rank.
        cells = dist.broadcast_object([[128, 64, 128, 32]] if rank == 0 else None)
        # The prediction gather's plan (InferenceSystem.set_gather): every
        # rank derives the same one; emulate the NCCL send/recv with gloo --
        # each rank's rows (labelled with their global row index) must land
        # at their place in rank 0's result.
        firsts, counts = bench.gather_plan(es, world, [64, 64, 128, 128], nb_per_gpu)
        plans = dist.gather([firsts, counts])
        import torch
        import torch.distributed as tdist
        mine = torch.arange(r0, r1, dtype=torch.int64)
        if rank == 0:
            result = torch.full((sum(counts),), -1, dtype=torch.int64)
            result[firsts[0]:firsts[0] + counts[0]] = mine
            for r in range(1, world):
                buf = torch.empty(counts[r], dtype=torch.int64)
                tdist.recv(buf, src=r)
                result[firsts[r]:firsts[r] + counts[r]] = buf
            gathered = result.tolist()
        else:
            tdist.send(mine, dst=0)
            gathered = None
        dist.barrier()
        q.put((rank, rows, t, shares, cells, plans, gathered))
    finally:
        dist.close()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_shards_cover_every_segment_once_and_max_time(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = world * 1037
    for rank, rows, t, shares, cells, plans, gathered in results:
        assert all(p == plans[0] for p in plans)  # one plan on every rank
        firsts, counts = plans[0]
        assert [(f, f + c) for f, c in zip(firsts, counts)] == [tuple(r) for r in rows]
        if rank == 0:
            assert gathered == list(range(total))  # every row once, in place
        assert t == pytest.approx(world * 0.5)  # max over ranks
        assert cells == [[128, 64, 128, 32]]
        spans = sorted(tuple(r) for r in rows)
        assert spans[0][0] == 0 and spans[-1][1] == total
        for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
            assert a1 == b0  # contiguous, no overlap, no gap
        assert len(shares) == 4  # one worker per member on this rank's device row


def test_segment_shares_exactly_once_for_mixed_layouts():
    sys.path.insert(0, str(REPO))
    import paper_2208_14049_b200 as es
    A = es.AllocationMatrix.from_array([[16, 0], [32, 8], [0, 64]])
    shares = es.segment_shares(A, 2000, 128)  # 16 segments
    assert [(d, m) for d, m, _, _ in shares] == [(0, 0), (1, 0), (1, 1), (2, 1)]
    for m in (0, 1):
        covered = []
        for d, mm, b, e in shares:
            if mm == m:
                covered += list(range(b, e))
        assert sorted(covered) == list(range(16))


def test_weighted_segment_shares_proportional_and_exactly_once():
    """SURVEY.md §8-E static fallback of the shared per-model FIFO: a model's
    data-parallel workers take contiguous runs proportional to their rates."""
    sys.path.insert(0, str(REPO))
    import paper_2208_14049_b200 as es
    A = es.AllocationMatrix.from_array([[16, 0], [32, 8], [0, 64], [128, 0]])
    S = 100  # 12800 rows / 128
    equal = es.segment_shares(A, 12800, 128)
    assert es.segment_shares(A, 12800, 128, [2.0] * 5) == equal  # equal weights: same split
    w = [1.0, 3.0, 5.0, 1.0, 4.0]  # workers (0,0) (1,0) (1,1) (2,1) (3,0)
    shares = es.segment_shares(A, 12800, 128, w)
    assert [(d, m) for d, m, _, _ in shares] == [(0, 0), (1, 0), (1, 1), (2, 1), (3, 0)]
    for m in (0, 1):
        mine = [(b, e, w[i]) for i, (d, mm, b, e) in enumerate(shares) if mm == m]
        assert mine[0][0] == 0 and mine[-1][1] == S
        for (a0, a1, _), (b0, b1, _) in zip(mine, mine[1:]):
            assert a1 == b0  # contiguous, exactly once, worker order kept
        tot = sum(x for _, _, x in mine)
        for b, e, x in mine:
            assert abs((e - b) - S * x / tot) <= 1.0
    # model 0: weights 1, 3, 4 of 8 -> cumulative 12.5, 50, 100 segments (half rounds up)
    assert [(b, e) for d, m, b, e in shares if m == 0] == [(0, 13), (13, 50), (50, 100)]
    import pytest
    with pytest.raises(es.InvalidArgument):
        es.segment_shares(A, 12800, 128, [1.0, 0.0, 1.0, 1.0, 1.0])
