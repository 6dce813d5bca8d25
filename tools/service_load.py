"""Closed-loop load on the deploy-mode service.

K client threads each submit requests of R rows back to back against the cfg2
ensemble for D seconds; reports samples/s, requests/s and latency
percentiles.  Usage: python tools/service_load.py [--clients 16] [--rows 4096]
[--seconds 5] [--flush-ms 2] [--config cfg2]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2208_14049_b200 as es  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--clients", type=int, default=16)
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--seconds", type=float, default=5.0)
    ap.add_argument("--flush-ms", type=int, default=2)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--matrix", default="128,128,128,128")
    ap.add_argument("--chunk", type=int, default=0, help="e2e_chunk_rows (0 = pool default)")
    ap.add_argument("--arena", type=int, default=-1, help="arena_rows (-1 = default)")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    cluster = bench.make_cluster(es, cfg)
    # The matrix bench.py's greedy picks for cfg2 (profiles/r1i_bench.json).
    A = es.AllocationMatrix.from_array([[int(b) for b in args.matrix.split(",")]])
    W = cluster.models[0].arch.input_width()
    rng = np.random.default_rng(0)
    pool = [rng.random((args.rows, W), dtype=np.float32) for _ in range(4)]
    lat: list = []
    lock = threading.Lock()
    stop_at = [0.0]
    with es.PredictionService(cluster, A, flush_timeout_ms=args.flush_ms, input_width=W,
                              e2e_chunk_rows=args.chunk, arena_rows=args.arena) as svc:
        assert svc.wait_ready(120.0), svc.startup_error
        svc.predict(pool[0])  # warm-up

        def client(i):
            k = i
            while time.perf_counter() < stop_at[0]:
                t0 = time.perf_counter()
                svc.predict(pool[k % 4])
                dt = time.perf_counter() - t0
                with lock:
                    lat.append(dt)
                k += 1

        base = svc.stats()
        t0 = time.perf_counter()
        stop_at[0] = t0 + args.seconds
        ts = [threading.Thread(target=client, args=(i,)) for i in range(args.clients)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        wall = time.perf_counter() - t0
        st = svc.stats()
    served = st.samples_served - base.samples_served
    lat_ms = np.array(lat) * 1e3
    print(json.dumps({
        "config": args.config, "matrix": A.cells.tolist(),
        "clients": args.clients, "chunk_rows": args.chunk, "arena_rows": args.arena, "rows_per_request": args.rows, "flush_timeout_ms": args.flush_ms,
        "samples_per_s": served / wall, "requests_per_s": len(lat) / wall,
        "flushes": st.flushes - base.flushes,
        "samples_per_flush": served / max(st.flushes - base.flushes, 1),
        "last_flush_device_samples_per_s": st.last_flush_throughput,
        "latency_ms": {"p50": float(np.percentile(lat_ms, 50)),
                       "p90": float(np.percentile(lat_ms, 90)),
                       "p99": float(np.percentile(lat_ms, 99))}}))


if __name__ == "__main__":
    main()
