#!/usr/bin/env python
"""Headline benchmark: ensemble samples/s (BASELINE.json `metric`).

Workload (N = 1): cfg2 of BASELINE.json — 4 heterogeneous MLP members
(784-512-10, 784-384-10, 784-256-10, 784-128-10) co-located on one B200,
batch sizes chosen by the bounded greedy over calib_data with the
device-timed bench (worst-fit-decreasing start), averaging of per-member
softmax probabilities + argmax.  A "step" is one InferenceSystem.run over
`--nb` samples already resident in HBM (bf16 replica, > L2, so no flush is
needed): 4 member kernels + 1 combine kernel.

N > 1 (torchrun, one process per GPU): the same ensemble replicated on every
GPU (each model data-parallel over the N devices), each rank runs its own
`--nb`-sample shard — no data-path collective; timing is the max over ranks
(weak scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

ROSTER = [("mlp512", [784, 512, 10], 11), ("mlp384", [784, 384, 10], 12),
          ("mlp256", [784, 256, 10], 13), ("mlp128", [784, 128, 10], 14)]
MENU = [8, 16, 32, 64, 128]
PEAKS_PATH = REPO / "MEASURED_PEAKS.json"
PROFILE_TRAFFIC = REPO / "profiles" / "roofline_traffic.json"


def peaks() -> dict:
    try:
        p = json.loads(PEAKS_PATH.read_text())
        return {"hbm_gbs": p["hbm_gbs"], "bf16_tflops": p["bf16_tflops"],
                "bf16_tflops_sustained": p.get("bf16_tflops_sustained", p["bf16_tflops"]),
                "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._proc = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            for line in self._proc.stdout:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 8:
                    self.rows.append(parts)
        except Exception:
            pass

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t.start()
            time.sleep(0.3)  # first sample lands before the timed region starts
        except Exception:
            self._proc = None
        return self

    def __exit__(self, *exc):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
            self._t.join(timeout=5)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ dist
class Dist:
    """One process per GPU (torchrun).  Plumbing only: a barrier around the
    timed region and the max-over-ranks of the device time.  The data path
    has no collective (each rank predicts its own segments)."""

    def __init__(self, backend: str | None = None):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = backend or os.environ.get("ES_DIST_BACKEND", "nccl")
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            if self.backend == "nccl":
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(self.backend)
            self.pg = dist

    def _device(self) -> str:
        return f"cuda:{self.local}" if self.backend == "nccl" else "cpu"

    def barrier(self):
        if self.pg:
            if self.backend == "nccl":
                import torch
                torch.cuda.synchronize()
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self._device())
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def gather(self, values: list) -> list:
        """All ranks' lists of ints (for the exactly-once check)."""
        if not self.pg:
            return [values]
        out = [None] * self.world
        self.pg.all_gather_object(out, values)
        return out

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


def rank_shard(es, world: int, rank: int, batches: list, nb_per_gpu: int, seg: int = 128):
    """Rows this rank predicts: the global matrix is `world` device rows, every
    member data-parallel over all of them; the library's own segment partition
    (es.segment_shares) assigns each rank a contiguous run of segments."""
    A = es.AllocationMatrix.from_array([list(batches)] * world)
    total = world * nb_per_gpu
    shares = [s for s in es.segment_shares(A, total, seg) if s[0] == rank]
    first = min(s[2] for s in shares)
    end = max(s[3] for s in shares)
    assert all((s[2], s[3]) == (first, end) for s in shares)
    return first * seg, min(end * seg, total), shares


# ------------------------------------------------------------------ workload
def make_cluster(es, devices: int = 1):
    models = [es.mlp_model(i, n, w, s) for i, (n, w, s) in enumerate(ROSTER)]
    devs = [es.DeviceSpec(d, es.GPU, 183359.0, 1e15, 0.0) for d in range(devices)]
    return es.ClusterSpec(devs, models, list(MENU), 128)


def choose_matrix(es, cluster, local_gpu: int, calib_nb: int, seed: int) -> dict:
    """WFD (A1) then bounded greedy (A2) with the device-timed bench on calib."""
    calib = es.SampleStore(synthetic_seed=seed + 1, nb=calib_nb, width=784, device=local_gpu)
    t0 = time.time()
    A1 = es.worst_fit_decreasing(cluster, cluster.min_batch())
    g = es.bounded_greedy(A1, cluster, es.DeviceBench(calib, 3, device_map=[local_gpu]),
                          es.GreedyConfig(10, 100, seed))
    bbs = {"applicable": False}
    try:
        es.bbs_baseline(cluster, es.DeviceBench(calib, 3, device_map=[local_gpu]))
    except es.BaselineError as e:
        bbs = {"applicable": False, "reason": str(e)}
    return {"A1": A1, "A2": g.matrix, "A1_score": g.trace.start_score,
            "A2_score": g.trace.final_score, "bench_calls": g.trace.calls,
            "greedy_s": time.time() - t0, "bbs": bbs}


def roofline_for(es, cluster, A, member_ms: list, nb: int, pk: dict) -> dict:
    """Dominant kernel = the member kernel with the largest device time."""
    i = int(np.argmax(member_ms))
    workers = [(d, m) for d in range(A.device_count()) for m in range(A.model_count())
               if A.at(d, m)]
    m = workers[i][1]
    arch = cluster.models[m].arch
    flops = arch.flops_per_sample() * nb
    achieved = flops / (member_ms[i] * 1e-3) / 1e12
    peak = pk["bf16_tflops_sustained"]
    traffic = None
    try:
        t = json.loads(PROFILE_TRAFFIC.read_text())
        traffic = t.get(cluster.models[m].name)
    except Exception:
        pass
    x_bytes = 784 * 2 * nb
    per_kernel = []
    for j, (d, mm) in enumerate(workers):
        a = cluster.models[mm].arch
        tf = a.flops_per_sample() * nb / (member_ms[j] * 1e-3) / 1e12
        gbs = (x_bytes + nb * 40) / (member_ms[j] * 1e-3) / 1e9
        per_kernel.append({"member": cluster.models[mm].name, "batch": A.at(d, mm),
                           "ms": round(member_ms[j], 4), "tflops": round(tf, 1),
                           "tensor_frac": round(tf / peak, 3), "hbm_gbs": round(gbs, 1),
                           "hbm_frac": round(gbs / pk["hbm_gbs"], 3)})
    return {"bound": "tensor", "kernel": f"member_mlp2_sm100[{cluster.models[m].name}]",
            "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "algorithmic_per_launch": {"flop": flops, "flop_per_sample": arch.flops_per_sample(),
                                       "samples": nb},
            "peak_source": f"{pk['source']} bf16 dense, sustained (kernel timed inside a long step)",
            "per_kernel": per_kernel}


def cpu_baseline(cluster, A_cells: np.ndarray, budget_s: float = 12.0) -> dict:
    """The reference InferenceSystem (compiled from /root/reference by
    oracle/Makefile) with the oracle CPU member, on this box's host cores:
    every model data-parallel over floor(cores / M) CPU 'devices' so all
    cores compute.  Bounded sample; returns samples/s."""
    from oracle import refcpu
    import paper_2208_14049_b200 as es
    cores = refcpu.host_cores()
    M = cluster.model_count()
    D = max(1, cores // M)
    cpu_cluster = es.ClusterSpec([es.DeviceSpec(d, es.CPU, 1e9, 1.0, 0.0) for d in range(D)],
                                 cluster.models, list(MENU), cluster.segment_size)
    A = np.tile(np.asarray(A_cells)[0], (D, 1)).astype(np.int32)
    sysr = refcpu.RefSystem(cpu_cluster, A, softmax=True)
    nb = 512 * D
    X = refcpu.features(5, nb, 784)
    el, _ = sysr.run(X)  # warm-up + size the sample to the budget
    per_sample = el / nb
    nb = int(min(max(nb, budget_s / 3 / max(per_sample, 1e-9)), 1 << 20))
    nb = max(128, nb // 128 * 128)
    X = refcpu.features(6, nb, 784)
    runs = []
    for _ in range(3):
        el, _ = sysr.run(X)
        runs.append(nb / el)
    sysr.close()
    return {"value": round(statistics.median(runs), 1), "unit": "samples/s", "cores": D * M,
            "kind": "reference",
            "sample": f"{nb} samples x 3 runs (median) of the reference InferenceSystem "
                      f"(pipeline.cpp, -O3) with the oracle CPU member (AVX2 fp32, bf16-quantised "
                      f"operands), matrix {A.tolist()} over {D} CPU rows x {M} members "
                      f"= {D * M} compute threads on {cores} host cores"}


# ------------------------------------------------------------------ arms
def run_b200(args, dist: Dist) -> dict | None:
    import paper_2208_14049_b200 as es
    pk = peaks()
    gpu = dist.local
    cluster = make_cluster(es)
    if args.matrix:
        A = es.AllocationMatrix.from_array([[int(b) for b in args.matrix.split(",")]])
        choice = {"A1": es.worst_fit_decreasing(cluster, cluster.min_batch()), "A2": A,
                  "A1_score": 0.0, "A2_score": 0.0, "bench_calls": 0,
                  "bbs": {"applicable": False, "reason": "matrix given on the command line"}}
    else:
        choice = choose_matrix(es, cluster, gpu, args.calib_nb, args.seed)
        A = choice["A2"]
    rule = es.CombinationRule.averaging(softmax=True)
    r0, r1, _ = rank_shard(es, dist.world, dist.rank, A.cells[0].tolist(), args.nb)
    local_nb = r1 - r0
    X = es.SampleStore(synthetic_seed=args.seed + dist.rank * 7919, nb=local_nb, width=784,
                       device=gpu)
    system = es.InferenceSystem(A, cluster, rule, device_map=[gpu], copy_outputs=False,
                                e2e_host_convert=bool(args.e2e_host_convert))
    for _ in range(args.warmup):
        system.run(X, copy=False)
    launches = 0
    step_s = []
    member_ms = np.zeros(system.worker_count())
    combine_ms = 0.0
    dist.barrier()
    with ClockSampler(gpu) as clocks:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            out = system.run(X, copy=False)
            step_s.append(out.stats.elapsed_s)
            launches += system.launches_last_run()
            ms, cm = system.timing()
            member_ms += np.asarray(ms)
            combine_ms += cm
        wall = time.perf_counter() - t0
    dist.barrier()
    device_s = dist.max(float(sum(step_s)))
    covered = sum(dist.gather([local_nb]), [])
    member_ms /= args.steps
    combine_ms /= args.steps

    # e2e: host (pinned) X in, combined probabilities + labels out, per step
    e2e_nb = max(1, min(args.e2e_nb, args.nb))
    try:
        import torch
        Xh_t = torch.empty((e2e_nb, 784), dtype=torch.float32, pin_memory=True)
        Xh = Xh_t.numpy()
        Yh = torch.empty((e2e_nb, 10), dtype=torch.float32, pin_memory=True).numpy()
        Lh = torch.empty((e2e_nb,), dtype=torch.int32, pin_memory=True).numpy()
    except Exception:
        Xh = np.empty((e2e_nb, 784), np.float32)
        Yh = np.empty((e2e_nb, 10), np.float32)
        Lh = np.empty(e2e_nb, np.int32)
    rng = np.random.default_rng(args.seed + dist.rank)
    Xh[:] = rng.random((e2e_nb, 784), dtype=np.float32)
    e2e_steps = args.steps if args.e2e else 1
    for _ in range(max(1, args.warmup // 2) if args.e2e else 0):
        system.run_host(Xh, Yh, Lh)
    dist.barrier()
    e2e_s = [system.run_host(Xh, Yh, Lh) for _ in range(e2e_steps)]
    dist.barrier()
    e2e_total = dist.max(float(sum(e2e_s)))
    system.close()

    if dist.rank != 0:
        return None
    n = dist.world
    value = sum(covered) * args.steps / device_s
    result = {
        "metric": "ensemble samples/sec at 1/2/4/8 B200 vs batch-only baseline and CPU ref",
        "value": round(value, 1),
        "unit": "samples/s",
        "n_gpus": n,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(device_s / args.steps * 1e3, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (U[0,1) features generated on device; Glorot-uniform synthetic weights)",
        "config": {
            "workload": "cfg2: 4 heterogeneous MLP members (784-{512,384,256,128}-10) co-located on "
                        "1 B200, batches from bounded greedy over calib_data; avg of softmax + argmax",
            "samples_per_gpu_per_step": args.nb,
            "x_bytes_per_gpu": args.nb * 784 * 2,
            "l2": "inputs (bf16 X) larger than L2, no flush",
            "matrix_A1_wfd": choice["A1"].cells.tolist(),
            "matrix_A2_greedy": A.cells.tolist(),
            "A1_score": round(choice["A1_score"], 1),
            "A2_score": round(choice["A2_score"], 1),
            "greedy_bench_calls": choice["bench_calls"],
            "calib_samples": args.calib_nb,
            "batch_only_baseline": choice["bbs"],
            "parallelism": f"ensemble replicated per GPU, dp{n} over samples",
            "segment_size": 128,
        },
        "roofline": roofline_for(es, cluster, A, list(member_ms), args.nb, pk),
        "combine_ms": round(combine_ms, 4),
        "combine_hbm_gbs": round(args.nb * (4 * 40 + 44) / (combine_ms * 1e-3) / 1e9, 1)
        if combine_ms > 0 else None,
        "e2e": {"value": round(n * e2e_nb * e2e_steps / e2e_total, 1), "unit": "samples/s",
                "h2d_bytes_per_step": e2e_nb * 784 * 4,
                "d2h_bytes_per_step": e2e_nb * (10 * 4 + 4),
                "samples_per_step": e2e_nb},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "host_wall_s": round(wall, 4),
    }
    if args.cpu_baseline and n == 1:
        result["cpu_baseline"] = cpu_baseline(cluster, A.cells)
    return result


def run_reference(args, dist: Dist) -> dict | None:
    """The reference's own CPU implementation of the path on this box's host
    cores: its InferenceSystem (compiled from /root/reference sources into
    oracle/_ref) with the oracle CPU member — same config, metric and unit."""
    if dist.rank != 0:
        return None
    import paper_2208_14049_b200 as es
    from oracle import refcpu
    cluster = make_cluster(es)
    # The reference cannot time a GPU bench: take the b200 arm's default matrix
    # shape with the batch sizes WFD gives (A1), which is what the reference's
    # optimizer starts from.
    A1 = es.worst_fit_decreasing(cluster, 32)
    base = cpu_baseline(cluster, A1.cells, budget_s=max(4.0, 2.0 * args.steps))
    value = base["value"]
    return {
        "impl": "reference",
        "metric": "ensemble samples/sec at 1/2/4/8 B200 vs batch-only baseline and CPU ref",
        "value": value, "unit": "samples/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (bf16-quantised operands)",
        "data": "synthetic", "config": {"workload": "cfg2 roster on host cores (reference runtime)"},
        "cpu_baseline": base,
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--nb", type=int, default=1 << 22)
    ap.add_argument("--e2e-nb", type=int, default=1 << 20)
    ap.add_argument("--calib-nb", type=int, default=1 << 16)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false",
                    help="profiling: a single e2e step")
    ap.add_argument("--e2e-host-convert", type=int, default=1,
                    help="e2e: 1 = host fp32->bf16 before the H2D copy, 0 = fp32 over PCIe")
    ap.add_argument("--matrix", default="",
                    help="profiling: batch per member (e.g. 64,64,128,128), skips the greedy")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    dist = Dist()
    try:
        res = run_b200(args, dist) if args.impl == "b200" else run_reference(args, dist)
    finally:
        dist.close()
    if res is not None:
        print(json.dumps(res))


if __name__ == "__main__":
    main()
