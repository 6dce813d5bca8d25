#!/usr/bin/env python
"""Headline benchmark: ensemble samples/s (BASELINE.json `metric`).

Workload (N = 1): cfg2 of BASELINE.json — 4 heterogeneous MLP/CNN members
co-located on one B200 (SURVEY.md §8-D roster: MLP-256 784-256-10,
MLP-512-512 784-512-512-10, MLP-1024 784-1024-10, CNN-s 28x28 -> conv4x4/4
64 -> conv3x3 32 -> 128 -> 10), batch sizes chosen by the bounded greedy over
calib_data with the device-timed bench (worst-fit-decreasing start),
averaging of per-member softmax probabilities + argmax.  A "step" is one
InferenceSystem.run over `--nb` samples already resident in HBM (bf16
replica, > L2, so no flush is needed): 7 member kernels + 1 combine kernel.

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

# (name, kind, widths, weight seed[, weight_mib, act_mib]); SURVEY.md §8-D rosters.
ROSTER = [("mlp256", "mlp", [784, 256, 10], 11), ("mlp512x2", "mlp", [784, 512, 512, 10], 12),
          ("mlp1024", "mlp", [784, 1024, 10], 13), ("cnn-s", "cnn", [28, 4, 64, 32, 128, 10], 14)]
# The twelve of cfg3/cfg5: MLP widths 128..2048 and three CNNs, with the
# memory budgets of the reference's "dozen" acceptance spec (weights
# 4600 - 100 m MiB, 10 MiB per sample: tests/acceptance.cpp:217-225), so WFD
# packs them exactly as the reference does.
DOZEN = [("mlp2048", "mlp", [784, 2048, 10]), ("mlp1024x2", "mlp", [784, 1024, 1024, 10]),
         ("cnn-s", "cnn", [28, 4, 64, 32, 128, 10]), ("mlp1024", "mlp", [784, 1024, 10]),
         ("mlp512x2", "mlp", [784, 512, 512, 10]), ("cnn-w", "cnn", [28, 4, 32, 64, 256, 10]),
         ("mlp768", "mlp", [784, 768, 10]), ("mlp512", "mlp", [784, 512, 10]),
         ("mlp384x2", "mlp", [784, 384, 384, 10]), ("mlp256", "mlp", [784, 256, 10]),
         ("cnn-s2", "cnn", [28, 4, 64, 32, 128, 10]), ("mlp128", "mlp", [784, 128, 10])]
DOZEN = [(n, k, w, 31 + m, 4600.0 - 100.0 * m, 10.0) for m, (n, k, w) in enumerate(DOZEN)]
CONFIGS = {
    "cfg1": {"roster": [("mlp256a", "mlp", [784, 256, 10], 1), ("mlp256b", "mlp", [784, 256, 10], 2)],
             "devices": 1, "device_mib": 183359.0, "matrix": "fixed", "batches": [32, 32],
             "softmax": False,
             "workload": "cfg1: 2-member MLP ensemble (784-256-10 x 2), batch 32, averaging rule, "
                         "1 device, as run by the CPU reference"},
    "cfg2": {"roster": ROSTER, "devices": 1, "device_mib": 183359.0, "matrix": "greedy",
             "softmax": True, "ref_matrix": [[128, 128, 128, 128]],
             "workload": "cfg2: 4 heterogeneous MLP/CNN members (784-256-10, 784-512-512-10, "
                         "784-1024-10, CNN-s 28x28-c4x4/4:64-c3x3:32-128-10) co-located on 1 B200, "
                         "batches from bounded greedy over calib_data; avg of softmax + argmax"},
    "cfg3": {"roster": DOZEN, "devices": 4, "device_mib": 16000.0, "matrix": "wfd", "softmax": True,
             "workload": "cfg3: 12 heterogeneous members (MLP 128..2048 wide, 3 CNNs; reference "
                         "dozen memory spec) worst-fit-decreasing packed into 4 device rows; avg of "
                         "softmax + argmax"},
    "cfg4": {"roster": [("mlp2048x2", "mlp", [784, 2048, 2048, 10], 41)], "devices": 1,
             "device_mib": 183359.0, "matrix": "greedy", "softmax": True, "ref_matrix": [[128]],
             "workload": "cfg4: single DNN (MLP 784-2048-2048-10) data-parallel, per-GPU batch "
                         "slices; batch from bounded greedy (batch-size-only baseline applies)"},
    "cfg5": {"roster": DOZEN, "devices": 8, "device_mib": 16000.0, "matrix": "greedy",
             "softmax": True,
             # the device greedy's result on B200 (profiles/r1k_configs.json)
             "ref_matrix": [[8, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0], [0, 64, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0],
                            [0, 0, 64, 0, 0, 0, 128, 0, 0, 0, 0, 0], [0, 0, 0, 8, 0, 0, 0, 0, 0, 0, 0, 0],
                            [0, 0, 0, 0, 64, 128, 0, 0, 0, 0, 0, 8], [0, 0, 0, 0, 0, 8, 0, 128, 0, 0, 128, 0],
                            [128, 0, 0, 0, 0, 0, 8, 0, 0, 8, 0, 0], [0, 0, 0, 128, 0, 0, 0, 8, 64, 0, 0, 0]],
             "workload": "cfg5: full allocation optimizer sweep (worst-fit-decreasing + bounded "
                         "greedy, device-timed bench) for the 12-member ensemble on 8 device rows"},
}
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

    def broadcast_object(self, obj):
        """rank 0's picklable object on every rank."""
        if not self.pg:
            return obj
        box = [obj]
        self.pg.broadcast_object_list(box, src=0)
        return box[0]

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


def gather_plan(es, world: int, batches: list, nb_per_gpu: int, seg: int = 128) -> tuple:
    """(first row, rows) of every rank's shard in the gathered result --
    the plan InferenceSystem.set_gather receives on every rank."""
    spans = [rank_shard(es, world, r, batches, nb_per_gpu, seg)[:2] for r in range(world)]
    return [a for a, _ in spans], [b - a for a, b in spans]


# ------------------------------------------------------------------ workload
def roster_models(es, roster):
    out = []
    for i, r in enumerate(roster):
        name, kind, w, seed = r[:4]
        extra = {} if len(r) < 6 else {"weight_mib": r[4], "act_mib": r[5]}
        if kind == "cnn":
            out.append(es.cnn_model(i, name, seed, S=w[0], P=w[1], c1=w[2], c2=w[3], hidden=w[4],
                                    classes=w[5], **extra))
        else:
            out.append(es.mlp_model(i, name, w, seed, **extra))
    return out


def make_cluster(es, cfg: dict, devices: int = 0):
    models = roster_models(es, cfg["roster"])
    devs = [es.DeviceSpec(d, es.GPU, cfg["device_mib"], 1e15, 0.0)
            for d in range(devices or cfg["devices"])]
    return es.ClusterSpec(devs, models, list(MENU), 128)


def choose_matrix(es, cluster, cfg: dict, device_map: list, calib_nb: int, seed: int) -> dict:
    """A1 = WFD at the smallest batch; A2 = bounded greedy from A1 with the
    device-timed bench on calib ("greedy"), A1 itself ("wfd"), or the
    config's fixed batches ("fixed").  The batch-size-only baseline (BBS) is
    run wherever the reference's bbs_baseline applies."""
    calib = es.SampleStore(synthetic_seed=seed + 1, nb=calib_nb, width=784, device=device_map[0])
    t0 = time.time()
    A1 = es.worst_fit_decreasing(cluster, cluster.min_batch())
    score = lambda A: es.bench(A, calib, cluster, 3, device_map=device_map).throughput  # noqa: E731
    if cfg["matrix"] == "greedy":
        g = es.bounded_greedy(A1, cluster, es.DeviceBench(calib, 3, device_map=device_map),
                              es.GreedyConfig(10, 100, seed))
        A2, s1, s2, calls = g.matrix, g.trace.start_score, g.trace.final_score, g.trace.calls
    else:
        A2 = A1 if cfg["matrix"] == "wfd" else es.AllocationMatrix.from_array([cfg["batches"]])
        s1, s2, calls = score(A1), score(A2), 2
    bbs = {"applicable": False}
    try:
        r = es.bbs_baseline(cluster, es.DeviceBench(calib, 3, device_map=device_map))
        bbs = {"applicable": True, "matrix": r.matrix.cells.tolist(),
               "score": round(score(r.matrix), 1), "bench_calls": r.bench_calls,
               "chosen_batches": r.chosen_batches}
    except es.BaselineError as e:
        bbs = {"applicable": False, "reason": str(e)}
    return {"A1": A1, "A2": A2, "A1_score": s1, "A2_score": s2, "bench_calls": calls,
            "greedy_s": time.time() - t0, "bbs": bbs}


def cfg_classes(cfg: dict) -> int:
    return int(cfg["roster"][0][2][-1])


def launch_work(arch, names: list) -> list:
    """Algorithmic (FLOP, HBM bytes) per sample of each member launch, in
    launch order (DeviceMember::kernel_names): bytes = bf16 input row + the
    launch's output row (bf16 activations, fp32 logits); weights are read once
    per launch and amortised over the samples."""
    dims = arch.layer_dims()
    if arch.kind == "cnn":
        G2 = (arch.widths[0] // arch.widths[1]) ** 2
        flops = [2 * G2 * a * b if l < 2 else 2 * a * b for l, (a, b) in enumerate(dims)]
        widths = [arch.widths[0] ** 2, G2 * arch.widths[2], G2 * arch.widths[3]] + \
            [b for _, b in dims[2:]]
    else:
        flops = [2 * a * b for a, b in dims]
        widths = [dims[0][0]] + [b for _, b in dims]
    L = len(dims)
    out, l = [], 0
    for n in names:
        take = 2 if n.startswith(("conv_stack", "conv_rows", "conv_sweep")) or n.startswith("member_mlp2") or \
            n.startswith("mlp2_simt") or n.startswith("f32_conv") else 1
        f = float(sum(flops[l:l + take]))
        last = l + take == L
        b = widths[l] * 2 + widths[l + take] * (4 if last else 2)
        out.append((f, float(b)))
        l += take
    return out


# fp32 mode runs on the CUDA cores: nominal FP32 FMA rate of this part
# (148 SMs x 128 lanes x 2 FLOP x 1.965 GHz), no measured figure exists.
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def roofline_for(es, cluster, A, kernels: list, nb: int, pk: dict, pack: bool = False,
                 fp32: bool = False) -> dict:
    """Dominant kernel = the member launch with the largest device time.
    kernels: per worker [(name, ms)] averaged over the timed steps."""
    workers = [(d, m) for d in range(A.device_count()) for m in range(A.model_count())
               if A.at(d, m)]
    peak_t, peak_b = pk["bf16_tflops_sustained"], pk["hbm_gbs"]
    if fp32:
        peak_t = FP32_SIMT_TFLOPS
    ridge = peak_t * 1e12 / (peak_b * 1e9)
    traffic_db = {}
    try:
        traffic_db = json.loads(PROFILE_TRAFFIC.read_text())
    except Exception:
        pass
    per_kernel, best = [], None
    for j, (d, mm) in enumerate(workers):
        model = cluster.models[mm]
        work = launch_work(model.arch, [n for n, _ in kernels[j]])
        if fp32:  # 4-byte activations and inputs
            work = [(f, 2.0 * b) for f, b in work]
        for (name, ms), (f, b) in zip(kernels[j], work):
            tf = f * nb / (ms * 1e-3) / 1e12
            gbs = b * nb / (ms * 1e-3) / 1e9
            bound = "tensor" if f / b >= ridge else "hbm"
            frac = tf / peak_t if bound == "tensor" else gbs / peak_b
            row = {"member": model.name, "kernel": name, "batch": A.at(d, mm),
                   "ms": round(ms, 4), "tflops": round(tf, 1), "tensor_frac": round(tf / peak_t, 3),
                   "hbm_gbs": round(gbs, 1), "hbm_frac": round(gbs / peak_b, 3),
                   "flop_per_sample": f, "bytes_per_sample": b, "bound": bound,
                   "frac": round(frac, 4)}
            # A b-row batch is one M = 128 UMMA tile (the batcher's split), so
            # the fused heads' tensor ceiling at batch b is b/128 of peak.
            bt = A.at(d, mm) if not pack else 128
            if name.startswith("member_mlp2") and bt < 128:
                row["b_ceiling_frac"] = round(tf / (peak_t * bt / 128.0), 4)
            per_kernel.append(row)
            if best is None or ms > best["ms"]:
                best = row
    key = f"{best['member']}/{best['kernel']}"
    tensor = best["bound"] == "tensor"
    achieved = best["tflops"] if tensor else best["hbm_gbs"]
    peak = peak_t if tensor else peak_b
    return {"bound": best["bound"], "kernel": f"{best['kernel']}[{best['member']}]",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s" if tensor else "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic_db.get(key),
            "algorithmic_per_launch": {"flop": best["flop_per_sample"] * nb,
                                       "bytes": best["bytes_per_sample"] * nb,
                                       "flop_per_sample": best["flop_per_sample"],
                                       "bytes_per_sample": best["bytes_per_sample"],
                                       "samples": nb},
            "peak_source": ("nominal fp32 CUDA-core FMA rate (148 SMs x 128 lanes x 2 x 1.965 "
                            "GHz)" if fp32 and tensor else
                            f"{pk['source']} " + ("bf16 dense, sustained (kernel timed inside a "
                                                  "long step)" if tensor else "HBM copy")),
            "per_kernel": per_kernel}


# ------------------------------------------------------------------ CPU reference (no product)
class _Ns:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def _arch_footprint(kind: str, w: list) -> tuple:
    """(weight_mib, act_mib_per_sample, cost_per_sample) of a member shape —
    the product's derive_footprint (spec.cpp parameter_count /
    activation_elems / flops_per_sample) restated so the reference arm
    imports nothing from the product."""
    if kind == "cnn":
        S, P, c1, c2, hidden, Cn = w
        G2 = (S // P) ** 2
        dims = [(P * P, c1), (9 * c1, c2), (G2 * c2, hidden), (hidden, Cn)]
        flops = 2.0 * (G2 * dims[0][0] * dims[0][1] + G2 * dims[1][0] * dims[1][1] +
                       dims[2][0] * dims[2][1] + dims[3][0] * dims[3][1])
        act = S * S + G2 * (c1 + c2) + hidden + Cn
    else:
        dims = list(zip(w[:-1], w[1:]))
        flops = float(sum(2.0 * a * b for a, b in dims))
        act = float(sum(w))
    params = sum(a * b + b for a, b in dims)
    mib = 1024.0 * 1024.0
    return params * 2.0 / mib, act * 2.0 / mib, flops


def plain_cluster(cfg: dict, devices: int = 0, kind: str = "GPU"):
    """The config's cluster as plain Python objects (duck-typed for
    oracle/refcpu): the reference arm must not load the product."""
    models = []
    for i, r in enumerate(cfg["roster"]):
        name, k, w, seed = r[:4]
        wm, am, cost = _arch_footprint(k, list(w))
        if len(r) >= 6:
            wm, am = r[4], r[5]
        models.append(_Ns(id=i, name=name, weight_mib=wm, act_mib_per_sample=am,
                          cost_per_sample=cost, output_width=list(w)[-1],
                          arch=_Ns(kind=k, widths=tuple(w), weight_seed=seed)))
    n = devices or cfg["devices"]
    devs = [_Ns(id=d, kind=kind, memory_mib=cfg["device_mib"] if kind == "GPU" else 1e9,
                compute_rate=1e15 if kind == "GPU" else 1.0, batch_overhead_s=0.0)
            for d in range(n)]
    return _Ns(devices=devs, models=models, batch_menu=list(MENU), segment_size=128)


def reference_matrix(cfg: dict) -> list:
    """The matrix both arms run: the config's fixed batches, WFD (reference's
    own worst_fit_decreasing from oracle/_ref), or the matrix the device
    greedy reaches on B200 (recorded per config)."""
    from oracle import refcpu
    if cfg["matrix"] == "fixed":
        return [list(cfg["batches"])]
    if cfg["matrix"] == "wfd":
        return refcpu.ref_wfd(plain_cluster(cfg), MENU[0]).tolist()
    return [list(r) for r in cfg["ref_matrix"]]


def _timed_ref_runs(sysr, nb: int, budget_s: float, seed: int, steps: int = 3) -> tuple:
    """Size nb to ~budget_s / steps per run (one probe run), then time `steps`
    runs of the reference InferenceSystem; returns (nb, [samples/s])."""
    from oracle import refcpu
    X = refcpu.features(seed, nb, 784)
    el, _ = sysr.run(X)
    per = el / nb
    nb = int(min(max(nb, budget_s / steps / max(per, 1e-9)), 1 << 20))
    nb = max(128, nb // 128 * 128)
    X = refcpu.features(seed + 1, nb, 784)
    runs = []
    for _ in range(steps):
        el, _ = sysr.run(X)
        runs.append(nb / el)
    return nb, runs


def cpu_baseline(cfg: dict, A_cells, budget_s: float = 12.0, faithful_budget_s: float = 4.0) -> dict:
    """The reference InferenceSystem (compiled from /root/reference by
    oracle/Makefile) with the oracle CPU member, on this box's host cores
    (BASELINE.md §4):
      (ii) all-cores — every model data-parallel over floor(cores / M) CPU
           device rows (batch = its largest batch in A), the headline figure;
      (i)  matrix-faithful — exactly A (one CPU device per row of A), one
           compute thread per nonzero cell, as the reference would run it.
    Bounded samples; samples/s medians."""
    from oracle import refcpu
    cores = refcpu.host_cores()
    M = len(cfg["roster"])
    A = np.asarray(A_cells, dtype=np.int32)
    D = max(1, cores // M)
    allc = np.tile(A.max(axis=0), (D, 1)).astype(np.int32)
    sysr = refcpu.RefSystem(plain_cluster(cfg, D, "CPU"), allc, softmax=cfg["softmax"])
    nb, runs = _timed_ref_runs(sysr, 512 * D, budget_s, 5)
    sysr.close()
    return {"value": round(statistics.median(runs), 1), "unit": "samples/s", "cores": D * M,
            "kind": "reference",
            "sample": f"{nb} samples x 3 runs (median) of the reference InferenceSystem "
                      f"(pipeline.cpp, -O3) with the oracle CPU member (AVX2 fp32, bf16-quantised "
                      f"operands), matrix {allc.tolist()} over {D} CPU rows x {M} members "
                      f"= {D * M} compute threads on {cores} host cores",
            "matrix_faithful": cpu_matrix_faithful(cfg, A, faithful_budget_s)}


def cpu_matrix_faithful(cfg: dict, A_cells, budget_s: float = 4.0) -> dict:
    """BASELINE.md §4 figure (i): the reference InferenceSystem on exactly A
    (one CPU device per row of A, one compute thread per nonzero cell)."""
    from oracle import refcpu
    A = np.asarray(A_cells, dtype=np.int32)
    sysf = refcpu.RefSystem(plain_cluster(cfg, A.shape[0], "CPU"), A, softmax=cfg["softmax"])
    nbf, runs_f = _timed_ref_runs(sysf, 512, budget_s, 7)
    sysf.close()
    return {"value": round(statistics.median(runs_f), 1), "unit": "samples/s",
            "matrix": A.tolist(), "compute_threads": int((A > 0).sum()),
            "sample": f"{nbf} samples x 3 runs (median), one CPU device per row of A, one "
                      f"compute thread per worker"}


# ------------------------------------------------------------------ arms
def run_b200(args, dist: Dist) -> dict | None:
    import paper_2208_14049_b200 as es
    pk = peaks()
    gpu = dist.local
    cfg = CONFIGS[args.config]
    # Multi-row configs (cfg3: 4 rows, cfg5: 8) place members on device rows;
    # one process drives every visible GPU (row d -> GPU d mod count, logits
    # of remote rows peer-copied to the combining GPU).  Under torchrun rank 0
    # runs them and the other ranks only join the barriers.  Single-row
    # configs are replicated: each rank predicts its own segment shard.
    multirow = cfg["devices"] > 1
    ngpu = es.device_count()
    device_map = [d % ngpu for d in range(cfg["devices"])] if multirow else [gpu]
    cluster = make_cluster(es, cfg)
    if args.matrix:
        A = es.AllocationMatrix.from_array([[int(b) for b in r.split(",")]
                                            for r in args.matrix.split(";")])
        choice = {"A1": es.worst_fit_decreasing(cluster, cluster.min_batch()), "A2": A,
                  "A1_score": 0.0, "A2_score": 0.0, "bench_calls": 0,
                  "bbs": {"applicable": False, "reason": "matrix given on the command line"}}
    elif dist.rank != 0:
        choice = None  # rank 0 optimizes; single-row configs take its matrix below
    else:
        choice = choose_matrix(es, cluster, cfg, device_map, args.calib_nb, args.seed)
    if not multirow and dist.world > 1:
        # Every rank must run the SAME matrix (one cluster, N device rows):
        # rank 0's greedy result is broadcast.
        cells = dist.broadcast_object(choice["A2"].cells.tolist() if choice else None)
        if choice is None:
            A0 = es.AllocationMatrix.from_array(cells)
            choice = {"A1": A0, "A2": A0, "A1_score": 0.0, "A2_score": 0.0, "bench_calls": 0,
                      "bbs": {"applicable": False, "reason": "rank 0 optimizes"}}
    rule = es.CombinationRule.averaging(softmax=cfg["softmax"])
    active = not multirow or dist.rank == 0
    local_nb = 0
    if active:
        A = choice["A2"]
        if multirow:
            r0, r1 = 0, args.nb
        else:
            r0, r1, _ = rank_shard(es, dist.world, dist.rank, A.cells[0].tolist(), args.nb)
        local_nb = r1 - r0
        X = es.SampleStore(synthetic_seed=args.seed + dist.rank * 7919, nb=local_nb, width=784,
                           device=device_map[0])
        system = es.InferenceSystem(A, cluster, rule, device_map=device_map, copy_outputs=False,
                                    e2e_host_convert=bool(args.e2e_host_convert),
                                    pack_batches=args.pack_batches, fp32=args.fp32)
    gather, comm = None, None
    if not multirow and dist.world > 1 and args.gather:
        # The reference's accumulator sees every worker's predictions
        # (pipeline.cpp:210-211, :258-279): each rank's probabilities + argmax
        # go to rank 0 over NCCL after every run, inside the timed window.
        # Every rank must agree on using it: a rank whose setup failed makes
        # all ranks run without it (and the line says why).
        firsts, counts = gather_plan(es, dist.world, A.cells[0].tolist(), args.nb)
        err, uid = None, None
        if dist.rank == 0:
            try:
                uid = es.nccl_unique_id()
            except Exception as e:  # noqa: BLE001 -- reported in the JSON line
                err = f"{type(e).__name__}: {e}"
        uid = dist.broadcast_object(uid)
        if uid is None:
            err = err or "rank 0 could not create an NCCL unique id"
        else:
            try:
                comm = es.Comm(uid, dist.world, dist.rank, gpu)
                system.set_gather(comm, 0, firsts, counts)
            except Exception as e:  # noqa: BLE001 -- reported in the JSON line
                err = f"{type(e).__name__}: {e}"
        errs = [e for e in dist.gather([err]) if e[0] is not None]
        total = sum(counts)
        if errs:
            system.set_gather(None)
            gather = {"error": errs[0][0]}
        else:
            gather = {"collective": "NCCL grouped send/recv to rank 0 (probabilities + argmax)",
                      "bytes_per_step": total * (cfg_classes(cfg) * 4 + 4),
                      "rows_per_step": total, "nccl_version": es.nccl_version()}
    if active:
        for _ in range(args.warmup):
            system.run(X, copy=False)
    launches = 0
    step_s = []
    kern = []
    combine_ms = 0.0
    dist.barrier()
    with ClockSampler(gpu) as clocks:
        t0 = time.perf_counter()
        for _ in range(args.steps if active else 0):
            out = system.run(X, copy=False)
            step_s.append(out.stats.elapsed_s)
            launches += system.launches_last_run()
            combine_ms += system.timing()[1]
            kt = [system.kernel_timing(w) for w in range(system.worker_count())]
            kern = kt if not kern else [[(n, a + b) for (n, a), (_, b) in zip(k0, k1)]
                                        for k0, k1 in zip(kern, kt)]
        wall = time.perf_counter() - t0
    dist.barrier()
    device_s = dist.max(float(sum(step_s)))
    covered = sum(dist.gather([local_nb]), [])
    combine_ms /= max(1, args.steps)
    kern = [[(n, t / args.steps) for n, t in k] for k in kern]

    # e2e: host (pinned) X in, combined probabilities + labels out, per step
    # (run_host: one lane per GPU hosting workers, each over its own PCIe link).
    e2e = None
    if active:
        e2e_nb = max(1, min(args.e2e_nb, args.nb))
        try:
            import torch
            Xh = torch.empty((e2e_nb, 784), dtype=torch.float32, pin_memory=True).numpy()
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
    else:
        e2e_steps, e2e_nb = 0, 0
    dist.barrier()
    e2e_s, h2d, d2h = [], 0, 0
    for _ in range(e2e_steps):
        e2e_s.append(system.run_host(Xh, Yh, Lh))
        hb, db = system.last_transfer()
        h2d, d2h = h2d + hb, d2h + db
    dist.barrier()
    e2e_total = dist.max(float(sum(e2e_s)))
    e2e_ranks = sum(1 for v in dist.gather([len(e2e_s)]) if v[0] > 0)
    if e2e_steps:
        e2e = {"value": round(e2e_ranks * e2e_nb * e2e_steps / e2e_total, 1), "unit": "samples/s",
               "h2d_bytes_per_step": h2d // e2e_steps, "d2h_bytes_per_step": d2h // e2e_steps,
               "input": "pinned fp32 X; 6 of 8 chunks converted fp32->bf16 by host threads "
                        "(2 B/feature on the wire), the rest DMA'd as fp32 and converted on the "
                        "device (host-memory bandwidth bound)",
               "samples_per_step": e2e_nb}
    if active:
        system.close()
    if comm is not None:
        comm.close()  # after the system (which holds its own reference)

    if dist.rank != 0:
        return None
    n = dist.world
    value = sum(covered) * args.steps / device_s
    ngpus_used = len(set(device_map)) if multirow else n
    result = {
        "metric": "ensemble samples/sec at 1/2/4/8 B200 vs batch-only baseline and CPU ref",
        "value": round(value, 1),
        "unit": "samples/s",
        "n_gpus": n,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(device_s / args.steps * 1e3, 4),
        "higher_is_better": True,
        "scaling": "strong" if multirow else "weak",
        "vs_baseline": None,
        "dtype": "f32" if args.fp32 else "bf16",
        "data": "synthetic (U[0,1) features generated on device; Glorot-uniform synthetic weights)",
        "config": {
            "workload": cfg["workload"],
            "config": args.config,
            "samples_per_gpu_per_step": args.nb if not multirow else None,
            "samples_per_step": sum(covered),
            "x_bytes_per_gpu": args.nb * 784 * 2,
            "l2": "inputs (bf16 X) larger than L2, no flush",
            "device_rows": cfg["devices"],
            "device_map": device_map,
            "gpus_used": ngpus_used,
            "matrix_A1_wfd": choice["A1"].cells.tolist(),
            "matrix_A2": A.cells.tolist(),
            "matrix_rule": cfg["matrix"],
            "A1_score": round(choice["A1_score"], 1),
            "A2_score": round(choice["A2_score"], 1),
            "greedy_bench_calls": choice["bench_calls"],
            "calib_samples": args.calib_nb,
            "batch_only_baseline": choice["bbs"],
            "parallelism": (f"members placed on {cfg['devices']} device rows over {ngpus_used} "
                            f"GPU(s), remote logits stored into the combining GPU over NVLink "
                            f"peer mappings") if multirow
            else f"ensemble replicated per GPU, dp{n} over samples" +
            (", predictions gathered to rank 0 over NCCL inside the timed window" if gather else ""),
            "gather": gather,
            "segment_size": 128,
            "tiles": "whole segments (pack_batches)" if args.pack_batches
            else "one b-row batch per UMMA tile (the reference batcher's split)",
        },
        "roofline": roofline_for(es, cluster, A, kern, args.nb, pk, args.pack_batches, args.fp32),
        "member_ms": [round(sum(t for _, t in k), 4) for k in kern],
        "combine_ms": round(combine_ms, 4),
        "combine_hbm_gbs": round(args.nb * (len(cfg["roster"]) * 40 + 44) / (combine_ms * 1e-3) / 1e9, 1)
        if combine_ms > 0 else None,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "host_wall_s": round(wall, 4),
    }
    result["config"]["same_config"] = (cfg["matrix"] == "wfd" or
                                       A.cells.tolist() == reference_matrix(cfg))
    if args.cpu_baseline and n == 1:
        result["cpu_baseline"] = cpu_baseline(cfg, A.cells)
    return result


def run_reference(args, dist: Dist) -> dict | None:
    """The reference's own CPU implementation of the path on this box's host
    cores: its InferenceSystem (compiled from /root/reference sources into
    oracle/_ref) with the oracle CPU member — same config, matrix, metric and
    unit as the b200 arm; nothing from the product is imported.  W warm-up
    and K timed steps, each a bounded sample (all cores busy)."""
    if dist.rank != 0:
        return None
    from oracle import refcpu
    cfg = CONFIGS[args.config]
    A = np.asarray(reference_matrix(cfg), dtype=np.int32)
    cores = refcpu.host_cores()
    M = len(cfg["roster"])
    D = max(1, cores // M)
    allc = np.tile(A.max(axis=0), (D, 1)).astype(np.int32)
    sysr = refcpu.RefSystem(plain_cluster(cfg, D, "CPU"), allc, softmax=cfg["softmax"])
    # step size: the whole W + K run within ~args.ref_budget_s seconds
    per_step = max(0.5, args.ref_budget_s / max(1, args.steps + args.warmup))
    X = refcpu.features(5, 512 * D, 784)
    el, _ = sysr.run(X)
    nb = int(min(max(128, per_step / max(el / len(X), 1e-9)), 1 << 20)) // 128 * 128
    nb = max(128, nb)
    X = refcpu.features(6, nb, 784)
    for _ in range(args.warmup):
        sysr.run(X)
    times = []
    for _ in range(args.steps):
        el, _ = sysr.run(X)
        times.append(el)
    sysr.close()
    total = float(sum(times))
    value = nb * args.steps / total
    faithful = cpu_matrix_faithful(cfg, A) if args.ref_faithful else None
    return {
        "impl": "reference",
        "metric": "ensemble samples/sec at 1/2/4/8 B200 vs batch-only baseline and CPU ref",
        "value": round(value, 1), "unit": "samples/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (bf16-quantised operands)", "data": "synthetic (U[0,1) features; Glorot-uniform weights)",
        "config": {"workload": cfg["workload"] + " -- on host cores (reference runtime)",
                   "config": args.config, "matrix": A.tolist(), "same_config": True,
                   "samples_per_step": nb,
                   "note": "same roster, weights, matrix and rule as the b200 arm; each step a "
                           "bounded sample (the b200 arm runs 2^22 samples per step)"},
        "cpu_baseline": {"value": round(value, 1), "unit": "samples/s", "cores": D * M,
                         "kind": "reference",
                         "sample": f"{args.steps} steps x {nb} samples of the reference "
                                   f"InferenceSystem, matrix {allc.tolist()} ({D} CPU rows x "
                                   f"{M} members, {cores} host cores)",
                         "matrix_faithful": faithful},
        "e2e": {"value": round(value, 1), "unit": "samples/s", "h2d_bytes_per_step": 0,
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
                    help="profiling: batch per member, rows separated by ';' (e.g. 64,64,128,128), "
                         "skips the greedy")
    ap.add_argument("--ref-budget-s", type=float, default=120.0,
                    help="--impl reference: seconds for the whole warm-up + timed run")
    ap.add_argument("--no-ref-faithful", dest="ref_faithful", action="store_false",
                    help="--impl reference: skip the matrix-faithful figure")
    ap.add_argument("--no-gather", dest="gather", action="store_false",
                    help="N > 1: skip the NCCL prediction gather to rank 0")
    ap.add_argument("--fp32", action="store_true",
                    help="fp32-accurate members on the CUDA cores (PoolOptions.fp32)")
    ap.add_argument("--pack-batches", action="store_true",
                    help="tiles pack whole segments whatever the batch (PoolOptions.pack_batches)")
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS),
                    help="BASELINE.json config (default cfg2, the metric's config)")
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
