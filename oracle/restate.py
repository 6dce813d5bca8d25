"""ORACLE — test infrastructure only (see oracle/__init__.py).

Plain-Python / numpy restatement of the reference's hot-path algorithms, each
citing the file:line it follows under /root/reference/proj.  Pinned by
tests/test_oracle.py against the reference's own known-answer tests (golden
values copied from tests/test_*.cpp, see tests/golden/) and against the
compiled reference (oracle/_ref).

Clusters are duck-typed: .devices[*].kind/memory_mib/compute_rate/
batch_overhead_s, .models[*].name/weight_mib/act_mib_per_sample/
cost_per_sample, .batch_menu, .segment_size.  Matrices are numpy int arrays.
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the engine of include/enserve/util/rng.hpp:13-38)."""
    NN, MM = 312, 156
    MATRIX_A = 0xB5026F5AA96619E9
    UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        mt = [0] * self.NN
        mt[0] = seed & MASK64
        for i in range(1, self.NN):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & MASK64
        self.mt, self.mti = mt, self.NN

    def _twist(self) -> None:
        mt, NN, MM = self.mt, self.NN, self.MM
        for i in range(NN):
            x = (mt[i] & self.UM) | (mt[(i + 1) % NN] & self.LM)
            mt[i] = mt[(i + MM) % NN] ^ (x >> 1) ^ (self.MATRIX_A if x & 1 else 0)
        self.mti = 0

    def __call__(self) -> int:
        if self.mti >= self.NN:
            self._twist()
        x = self.mt[self.mti]
        self.mti += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & MASK64


def uniform_index(rng: MT19937_64, n: int) -> int:
    """rng.hpp:13-22."""
    if n <= 1:
        return 0
    limit = MASK64 - MASK64 % n
    while True:
        x = rng()
        if x < limit:
            return x % n


def sample_indices(rng: MT19937_64, n: int, k: int) -> list:
    """rng.hpp:26-38."""
    idx = list(range(n))
    k = min(k, n)
    for i in range(k):
        j = i + uniform_index(rng, n - i)
        idx[i], idx[j] = idx[j], idx[i]
    return sorted(idx[:k])


def _kind(d) -> str:
    return "CPU" if str(d.kind).upper() == "CPU" else "GPU"


# ---------------------------------------------------------------- validation
def validate_matrix(A: np.ndarray, cluster) -> bool:
    """types.cpp:102-127 (ok flag only)."""
    A = np.asarray(A)
    menu = set(cluster.batch_menu)
    if any(int(b) != 0 and int(b) not in menu for b in A.ravel()):
        return False
    return bool(np.all(np.count_nonzero(A, axis=0) > 0))


def num_segments(nb: int, N: int) -> int:
    """types.cpp:129-134."""
    return 0 if nb == 0 else (nb + N - 1) // N


def segment_bounds(s: int, N: int, nb: int) -> tuple:
    """types.cpp:136-149."""
    start = s * N
    if start >= nb:
        raise IndexError("segment starts past the samples")
    return start, min(start + N, nb)


# ---------------------------------------------------------------- memory model
def worker_memory(model, b: int) -> float:
    """memory_model.cpp:7-10."""
    return model.weight_mib + b * model.act_mib_per_sample


def device_load(A: np.ndarray, d: int, cluster) -> float:
    """memory_model.cpp:12-20 — summed in model-id order."""
    used = 0.0
    for m in range(A.shape[1]):
        b = int(A[d, m])
        if b > 0:
            used += worker_memory(cluster.models[m], b)
    return used


def fit_mem(A: np.ndarray, cluster) -> tuple:
    """memory_model.cpp:22-32 -> (used per device, fits)."""
    used = [device_load(A, d, cluster) for d in range(len(cluster.devices))]
    fits = all(not (u > cluster.devices[d].memory_mib) for d, u in enumerate(used))
    return used, fits


def more_remaining_memory(A: np.ndarray, kind: str, cluster):
    """memory_model.cpp:34-50 — strict >, ties keep the lower id."""
    best, best_rem = None, 0.0
    for d, dev in enumerate(cluster.devices):
        if _kind(dev) != kind:
            continue
        rem = dev.memory_mib - device_load(A, d, cluster)
        if best is None or rem > best_rem:
            best, best_rem = d, rem
    return best


# ---------------------------------------------------------------- cost model
def service_time(m: int, d: int, b: int, n: int, cluster) -> float:
    """cost_model.cpp:13-20: b*c/(R/n) + o."""
    shared = cluster.devices[d].compute_rate / n
    return b * cluster.models[m].cost_per_sample / shared + cluster.devices[d].batch_overhead_s


def worker_throughput(m: int, d: int, b: int, n: int, cluster) -> float:
    """cost_model.cpp:22-27."""
    t = service_time(m, d, b, n, cluster)
    return math.inf if t <= 0.0 else b / t


def predict_ensemble_throughput(A: np.ndarray, cluster) -> float:
    """cost_model.cpp:29-46."""
    A = np.asarray(A)
    if not validate_matrix(A, cluster) or not fit_mem(A, cluster)[1]:
        return 0.0
    slowest = math.inf
    for m in range(A.shape[1]):
        rate = 0.0
        for d in range(A.shape[0]):
            b = int(A[d, m])
            if b:
                rate += worker_throughput(m, d, b, int(np.count_nonzero(A[d])), cluster)
        slowest = min(slowest, rate)
    return slowest


# ---------------------------------------------------------------- placement
def models_by_decreasing_weight(cluster) -> list:
    """optimizer.cpp:26-33 (stable: ties keep the lower id)."""
    return sorted(range(len(cluster.models)), key=lambda m: -cluster.models[m].weight_mib)


def worst_fit_decreasing(cluster, default_batch: int) -> np.ndarray:
    """optimizer.cpp:37-64.  Raises LookupError(model name) when nothing fits."""
    if default_batch not in cluster.batch_menu:
        raise ValueError("default batch not in menu")
    A = np.zeros((len(cluster.devices), len(cluster.models)), dtype=np.int32)
    for m in models_by_decreasing_weight(cluster):
        placed = False
        for kind in ("GPU", "CPU"):
            d = more_remaining_memory(A, kind, cluster)
            if d is None:
                continue
            cand = A.copy()
            cand[d, m] = default_batch
            if fit_mem(cand, cluster)[1]:
                A, placed = cand, True
                break
        if not placed:
            raise LookupError(cluster.models[m].name)
    return A


# ---------------------------------------------------------------- search
def neighborhood(A: np.ndarray, cluster) -> list:
    """optimizer.cpp:66-84: row-major cells, values {0}+menu ascending."""
    out = []
    D, M = A.shape
    for d in range(D):
        for m in range(M):
            cur = int(A[d, m])
            for v in [0] + list(cluster.batch_menu):
                if v == cur:
                    continue
                if v == 0 and np.count_nonzero(A[:, m]) == 1:
                    continue
                B = A.copy()
                B[d, m] = v
                out.append(B)
    return out


def count_total_matrices(B: int, D: int, M: int) -> int:
    """optimizer.cpp:105-111."""
    return ((B + 1) ** D - 1) ** M


def count_total_neighs(B: int, D: int, M: int, forbidden: int) -> int:
    """optimizer.cpp:113-118."""
    return (B + 1) * D * M - forbidden


def effective_max_iter(D: int, M: int, max_iter: int) -> int:
    """optimizer.cpp:173-176."""
    return max(D - M, max_iter)


def bounded_greedy(A0: np.ndarray, cluster, bench, max_iter=10, max_neighs=100, seed=0) -> dict:
    """optimizer.cpp:178-227."""
    rng = MT19937_64(seed)
    cur_A = np.asarray(A0).copy()
    current = bench(cur_A)
    trace = {"start": current, "neighbors": [], "best": [], "accepted": [], "stop": "iter_cap"}
    cap = effective_max_iter(len(cluster.devices), len(cluster.models), max_iter)
    calls = 1
    for _ in range(cap):
        neighs = neighborhood(cur_A, cluster)
        if len(neighs) > max_neighs:
            keep = sample_indices(rng, len(neighs), max_neighs)
            neighs = [neighs[i] for i in keep]
        best, best_score = None, 0.0
        for cand in neighs:
            s = bench(cand)
            calls += 1
            if best is None or s > best_score:
                best, best_score = cand, s
        accepted = best is not None and best_score > current
        trace["neighbors"].append(len(neighs))
        trace["best"].append(best_score)
        trace["accepted"].append(accepted)
        if not accepted:
            trace["stop"] = "local_optimum"
            break
        cur_A, current = best, best_score
    trace.update(final=current, matrix=cur_A, calls=calls)
    return trace


# ---------------------------------------------------------------- combine
def fold(rule: str, blocks, weights=None) -> tuple:
    """combine.cpp:93-136 over whole arrays: avg y += b*(1/M), wavg y += b*w_m,
    both with separately rounded fp32 multiply and add in model-id order; vote
    tallies per-model argmax (strict >).  Returns (y, argmax of y)."""
    blocks = [np.asarray(b, dtype=np.float32) for b in blocks]
    M = len(blocks)
    y = np.zeros_like(blocks[0])
    if rule in ("avg", "wavg"):
        inv = np.float32(1.0) / np.float32(M)
        for m, b in enumerate(blocks):
            w = inv if rule == "avg" else np.float32(weights[m])
            y = (y + (b * w).astype(np.float32)).astype(np.float32)
    else:
        rows = np.arange(y.shape[0])
        for b in blocks:
            y[rows, np.argmax(b, axis=1)] += np.float32(1.0)  # np.argmax: first max
    return y, np.argmax(y, axis=1).astype(np.int32)


def softmax_rows(z: np.ndarray) -> np.ndarray:
    """The combiner's per-member softmax (new in this build): fp32
    exp(z - max) / sum, sum in class order."""
    z = np.asarray(z, dtype=np.float32)
    e = np.exp((z - z.max(axis=1, keepdims=True)).astype(np.float32)).astype(np.float32)
    s = np.zeros(z.shape[0], dtype=np.float32)
    for c in range(z.shape[1]):
        s = (s + e[:, c]).astype(np.float32)
    inv = (np.float32(1.0) / s).astype(np.float32)
    return (e * inv[:, None]).astype(np.float32)


# ---------------------------------------------------------------- synthetic member
def splitmix64(x: int) -> int:
    """backend.cpp:12-17."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def synthetic_prediction(model_id: int, sample: int, cls: int) -> np.float32:
    """backend.cpp:21-29."""
    key = splitmix64(splitmix64(model_id + 1) ^ splitmix64((sample * 0x9E3779B9) & MASK64) ^
                     splitmix64(cls + 0x51ED270B))
    return np.float32(key >> 40) / np.float32(16777216.0)


def synthetic_block(model_id: int, rows: int, C: int, first: int = 0) -> np.ndarray:
    out = np.zeros((rows, C), dtype=np.float32)
    for r in range(rows):
        for c in range(C):
            out[r, c] = synthetic_prediction(model_id, first + r, c)
    return out
