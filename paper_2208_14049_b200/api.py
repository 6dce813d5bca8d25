"""Python mirror of the enserve API over the enserve-b200 C ABI.

Names, argument meaning and raised error classes follow the reference's C++
API (/root/reference/proj/include/enserve/**; file:line on each item), so the
parity tests read like the reference's own doctest suites.  All work happens in
libenserve_b200.so (C++ host core + sm_100a kernels); this module only marshals.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import lib


# ------------------------------------------------------------------ errors
class EnserveError(RuntimeError):
    """enserve::Error (include/enserve/core/errors.hpp:9-12)."""


class SpecError(EnserveError):
    """errors.hpp:16-19."""


class AllocationError(EnserveError):
    """errors.hpp:22-27; .model_name parsed from the message."""

    @property
    def model_name(self) -> str:
        msg = str(self)
        return msg.split("'")[1] if "'" in msg else ""


class BaselineError(EnserveError):
    """errors.hpp:30-33."""


class CapExceededError(EnserveError):
    """errors.hpp:36-39."""


class StartupError(EnserveError):
    """errors.hpp:42-45."""


class ProtocolError(EnserveError):
    """errors.hpp:48-51."""


class DeviceError(EnserveError):
    """CUDA failure other than out-of-memory (no reference counterpart)."""


class NotReadyError(EnserveError):
    """The service is still loading or has stopped (the reference server's 503)."""


class InvalidArgument(ValueError):
    """std::invalid_argument / std::out_of_range thrown by the reference."""


_STATUS = {1: InvalidArgument, 2: SpecError, 3: AllocationError, 4: StartupError,
           5: BaselineError, 6: CapExceededError, 7: ProtocolError, 8: DeviceError,
           9: EnserveError, 10: EnserveError, 11: NotReadyError}


def _check(status: int) -> None:
    if status != 0:
        msg = lib().es_last_error().decode(errors="replace")
        raise _STATUS.get(status, EnserveError)(msg)


# K3 combine limits (csrc/cuda/aux_kernels.cuh kMaxMembers / kMaxClasses).
MAX_MEMBERS = 32
MAX_CLASSES = 16


def _require_out(a, dtype, shape: tuple, what: str) -> None:
    """An output array the C side writes rows * C elements into: it must have
    exactly that dtype, shape and C-contiguous layout (None = not wanted)."""
    if a is None:
        return
    if not isinstance(a, np.ndarray) or a.dtype != dtype or a.shape != shape or \
            not a.flags.c_contiguous or not a.flags.writeable:
        got = (a.dtype, a.shape) if isinstance(a, np.ndarray) else type(a).__name__
        raise InvalidArgument(f"{what} must be a writable C-contiguous {np.dtype(dtype).name} "
                              f"array of shape {shape}, got {got}")


# ------------------------------------------------------------------ specs
GPU, CPU = "GPU", "CPU"


@dataclass
class DeviceSpec:
    """types.hpp:17-26."""
    id: int = 0
    kind: str = GPU
    memory_mib: float = 0.0
    compute_rate: float = 0.0
    batch_overhead_s: float = 0.0

    def label(self) -> str:
        return ("gpu" if self.kind == GPU else "cpu") + str(self.id)


@dataclass
class MemberArch:
    """What the device executes for a member (spec.hpp MemberArch).

    kind "synthetic": synthetic_prediction(model, sample, class)
    (src/runtime/backend.cpp:21-29); kind "mlp": dense layers over `widths`;
    kind "cnn": widths = (S, P, c1, c2, hidden, classes) -- an S x S image,
    conv PxP stride P -> c1, conv 3x3 pad 1 -> c2, dense -> hidden -> classes.
    """
    kind: str = "synthetic"
    widths: tuple = ()
    weight_seed: int = 0

    def layer_dims(self) -> list:
        """(fan_in, fan_out) of every weight matrix, in generation order."""
        w = self.widths
        if self.kind == "cnn":
            S, P, c1, c2, hidden, C = w
            G = S // P
            return [(P * P, c1), (9 * c1, c2), (G * G * c2, hidden), (hidden, C)]
        return list(zip(w[:-1], w[1:]))

    def input_width(self) -> int:
        return self.widths[0] ** 2 if self.kind == "cnn" else self.widths[0]

    def flops_per_sample(self) -> float:
        d = self.layer_dims()
        if self.kind == "cnn":
            G2 = (self.widths[0] // self.widths[1]) ** 2
            return float(2 * (G2 * d[0][0] * d[0][1] + G2 * d[1][0] * d[1][1]
                              + d[2][0] * d[2][1] + d[3][0] * d[3][1]))
        return float(sum(2 * a * b for a, b in d))

    def parameter_count(self) -> int:
        return int(sum(a * b + b for a, b in self.layer_dims()))

    def activation_elems(self) -> int:
        if self.kind == "cnn":
            S, P, c1, c2, hidden, C = self.widths
            return S * S + (S // P) ** 2 * (c1 + c2) + hidden + C
        return int(sum(self.widths))


@dataclass
class ModelSpec:
    """types.hpp:28-35 (+ arch)."""
    id: int = 0
    name: str = ""
    weight_mib: float = 0.0
    act_mib_per_sample: float = 0.0
    cost_per_sample: float = 0.0
    output_width: int = 1
    arch: MemberArch = field(default_factory=MemberArch)
    # B200 calibration (extension): 1/throughput(b) = b200_cost_s + b200_overhead_s/b
    b200_cost_s: float = 0.0
    b200_overhead_s: float = 0.0


def mlp_model(id: int, name: str, widths: Sequence[int], seed: int, *,
              weight_mib: Optional[float] = None, act_mib: Optional[float] = None,
              cost: Optional[float] = None) -> ModelSpec:
    """A ModelSpec whose footprint is derived from its MLP shape (bf16 weights
    and activations), unless given explicitly (runtime.cpp derive_footprint)."""
    arch = MemberArch("mlp", tuple(int(w) for w in widths), int(seed))
    mib = 1024.0 * 1024.0
    return ModelSpec(
        id=id, name=name,
        weight_mib=weight_mib if weight_mib is not None else arch.parameter_count() * 2 / mib,
        act_mib_per_sample=act_mib if act_mib is not None else sum(widths) * 2 / mib,
        cost_per_sample=cost if cost is not None else arch.flops_per_sample(),
        output_width=int(widths[-1]), arch=arch)


def cnn_model(id: int, name: str, seed: int, *, S: int = 28, P: int = 4, c1: int = 64,
              c2: int = 32, hidden: int = 128, classes: int = 10,
              weight_mib: Optional[float] = None, act_mib: Optional[float] = None,
              cost: Optional[float] = None) -> ModelSpec:
    """A CNN member ("CNN-s" by default: 28x28 -> conv4x4/4 64 -> conv3x3 32 ->
    128 -> 10), footprint derived like mlp_model's."""
    arch = MemberArch("cnn", (int(S), int(P), int(c1), int(c2), int(hidden), int(classes)),
                      int(seed))
    mib = 1024.0 * 1024.0
    return ModelSpec(
        id=id, name=name,
        weight_mib=weight_mib if weight_mib is not None else arch.parameter_count() * 2 / mib,
        act_mib_per_sample=act_mib if act_mib is not None else arch.activation_elems() * 2 / mib,
        cost_per_sample=cost if cost is not None else arch.flops_per_sample(),
        output_width=int(classes), arch=arch)


@dataclass
class ClusterSpec:
    """types.hpp:38-52."""
    devices: list = field(default_factory=list)
    models: list = field(default_factory=list)
    batch_menu: list = field(default_factory=list)
    segment_size: int = 128

    def device_count(self) -> int:
        return len(self.devices)

    def model_count(self) -> int:
        return len(self.models)

    def min_batch(self) -> int:
        if not self.batch_menu:
            raise SpecError("batch menu is empty")
        return self.batch_menu[0]

    def validate(self) -> list:
        buf = C.create_string_buffer(4096)
        with _Desc(self) as d:
            _check(lib().es_cluster_validate(d.ptr, buf, len(buf)))
        return [w for w in buf.value.decode().split("\n") if w]


class _Desc:
    """Keeps the ctypes cluster descriptor and its arrays alive."""

    def __init__(self, c: ClusterSpec):
        nd, nm = len(c.devices), len(c.models)
        self.devs = (_abi.DeviceDesc * max(nd, 1))()
        for i, d in enumerate(c.devices):
            self.devs[i] = _abi.DeviceDesc(0 if d.kind == CPU else 1, d.memory_mib,
                                           d.compute_rate, d.batch_overhead_s)
        self.models = (_abi.ModelDesc * max(nm, 1))()
        self.names = [m.name.encode() for m in c.models]
        for i, m in enumerate(c.models):
            md = self.models[i]
            md.name = self.names[i]
            md.weight_mib = m.weight_mib
            md.act_mib_per_sample = m.act_mib_per_sample
            md.cost_per_sample = m.cost_per_sample
            md.output_width = m.output_width
            md.arch = {"mlp": 1, "cnn": 2}.get(m.arch.kind, 0)
            md.n_widths = len(m.arch.widths)
            for j, w in enumerate(m.arch.widths):
                md.widths[j] = int(w)
            md.weight_seed = int(m.arch.weight_seed)
            md.b200_cost_s = m.b200_cost_s
            md.b200_overhead_s = m.b200_overhead_s
        self.menu = (C.c_int * max(len(c.batch_menu), 1))(*c.batch_menu)
        self.desc = _abi.ClusterDesc(self.devs, nd, self.models, nm, self.menu,
                                     len(c.batch_menu), c.segment_size)
        self.ptr = C.byref(self.desc)
        self.D, self.M = nd, nm

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


# ------------------------------------------------------------------ matrix
class AllocationMatrix:
    """D x M batch grid, 0 = no worker (types.hpp:55-88)."""

    def __init__(self, devices: int = 0, models: int = 0, cells=None):
        if cells is not None:
            self.cells = np.ascontiguousarray(np.asarray(cells, dtype=np.int32).reshape(devices, models))
        else:
            self.cells = np.zeros((devices, models), dtype=np.int32)

    @classmethod
    def from_array(cls, a) -> "AllocationMatrix":
        a = np.asarray(a, dtype=np.int32)
        return cls(a.shape[0], a.shape[1], a)

    def device_count(self) -> int:
        return self.cells.shape[0]

    def model_count(self) -> int:
        return self.cells.shape[1]

    def at(self, d: int, m: int) -> int:
        return int(self.cells[d, m])

    def set(self, d: int, m: int, b: int) -> None:
        self.cells[d, m] = b

    def worker_count(self) -> int:
        return int(np.count_nonzero(self.cells))

    def row_worker_count(self, d: int) -> int:
        return int(np.count_nonzero(self.cells[d]))

    def column_worker_count(self, m: int) -> int:
        return int(np.count_nonzero(self.cells[:, m]))

    def is_data_parallel(self, m: int) -> bool:
        return self.column_worker_count(m) >= 2

    def is_colocated(self, d: int) -> bool:
        return self.row_worker_count(d) >= 2

    def copy(self) -> "AllocationMatrix":
        return AllocationMatrix.from_array(self.cells.copy())

    def ptr(self):
        return self.cells.ctypes.data_as(_abi.c_int_p)

    def __eq__(self, other) -> bool:
        return isinstance(other, AllocationMatrix) and self.cells.shape == other.cells.shape and \
            bool(np.array_equal(self.cells, other.cells))

    def __repr__(self) -> str:
        return f"AllocationMatrix({self.cells.tolist()})"


@dataclass
class MatrixViolation:
    kind: str  # "EntryNotInMenu" | "EmptyColumn"
    device: int
    model: int
    value: int


@dataclass
class MatrixValidation:
    ok: bool
    violations: list


def validate_matrix(A: AllocationMatrix, cluster: ClusterSpec) -> MatrixValidation:
    """types.cpp:102-127."""
    if A.device_count() != cluster.device_count() or A.model_count() != cluster.model_count():
        raise SpecError(f"matrix is {A.device_count()}x{A.model_count()} but the cluster has "
                        f"{cluster.device_count()} devices and {cluster.model_count()} models")
    cap = A.cells.size + A.model_count() + 1
    buf = (C.c_int * (4 * cap))()
    ok, n = C.c_int(), C.c_int()
    with _Desc(cluster) as d:
        _check(lib().es_matrix_validate(d.ptr, A.ptr(), C.byref(ok), buf, cap, C.byref(n)))
    v = [MatrixViolation("EmptyColumn" if buf[4 * i] else "EntryNotInMenu", buf[4 * i + 1],
                         buf[4 * i + 2], buf[4 * i + 3]) for i in range(n.value)]
    return MatrixValidation(bool(ok.value), v)


def num_segments(nb: int, segment_size: int) -> int:
    """types.cpp:129-134."""
    out = C.c_size_t()
    _check(lib().es_num_segments(nb, segment_size, C.byref(out)))
    return out.value


def segment_bounds(segment_id: int, segment_size: int, nb: int) -> tuple:
    """types.cpp:136-149 -> (start, end)."""
    s, e = C.c_size_t(), C.c_size_t()
    _check(lib().es_segment_bounds(segment_id, segment_size, nb, C.byref(s), C.byref(e)))
    return s.value, e.value


def batch_rows(nb: int, segment_size: int, batch: int, seg_begin: int = 0,
               seg_end: int = None) -> list:
    """[(first_row, rows)] of the member kernels' tiles over segments
    [seg_begin, seg_end): the reference batcher (pipeline.cpp:143-166)."""
    if seg_end is None:
        seg_end = num_segments(nb, segment_size)
    n = C.c_int()
    _check(lib().es_batch_rows(nb, segment_size, seg_begin, seg_end, batch, None, None, 0,
                               C.byref(n)))
    r0 = (C.c_longlong * max(n.value, 1))()
    rows = (C.c_int * max(n.value, 1))()
    _check(lib().es_batch_rows(nb, segment_size, seg_begin, seg_end, batch, r0, rows, n.value,
                               C.byref(n)))
    return [(r0[i], rows[i]) for i in range(n.value)]


def segment_shares(A: AllocationMatrix, nb: int, segment_size: int, weights=None) -> list:
    """[(device, model, first_segment, end_segment)] per worker, row-major;
    with `weights` (one per worker) a model's runs are proportional to them."""
    cap = max(A.worker_count(), 1)
    out = (C.c_longlong * (4 * cap))()
    n = C.c_int()
    if weights is None:
        _check(lib().es_segment_shares(A.ptr(), A.device_count(), A.model_count(), nb,
                                       segment_size, out, cap, C.byref(n)))
    else:
        w = (C.c_double * cap)(*[float(x) for x in weights])
        _check(lib().es_segment_shares_weighted(A.ptr(), A.device_count(), A.model_count(), nb,
                                                segment_size, w, out, cap, C.byref(n)))
    return [tuple(out[4 * i: 4 * i + 4]) for i in range(n.value)]


@dataclass
class MemoryReport:
    used_mib: list
    fits: bool


def fit_mem(A: AllocationMatrix, cluster: ClusterSpec) -> MemoryReport:
    """memory_model.cpp:22-32."""
    used = (C.c_double * max(cluster.device_count(), 1))()
    fits = C.c_int()
    with _Desc(cluster) as d:
        _check(lib().es_fit_mem(d.ptr, A.ptr(), used, C.byref(fits)))
    return MemoryReport(list(used)[: cluster.device_count()], bool(fits.value))


def more_remaining_memory(A: AllocationMatrix, kind: str, cluster: ClusterSpec) -> Optional[int]:
    """memory_model.cpp:34-50."""
    dev = C.c_int()
    with _Desc(cluster) as d:
        _check(lib().es_more_remaining_memory(d.ptr, A.ptr(), 0 if kind == CPU else 1, C.byref(dev)))
    return None if dev.value < 0 else dev.value


def predict_ensemble_throughput(A: AllocationMatrix, cluster: ClusterSpec) -> float:
    """cost_model.cpp:29-46."""
    out = C.c_double()
    with _Desc(cluster) as d:
        _check(lib().es_predict_ensemble_throughput(d.ptr, A.ptr(), C.byref(out)))
    return out.value


def worst_fit_decreasing(cluster: ClusterSpec, default_batch: int) -> AllocationMatrix:
    """optimizer.cpp:37-64."""
    A = AllocationMatrix(cluster.device_count(), cluster.model_count())
    with _Desc(cluster) as d:
        _check(lib().es_worst_fit_decreasing(d.ptr, default_batch, A.ptr()))
    return A


def neighborhood(A: AllocationMatrix, cluster: ClusterSpec) -> list:
    """optimizer.cpp:66-84."""
    D, M = A.device_count(), A.model_count()
    cap = (len(cluster.batch_menu) + 1) * D * M + 1
    out = np.zeros((cap, D, M), dtype=np.int32)
    n = C.c_int()
    with _Desc(cluster) as d:
        _check(lib().es_neighborhood(d.ptr, A.ptr(), out.ctypes.data_as(_abi.c_int_p), cap,
                                     C.byref(n)))
    return [AllocationMatrix.from_array(out[i]) for i in range(n.value)]


def enumerated_neighborhood_stats(A: AllocationMatrix, cluster: ClusterSpec) -> tuple:
    """optimizer.cpp:86-103 -> (size, forbidden)."""
    s, f = C.c_size_t(), C.c_size_t()
    with _Desc(cluster) as d:
        _check(lib().es_neighborhood_stats(d.ptr, A.ptr(), C.byref(s), C.byref(f)))
    return s.value, f.value


def count_total_matrices(menu_size: int, devices: int, models: int) -> int:
    """optimizer.cpp:105-111 (exact)."""
    buf = C.create_string_buffer(4096)
    _check(lib().es_count_total_matrices(menu_size, devices, models, buf, len(buf)))
    return int(buf.value.decode())


def count_total_neighs(menu_size: int, devices: int, models: int, forbidden: int) -> int:
    """optimizer.cpp:113-118."""
    out = C.c_longlong()
    _check(lib().es_count_total_neighs(menu_size, devices, models, forbidden, C.byref(out)))
    return out.value


def effective_max_iter(devices: int, models: int, max_iter: int) -> int:
    """optimizer.cpp:173-176."""
    out = C.c_int()
    _check(lib().es_effective_max_iter(devices, models, max_iter, C.byref(out)))
    return out.value


def enumerate_all_matrices(cluster: ClusterSpec, cap: int) -> list:
    """optimizer.cpp:165-171."""
    D, M = cluster.device_count(), cluster.model_count()
    count = C.c_size_t()
    with _Desc(cluster) as d:
        _check(lib().es_enumerate_matrices(d.ptr, str(int(cap)).encode(), None, 0, C.byref(count)))
        out = np.zeros((max(count.value, 1), D, M), dtype=np.int32)
        _check(lib().es_enumerate_matrices(d.ptr, str(int(cap)).encode(),
                                           out.ctypes.data_as(_abi.c_int_p), count.value,
                                           C.byref(count)))
    return [AllocationMatrix.from_array(out[i]) for i in range(count.value)]


def sample_indices(seed: int, n: int, k: int) -> list:
    """rng.hpp:26-38 on a fresh mt19937_64(seed)."""
    out = (C.c_size_t * max(min(n, k), 1))()
    _check(lib().es_sample_indices(seed, n, k, out))
    return list(out)[: min(n, k)]


# ------------------------------------------------------------------ optimizer
@dataclass
class GreedyConfig:
    """optimizer.hpp:23-27."""
    max_iter: int = 10
    max_neighs: int = 100
    rng_seed: int = 0


@dataclass
class GreedyIteration:
    index: int
    neighbors_evaluated: int
    best_score: float
    accepted: bool


@dataclass
class OptimizationTrace:
    """optimizer.hpp:40-47."""
    iterations: list
    start_score: float
    final_score: float
    stop_reason: str
    calls: int

    def bench_calls(self) -> int:
        return 1 + sum(it.neighbors_evaluated for it in self.iterations)


@dataclass
class GreedyResult:
    matrix: AllocationMatrix
    trace: OptimizationTrace


class DeviceBench:
    """bench(A, calib) on the GPUs as the greedy's ScoreFn (commands.cpp:132-150)."""

    def __init__(self, calib: "SampleStore", repeats: int = 1, **pool):
        self.calib, self.repeats, self.pool = calib, repeats, pool


class CalibratedBench:
    """calibrated_throughput as a ScoreFn: the per-member B200 fit
    (ModelSpec.b200_cost_s / b200_overhead_s); device_map groups rows that
    share a GPU."""

    def __init__(self, device_map=None):
        self.device_map = list(device_map) if device_map else None


def _bench_cfg(bench, keep: list):
    cfg = _abi.BenchCfg()
    if bench is None or bench == "analytic":
        cfg.mode = 0
    elif isinstance(bench, CalibratedBench):
        cfg.mode = 3
        opts = _pool_opts(keep, device_map=bench.device_map)
        cfg.opts = C.pointer(opts)
    elif isinstance(bench, DeviceBench):
        cfg.mode = 1
        cfg.calib = bench.calib._h
        cfg.repeats = bench.repeats
        opts = _pool_opts(keep, **bench.pool)
        cfg.opts = C.pointer(opts)
    elif callable(bench):
        def trampoline(a_ptr, D, M, _user):
            arr = np.ctypeslib.as_array(a_ptr, shape=(D * M,)).reshape(D, M).copy()
            return float(bench(AllocationMatrix.from_array(arr)))
        cb = _abi.SCORE_FN(trampoline)
        keep.append(cb)
        cfg.mode = 2
        cfg.fn = cb
    else:
        raise TypeError("bench must be None/'analytic', a DeviceBench or a callable")
    keep.append(cfg)
    return cfg


def bounded_greedy(A0: AllocationMatrix, cluster: ClusterSpec, bench=None,
                   config: GreedyConfig = GreedyConfig()) -> GreedyResult:
    """optimizer.cpp:178-227; bench = 'analytic' | DeviceBench | callable(A) -> score."""
    keep: list = []
    cfg = _bench_cfg(bench, keep)
    out = AllocationMatrix(A0.device_count(), A0.model_count())
    cap = effective_max_iter(cluster.device_count(), cluster.model_count(), config.max_iter) + 1
    nbr = (C.c_int * cap)()
    best = (C.c_double * cap)()
    acc = (C.c_int * cap)()
    tr = _abi.GreedyTrace(0, 0, 0, 0, 0, cap, nbr, best, acc)
    with _Desc(cluster) as d:
        _check(lib().es_bounded_greedy(d.ptr, A0.ptr(), config.max_iter, config.max_neighs,
                                       config.rng_seed, C.byref(cfg), out.ptr(), C.byref(tr)))
    its = [GreedyIteration(i, nbr[i], best[i], bool(acc[i])) for i in range(tr.n_iters)]
    trace = OptimizationTrace(its, tr.start_score, tr.final_score,
                              "local_optimum" if tr.stop_reason == 0 else "iter_cap", tr.bench_calls)
    return GreedyResult(out, trace)


def screened_greedy(A0: AllocationMatrix, cluster: ClusterSpec, bench, screen,
                    config: GreedyConfig = GreedyConfig(), top_k: int = 4) -> GreedyResult:
    """bounded_greedy whose iterations bench only the `top_k` sampled
    neighbours `screen` ranks best (search.hpp screened_greedy)."""
    keep: list = []
    cfg = _bench_cfg(bench, keep)
    scfg = _bench_cfg(screen, keep)
    out = AllocationMatrix(A0.device_count(), A0.model_count())
    cap = effective_max_iter(cluster.device_count(), cluster.model_count(), config.max_iter) + 1
    nbr = (C.c_int * cap)()
    best = (C.c_double * cap)()
    acc = (C.c_int * cap)()
    tr = _abi.GreedyTrace(0, 0, 0, 0, 0, cap, nbr, best, acc)
    with _Desc(cluster) as d:
        _check(lib().es_screened_greedy(d.ptr, A0.ptr(), config.max_iter, config.max_neighs,
                                        config.rng_seed, int(top_k), C.byref(cfg), C.byref(scfg),
                                        out.ptr(), C.byref(tr)))
    its = [GreedyIteration(i, nbr[i], best[i], bool(acc[i])) for i in range(tr.n_iters)]
    trace = OptimizationTrace(its, tr.start_score, tr.final_score,
                              "local_optimum" if tr.stop_reason == 0 else "iter_cap", tr.bench_calls)
    return GreedyResult(out, trace)


def calibrated_throughput(A: AllocationMatrix, cluster: ClusterSpec, row_gpu=None) -> float:
    """calibrate.hpp calibrated_throughput (per-member B200 fit)."""
    out = C.c_double()
    rg = (C.c_int * len(row_gpu))(*row_gpu) if row_gpu else None
    with _Desc(cluster) as d:
        _check(lib().es_calibrated_throughput(d.ptr, A.ptr(), rg, C.byref(out)))
    return out.value


@dataclass
class BaselineResult:
    matrix: AllocationMatrix
    bench_calls: int
    chosen_batches: list


def bbs_baseline(cluster: ClusterSpec, bench=None) -> BaselineResult:
    """optimizer.cpp:229-269."""
    keep: list = []
    cfg = _bench_cfg(bench, keep)
    out = AllocationMatrix(cluster.device_count(), cluster.model_count())
    chosen = (C.c_int * max(cluster.model_count(), 1))()
    calls = C.c_int()
    with _Desc(cluster) as d:
        _check(lib().es_bbs_baseline(d.ptr, C.byref(cfg), out.ptr(), chosen, C.byref(calls)))
    return BaselineResult(out, calls.value, list(chosen)[: cluster.model_count()])


# ------------------------------------------------------------------ runtime
@dataclass
class CombinationRule:
    """combine.hpp:14-27 (+ member_softmax)."""
    kind: str = "avg"  # avg | vote | wavg
    weights: tuple = ()
    member_softmax: bool = False

    @staticmethod
    def averaging(softmax: bool = False) -> "CombinationRule":
        return CombinationRule("avg", (), softmax)

    @staticmethod
    def majority_vote(softmax: bool = False) -> "CombinationRule":
        return CombinationRule("vote", (), softmax)

    @staticmethod
    def weighted(weights, softmax: bool = False) -> "CombinationRule":
        w = [float(x) for x in weights]
        if any(x < 0 for x in w):
            raise SpecError("combination weights must be nonnegative")
        if abs(sum(w) - 1.0) > 1e-9:
            raise SpecError(f"combination weights must sum to 1, got {sum(w)}")
        return CombinationRule("wavg", tuple(w), softmax)

    def _desc(self, keep: list):
        kind = {"avg": 0, "vote": 1, "wavg": 2}[self.kind]
        w = (C.c_double * max(len(self.weights), 1))(*self.weights)
        keep.append(w)
        d = _abi.RuleDesc(kind, int(self.member_softmax), C.cast(w, _abi.c_double_p))
        keep.append(d)
        return d


def _pool_opts(keep: list, device_map=None, copy_outputs=True, warmup=True,
               sms_per_worker=0, overlap_colocated=False, e2e_chunk_rows=0,
               e2e_host_convert=True, e2e_convert_eighths=0,
               dp_equal_split=False, row_partials=False, peer_stores=True,
               row_nodes=False, dp_claim="auto", claim_chunk=0,
               pack_batches=False, fp32=False) -> _abi.PoolOpts:
    """PoolOptions (runtime.hpp)."""
    dm = None
    n = 0
    if device_map:
        dm = (C.c_int * len(device_map))(*device_map)
        keep.append(dm)
        n = len(device_map)
    o = _abi.PoolOpts(C.cast(dm, _abi.c_int_p) if dm is not None else None, n, int(copy_outputs),
                      int(warmup), int(sms_per_worker), int(overlap_colocated),
                      int(e2e_chunk_rows), int(e2e_host_convert), int(e2e_convert_eighths),
                      int(dp_equal_split), int(row_partials), int(not peer_stores),
                      int(row_nodes), {"auto": 0, True: 1, False: -1}[dp_claim],
                      int(claim_chunk), int(pack_batches), int(fp32))
    keep.append(o)
    return o


def host_convert_bf16(x: np.ndarray) -> np.ndarray:
    """The e2e host converter: bf16 bits (uint16) of x, round-to-nearest-even."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty(x.shape, dtype=np.uint16)
    _check(lib().es_host_convert_bf16(x.ctypes.data_as(_abi.c_float_p),
                                      y.ctypes.data_as(C.POINTER(C.c_uint16)), x.size))
    return y


def device_count() -> int:
    n = C.c_int()
    _check(lib().es_device_count(C.byref(n)))
    return n.value


class SampleStore:
    """Immutable nb x width fp32 samples (message.hpp:12-34); device replicas
    are created lazily per GPU."""

    def __init__(self, X=None, *, synthetic_seed: Optional[int] = None, nb: int = 0,
                 width: int = 0, device: int = 0):
        h = C.c_void_p()
        if X is not None:
            self._X = np.ascontiguousarray(X, dtype=np.float32)
            if self._X.ndim != 2:
                raise SpecError("sample store needs a 2-D array")
            nb, width = self._X.shape
            _check(lib().es_store_create(self._X.ctypes.data_as(_abi.c_float_p), nb, width, 0,
                                         C.byref(h)))
        else:
            self._X = None
            _check(lib().es_store_synthetic(int(synthetic_seed or 0), nb, width, device, C.byref(h)))
        self._h = h
        self.nb, self.width = nb, width

    def nb_samples(self) -> int:
        return self.nb

    def __del__(self):
        if getattr(self, "_h", None):
            lib().es_store_destroy(self._h)
            self._h = None


@dataclass
class RunStats:
    nb_samples: int
    segments: int
    data_messages: int
    elapsed_s: float


@dataclass
class RunOutput:
    combined: np.ndarray
    winners: np.ndarray
    output_width: int
    stats: RunStats


class InferenceSystem:
    """pipeline.hpp:62-117, GPU-resident."""

    def __init__(self, A: AllocationMatrix, cluster: ClusterSpec, rule: CombinationRule = None,
                 **pool):
        self._keep: list = []
        rule = rule or CombinationRule.averaging()
        self.cluster = cluster
        self.C = cluster.models[0].output_width if cluster.models else 1
        h = C.c_void_p()
        with _Desc(cluster) as d:
            _check(lib().es_system_create(d.ptr, A.ptr(), C.byref(rule._desc(self._keep)),
                                          C.byref(_pool_opts(self._keep, **pool)), C.byref(h)))
        self._h = h
        self._store = None

    def worker_count(self) -> int:
        n = C.c_int()
        _check(lib().es_system_info(self._h, C.byref(n), None, None, None))
        return n.value

    def workers_per_model(self) -> list:
        M = self.cluster.model_count()
        w = (C.c_int * max(M, 1))()
        _check(lib().es_system_info(self._h, None, w, None, None))
        return list(w)[:M]

    def launches_last_run(self) -> int:
        n = C.c_int()
        _check(lib().es_system_info(self._h, None, None, C.byref(n), None))
        return n.value

    def timing(self) -> tuple:
        """(member_ms per worker, combine_ms) of the last run, CUDA events."""
        w = self.worker_count()
        ms = (C.c_double * max(w, 1))()
        cm = C.c_double()
        _check(lib().es_system_timing(self._h, ms, C.byref(cm)))
        return list(ms)[:w], cm.value

    def shares(self) -> tuple:
        """([(begin, end)] segment runs per worker in the last run, [rows/s]
        probed per data-parallel worker; 1.0 for single workers)."""
        w = self.worker_count()
        sh = (C.c_int64 * max(2 * w, 1))()
        r = (C.c_double * max(w, 1))()
        _check(lib().es_system_shares(self._h, sh, r))
        return [(sh[2 * i], sh[2 * i + 1]) for i in range(w)], list(r)[:w]

    def last_transfer(self) -> tuple:
        """(h2d_bytes, d2h_bytes) moved by the last run_host."""
        h, d = C.c_size_t(), C.c_size_t()
        _check(lib().es_system_last_transfer(self._h, C.byref(h), C.byref(d)))
        return h.value, d.value

    def kernel_timing(self, worker: int) -> list:
        """[(kernel name, ms)] of one worker's launches in the last run (CUDA
        events recorded on the worker's stream between launches)."""
        ms = (C.c_double * 16)()
        names = C.create_string_buffer(512)
        n = C.c_int()
        _check(lib().es_system_kernel_timing(self._h, worker, ms, names, 512, 16, C.byref(n)))
        return list(zip(names.value.decode().split(";"), list(ms)[:n.value]))

    def routes(self) -> tuple:
        """([route per worker], [peer CUDA ordinals]): 0 = on the combining
        node, 1 = remote with direct NVLink peer stores, 2 = remote through a
        staging buffer + peer copy."""
        w = self.worker_count()
        r = (C.c_int * max(w, 1))()
        p = (C.c_int * 64)()
        n = C.c_int()
        _check(lib().es_system_routes(self._h, r, p, 64, C.byref(n)))
        return list(r)[:w], list(p)[:n.value]

    def claim_models(self) -> list:
        """Models whose data-parallel workers pop a device queue."""
        out = (C.c_int * 64)()
        n = C.c_int()
        _check(lib().es_system_claim_models(self._h, out, 64, C.byref(n)))
        return list(out)[:n.value]

    def claims(self, model: int) -> Optional[np.ndarray]:
        """Device FIFO of the last run for `model`: the worker index (row-major
        cells) that claimed each segment, or None if the model has no queue."""
        n = C.c_size_t()
        _check(lib().es_system_claims(self._h, int(model), None, 0, C.byref(n)))
        if n.value == 0:
            return None
        out = np.zeros(n.value, dtype=np.int32)
        _check(lib().es_system_claims(self._h, int(model), out.ctypes.data_as(_abi.c_int_p),
                                      n.value, C.byref(n)))
        return out

    def set_gather(self, comm: "Comm" = None, root: int = 0, first_rows=None, rows=None) -> None:
        """One process per GPU: after every run this rank's probabilities +
        argmax go to `root` over NCCL (inside the timed window), landing at
        row first_rows[rank] of a sum(rows)-row result that the root's run()
        returns.  comm=None detaches."""
        if comm is None:
            _check(lib().es_system_set_gather(self._h, None, 0, None, None, 0))
            self._gather = None
            return
        n = comm.size
        f = (C.c_int64 * n)(*[int(v) for v in first_rows])
        k = (C.c_int64 * n)(*[int(v) for v in rows])
        _check(lib().es_system_set_gather(self._h, comm._h, int(root), f, k, n))
        self._gather = (comm, int(root), [int(v) for v in rows])

    def begin_run(self, X: SampleStore, rule: CombinationRule = None) -> None:
        keep: list = []
        self._store = X
        self._pending = X.nb
        g = getattr(self, "_gather", None)
        if g is not None and g[0].rank == g[1]:
            self._pending = sum(g[2])  # the root receives every rank's rows
        _check(lib().es_system_begin_run(self._h, X._h,
                                         C.byref(rule._desc(keep)) if rule else None))

    def broadcast(self) -> int:
        n = C.c_size_t()
        _check(lib().es_system_broadcast(self._h, C.byref(n)))
        return n.value

    def await_run(self, copy: bool = True) -> RunOutput:
        nb = self._pending
        Y = np.zeros((nb, self.C), dtype=np.float32) if copy else None
        W = np.zeros(nb, dtype=np.int32) if copy else None
        st = _abi.RunStats()
        _check(lib().es_system_await_run(
            self._h, Y.ctypes.data_as(_abi.c_float_p) if copy else None,
            W.ctypes.data_as(_abi.c_int32_p) if copy else None, C.byref(st)))
        return RunOutput(Y, W, self.C, RunStats(st.nb_samples, st.segments, st.data_messages,
                                               st.elapsed_s))

    def run(self, X: SampleStore, rule: CombinationRule = None, copy: bool = True) -> RunOutput:
        self.begin_run(X, rule)
        self.broadcast()
        return self.await_run(copy)

    def run_host(self, X: np.ndarray, Y: np.ndarray = None, labels: np.ndarray = None) -> float:
        """End-to-end from host memory: X (nb, width) fp32 in, the combined
        output into Y (nb, C) float32 and the argmax into labels (nb,) int32
        (each optional, C-contiguous, written in place).  Returns the host
        wall-clock seconds of the whole pipelined call (host conversion,
        copies and kernels)."""
        X = np.ascontiguousarray(X, dtype=np.float32)
        if X.ndim != 2:
            raise InvalidArgument(f"run_host: X must be 2-D (nb, width), got shape {X.shape}")
        nb, width = X.shape
        _require_out(Y, np.float32, (nb, self.C), "Y")
        _require_out(labels, np.int32, (nb,), "labels")
        el = C.c_double()
        _check(lib().es_system_run_host(
            self._h, X.ctypes.data_as(_abi.c_float_p), nb, width,
            Y.ctypes.data_as(_abi.c_float_p) if Y is not None else None,
            labels.ctypes.data_as(_abi.c_int32_p) if labels is not None else None, C.byref(el)))
        return el.value

    def shutdown(self) -> None:
        if self._h:
            _check(lib().es_system_shutdown(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().es_system_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes) for Comm on every rank."""
    buf = (C.c_uint8 * 128)()
    _check(lib().es_comm_unique_id(buf, 128))
    return bytes(buf)


def nccl_version() -> int:
    v = C.c_int()
    _check(lib().es_nccl_version(C.byref(v)))
    return v.value


class Comm:
    """NCCL communicator of one process per GPU (ncclCommInitRank; every
    rank constructs it collectively with rank 0's nccl_unique_id())."""

    def __init__(self, unique_id: bytes, size: int, rank: int, device: int):
        if len(unique_id) != 128:
            raise InvalidArgument("NCCL unique id must be 128 bytes")
        buf = (C.c_uint8 * 128)(*unique_id)
        h = C.c_void_p()
        _check(lib().es_comm_create(buf, 128, int(size), int(rank), int(device), C.byref(h)))
        self._h = h
        self.size, self.rank, self.device = int(size), int(rank), int(device)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().es_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def run_inference(X: SampleStore, A: AllocationMatrix, cluster: ClusterSpec,
                  rule: CombinationRule = None, **pool) -> RunOutput:
    """pipeline.cpp:418-444, Deploy mode."""
    keep: list = []
    rule = rule or CombinationRule.averaging()
    Cw = cluster.models[0].output_width
    Y = np.zeros((X.nb, Cw), dtype=np.float32)
    W = np.zeros(X.nb, dtype=np.int32)
    st = _abi.RunStats()
    with _Desc(cluster) as d:
        _check(lib().es_run_inference(d.ptr, A.ptr(), C.byref(rule._desc(keep)), X._h,
                                      C.byref(_pool_opts(keep, **pool)),
                                      Y.ctypes.data_as(_abi.c_float_p),
                                      W.ctypes.data_as(_abi.c_int32_p), C.byref(st)))
    return RunOutput(Y, W, Cw, RunStats(st.nb_samples, st.segments, st.data_messages, st.elapsed_s))


@dataclass
class BenchResult:
    """pipeline.hpp:35-41."""
    throughput: float
    elapsed_s: float
    nb_samples: int
    runs: list
    rsd: float


def bench(A: AllocationMatrix, calib: SampleStore, cluster: ClusterSpec, repeats: int,
          **pool) -> BenchResult:
    """pipeline.cpp:465-501 on the GPUs (CUDA-event timed)."""
    keep: list = []
    r = _abi.BenchResultC()
    with _Desc(cluster) as d:
        _check(lib().es_bench(d.ptr, A.ptr(), calib._h if calib is not None else None, repeats,
                              C.byref(_pool_opts(keep, **pool)), C.byref(r)))
    return BenchResult(r.throughput, r.elapsed_s, r.nb_samples, list(r.runs)[: r.n_runs], r.rsd)



@dataclass
class ServiceStats:
    """GET /v1/stats (server.cpp:88-107)."""
    ready: bool
    requests_served: int
    samples_served: int
    flushes: int
    last_flush_throughput: float
    pending_requests: int
    pending_samples: int
    uptime_s: float
    matrix: list = None  # the allocation matrix being served (server.cpp:88-107 "matrix")


class PendingPrediction:
    """One POST /v1/predict in flight; result() blocks until its flush ran."""

    def __init__(self, handle, rows: int, width: int):
        self._h = handle
        self.rows = rows
        self._C = width
        self._out = None

    def result(self) -> tuple:
        """(combined [rows, C] fp32, winners [rows] int32); raises the flush's error."""
        if self._out is None:
            Y = np.zeros((self.rows, self._C), dtype=np.float32)
            W = np.zeros(self.rows, dtype=np.int32)
            try:
                _check(lib().es_request_wait(self._h, Y.ctypes.data_as(_abi.c_float_p),
                                             W.ctypes.data_as(_abi.c_int32_p)))
            finally:
                lib().es_request_destroy(self._h)
                self._h = None
            self._out = (Y, W)
        return self._out

    def __del__(self):
        if getattr(self, "_h", None):
            lib().es_request_destroy(self._h)
            self._h = None


class PredictionService:
    """Deploy-mode serving core of PredictionServer (server.hpp:28-60,
    server.cpp:65-288) without the HTTP listener.

    Requests are buffered and flushed into one device run when a full segment is
    waiting or the oldest request has waited `flush_timeout_ms`; each request
    receives its own rows of the combined output."""

    def __init__(self, cluster: ClusterSpec, A: AllocationMatrix,
                 rule: CombinationRule = None, flush_timeout_ms: int = 50,
                 input_width: int = None, arena_rows: int = -1, **pool):
        keep: list = []
        rule = rule or CombinationRule.averaging()
        if input_width is None:  # real members define it; synthetic ones need it given
            arch = cluster.models[0].arch
            if arch is None or arch.kind == "synthetic":
                raise InvalidArgument("input_width is required for synthetic members")
            input_width = arch.input_width()
        self.input_width = int(input_width)
        self.C = cluster.models[0].output_width
        self.matrix = A.cells.tolist()
        h = C.c_void_p()
        with _Desc(cluster) as d:
            _check(lib().es_service_create(d.ptr, A.ptr(), C.byref(rule._desc(keep)),
                                           C.byref(_pool_opts(keep, **pool)),
                                           int(flush_timeout_ms), self.input_width,
                                           int(arena_rows), C.byref(h)))
        self._h = h

    def wait_ready(self, timeout_s: float = 60.0) -> bool:
        ready = C.c_int()
        err = C.create_string_buffer(512)
        _check(lib().es_service_wait_ready(self._h, int(timeout_s * 1000), C.byref(ready), err,
                                           len(err)))
        self.startup_error = err.value.decode() or None
        return bool(ready.value)

    def submit(self, samples: np.ndarray) -> PendingPrediction:
        x = np.ascontiguousarray(samples, dtype=np.float32)
        if x.size == 0:
            x = x.reshape(0, self.input_width)
        if x.ndim != 2 or x.shape[1] != self.input_width:  # server.cpp:118-135 -> 400
            raise InvalidArgument(f"expected rows of {self.input_width} features, got shape "
                                  f"{x.shape}")
        r = C.c_void_p()
        _check(lib().es_service_submit(self._h, x.ctypes.data_as(_abi.c_float_p), x.shape[0],
                                       C.byref(r)))
        return PendingPrediction(r, x.shape[0], self.C)

    def predict(self, samples: np.ndarray) -> tuple:
        """Blocking POST /v1/predict."""
        return self.submit(samples).result()

    def stats(self) -> ServiceStats:
        st = _abi.ServiceStatsC()
        _check(lib().es_service_stats(self._h, C.byref(st)))
        return ServiceStats(bool(st.ready), st.requests_served, st.samples_served, st.flushes,
                            st.last_flush_throughput, st.pending_requests, st.pending_samples,
                            st.uptime_s, self.matrix)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().es_service_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def __del__(self):
        self.close()


class Member:
    """Predictor seam (backend.hpp:25-34): es_member_create = make + load."""

    def __init__(self, model: ModelSpec, batch: int, device: int = 0,
                 device_load_mib: float = 0.0, capacity_mib: float = float("inf")):
        keep: list = []
        c = ClusterSpec(models=[model])
        d = _Desc(c)
        keep.append(d)
        h = C.c_void_p()
        _check(lib().es_member_create(device, C.byref(d.models[0]), model.id, batch,
                                      device_load_mib, capacity_mib, C.byref(h)))
        self._h = h
        self.C = model.output_width

    def predict(self, features: np.ndarray, first_index: int = 0) -> np.ndarray:
        f = np.ascontiguousarray(features, dtype=np.float32)
        if f.ndim != 2:
            raise InvalidArgument(f"predict: features must be 2-D (rows, width), got shape {f.shape}")
        out = np.zeros((f.shape[0], self.C), dtype=np.float32)
        _check(lib().es_member_predict(self._h, f.ctypes.data_as(_abi.c_float_p), first_index,
                                       f.shape[0], f.shape[1], out.ctypes.data_as(_abi.c_float_p)))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            lib().es_member_destroy(self._h)
            self._h = None


def combine(rule: CombinationRule, blocks: Sequence[np.ndarray]) -> tuple:
    """Device fold of per-model blocks (combine.cpp:93-136) -> (Y, winners)."""
    keep: list = []
    arrs = [np.ascontiguousarray(b, dtype=np.float32) for b in blocks]
    if not arrs:
        raise InvalidArgument("combine: no member blocks")
    if len(arrs) > MAX_MEMBERS:
        raise InvalidArgument(f"combine: at most {MAX_MEMBERS} member blocks, got {len(arrs)}")
    # PredictionAccumulator::add rejects a block of the wrong shape
    # (combine.cpp:63-77): every block must be rows x C like the first.
    if arrs[0].ndim != 2:
        raise ProtocolError(f"combine: block 0 must be 2-D (rows, C), got shape {arrs[0].shape}")
    rows, Cw = arrs[0].shape
    if Cw > MAX_CLASSES:
        raise InvalidArgument(f"combine: at most {MAX_CLASSES} classes, got {Cw}")
    for m, a in enumerate(arrs):
        if a.shape != (rows, Cw):
            raise ProtocolError(f"combine: block {m} has shape {a.shape}, expected {(rows, Cw)}")
    ptrs = (_abi.c_float_p * len(arrs))(*[a.ctypes.data_as(_abi.c_float_p) for a in arrs])
    Y = np.zeros((rows, Cw), dtype=np.float32)
    W = np.zeros(rows, dtype=np.int32)
    _check(lib().es_combine(C.byref(rule._desc(keep)), len(arrs), Cw, rows, ptrs,
                            Y.ctypes.data_as(_abi.c_float_p), W.ctypes.data_as(_abi.c_int32_p)))
    return Y, W


# ------------------------------------------------------------------ documents
def _text(call) -> str:
    """Two-pass text result: ask for the size, then fill."""
    need = C.c_size_t()
    _check(call(None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _check(call(buf, need.value, C.byref(need)))
    return buf.value.decode()


def _cluster_from_desc(d: "_abi.ClusterDesc") -> ClusterSpec:
    devs = [DeviceSpec(i, CPU if d.devices[i].kind == 0 else GPU, d.devices[i].memory_mib,
                       d.devices[i].compute_rate, d.devices[i].batch_overhead_s)
            for i in range(d.n_devices)]
    models = []
    for i in range(d.n_models):
        m = d.models[i]
        kind = {1: "mlp", 2: "cnn"}.get(m.arch, "synthetic")
        arch = MemberArch(kind, tuple(m.widths[j] for j in range(m.n_widths)), int(m.weight_seed))
        models.append(ModelSpec(i, m.name.decode(), m.weight_mib, m.act_mib_per_sample,
                                m.cost_per_sample, m.output_width, arch, m.b200_cost_s,
                                m.b200_overhead_s))
    return ClusterSpec(devs, models, [d.batch_menu[i] for i in range(d.menu_size)], d.segment_size)


def _spec_handle_to_cluster(h: C.c_void_p) -> ClusterSpec:
    try:
        d = _abi.ClusterDesc()
        _check(lib().es_spec_describe(h, C.byref(d)))
        return _cluster_from_desc(d)
    finally:
        lib().es_spec_destroy(h)


def cluster_to_json(cluster: ClusterSpec, indent: int = -1, with_arch: bool = False) -> str:
    """spec_io.cpp:7-28, dumped like nlohmann's dump(indent)."""
    with _Desc(cluster) as d:
        return _text(lambda b, n, need: lib().es_cluster_to_json(d.ptr, indent, int(with_arch),
                                                                 b, n, need))


def cluster_from_json(text: str, overlay: Optional[str] = None) -> ClusterSpec:
    """cluster_from_documents + cluster_from_json (spec_io.cpp:47-89)."""
    h = C.c_void_p()
    _check(lib().es_spec_from_json(text.encode(), overlay.encode() if overlay else None,
                                   C.byref(h)))
    return _spec_handle_to_cluster(h)


def load_spec(path: str, overlay_path: Optional[str] = None) -> ClusterSpec:
    """A --cluster file merged with an optional --ensemble file."""
    h = C.c_void_p()
    _check(lib().es_spec_load(str(path).encode(),
                              str(overlay_path).encode() if overlay_path else None, C.byref(h)))
    return _spec_handle_to_cluster(h)


def save_json_file(path: str, text: str) -> None:
    """spec_io.cpp:145-149 (indent 2 + newline)."""
    _check(lib().es_save_json_file(str(path).encode(), text.encode()))


def matrix_to_json(A: AllocationMatrix, cluster: ClusterSpec, indent: int = -1) -> str:
    with _Desc(cluster) as d:
        return _text(lambda b, n, need: lib().es_matrix_to_json(d.ptr, A.ptr(), indent, b, n, need))


def matrix_from_json(text: str, cluster: ClusterSpec) -> AllocationMatrix:
    A = AllocationMatrix(cluster.device_count(), cluster.model_count())
    with _Desc(cluster) as d:
        _check(lib().es_matrix_from_json(d.ptr, text.encode(), A.ptr()))
    return A


def digest_hex(text: str) -> str:
    out = C.create_string_buffer(17)
    _check(lib().es_digest_hex(text.encode(), out))
    return out.value.decode()


@dataclass
class OptimizerKey:
    """cache.hpp OptimizerKey: settings that change the optimized matrix."""
    greedy: GreedyConfig = field(default_factory=GreedyConfig)
    default_batch: int = 0
    bench_mode: str = "measured"
    calib_samples: int = 0
    repeats: int = 1
    # opt-in hardware identity (device_identity()); "" = the reference's key
    device: str = ""


def device_identity() -> str:
    """'<name>/sm_<cc>/<SMs> SMs/<GiB> GiB x<count>' of the visible GPUs."""
    out = C.create_string_buffer(256)
    _check(lib().es_device_identity(out, 256))
    return out.value.decode()


def cache_key(cluster: ClusterSpec, key: OptimizerKey) -> str:
    """cache.cpp:22-33 (plus the opt-in device identity when key.device is set)."""
    out = C.create_string_buffer(17)
    with _Desc(cluster) as d:
        _check(lib().es_cache_key_device(d.ptr, key.greedy.max_iter, key.greedy.max_neighs,
                                         key.greedy.rng_seed, key.default_batch,
                                         key.bench_mode.encode(), key.calib_samples, key.repeats,
                                         key.device.encode(), out))
    return out.value.decode()


@dataclass
class MatrixCacheEntry:
    key: str
    matrix: AllocationMatrix
    score: float = 0.0
    created_at: int = 0


class MatrixCache:
    """One JSON document per key under a directory (cache.cpp:35-88)."""

    def __init__(self, directory: str):
        self.directory = str(directory)

    def lookup(self, key: str, cluster: ClusterSpec) -> Optional[MatrixCacheEntry]:
        A = AllocationMatrix(cluster.device_count(), cluster.model_count())
        score, created, hit = C.c_double(), C.c_int64(), C.c_int()
        with _Desc(cluster) as d:
            _check(lib().es_cache_lookup(self.directory.encode(), key.encode(), d.ptr, A.ptr(),
                                         C.byref(score), C.byref(created), C.byref(hit)))
        return MatrixCacheEntry(key, A, score.value, created.value) if hit.value else None

    def store(self, entry: MatrixCacheEntry, cluster: ClusterSpec) -> None:
        with _Desc(cluster) as d:
            _check(lib().es_cache_store(self.directory.encode(), entry.key.encode(), d.ptr,
                                        entry.matrix.ptr(), entry.score, entry.created_at))


# ------------------------------------------------------------------ calibrated cost model (§8-F F4)
@dataclass
class CostFit:
    """Fitted inputs of the analytic cost model (compute_rate = 1)."""
    cost_per_sample: list
    batch_overhead_s: float
    rms_rel_error: float
    measured: Optional[list] = None  # [(model, batch, samples/s)] when benched here
    # per-member form 1/throughput = member_cost_s[m] + member_overhead_s[m] / b
    member_cost_s: Optional[list] = None
    member_overhead_s: Optional[list] = None
    member_rms_rel_error: float = 0.0


def fit_cost_model(samples: Sequence[tuple], n_models: int) -> CostFit:
    """samples: (model, batch, throughput) triples -> least-squares fit of
    1/throughput = c_m + o/b (calibrate.hpp)."""
    n = len(samples)
    mi = (C.c_int * max(n, 1))(*[int(s[0]) for s in samples])
    bi = (C.c_int * max(n, 1))(*[int(s[1]) for s in samples])
    th = (C.c_double * max(n, 1))(*[float(s[2]) for s in samples])
    cost = (C.c_double * n_models)()
    mc, mo = (C.c_double * n_models)(), (C.c_double * n_models)()
    o, rms, mrms = C.c_double(), C.c_double(), C.c_double()
    _check(lib().es_fit_cost_model(mi, bi, th, n, n_models, cost, C.byref(o), C.byref(rms),
                                   mc, mo, C.byref(mrms)))
    return CostFit(list(cost), o.value, rms.value, None, list(mc), list(mo), mrms.value)


def calibrate_cost_model(cluster: ClusterSpec, device: int = 0, calib_nb: int = 65536,
                         repeats: int = 3) -> CostFit:
    """Bench every member alone on `device` at every menu batch, then fit."""
    M, B = cluster.model_count(), len(cluster.batch_menu)
    cost = (C.c_double * M)()
    meas = (C.c_double * (M * B))()
    mc, mo = (C.c_double * M)(), (C.c_double * M)()
    o, rms, mrms = C.c_double(), C.c_double(), C.c_double()
    with _Desc(cluster) as d:
        _check(lib().es_calibrate_cost_model(d.ptr, device, calib_nb, repeats, cost, C.byref(o),
                                             C.byref(rms), meas, mc, mo, C.byref(mrms)))
    samples = [(m, cluster.batch_menu[j], meas[m * B + j]) for m in range(M) for j in range(B)]
    return CostFit(list(cost), o.value, rms.value, samples, list(mc), list(mo), mrms.value)


def apply_cost_fit(cluster: ClusterSpec, fit: CostFit) -> ClusterSpec:
    """GPU rows: compute_rate 1, the fitted overhead; models: fitted costs."""
    import copy
    out = copy.deepcopy(cluster)
    for d in out.devices:
        if d.kind == GPU:
            d.compute_rate, d.batch_overhead_s = 1.0, fit.batch_overhead_s
    for i, (m, c) in enumerate(zip(out.models, fit.cost_per_sample)):
        m.cost_per_sample = c
        if fit.member_cost_s:
            m.b200_cost_s, m.b200_overhead_s = fit.member_cost_s[i], fit.member_overhead_s[i]
    return out
