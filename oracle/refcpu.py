"""ORACLE — test infrastructure only (see oracle/__init__.py).

ctypes access to
  * liboracle.so            — cpu_member.c: CPU MLP member, softmax, fold;
  * _ref/libenserve_ref.so  — the reference library itself (compiled from
                              /root/reference/proj/src by oracle/Makefile) plus
                              ref_capi.cpp.
Cluster arguments are duck-typed (attributes devices/models/batch_menu/
segment_size, devices with kind/memory_mib/compute_rate/batch_overhead_s,
models with name/weight_mib/act_mib_per_sample/cost_per_sample/output_width and
optionally arch.widths / arch.weight_seed), so this module imports nothing from
the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libenserve_ref.so"
REF_SRC = Path("/root/reference/proj")

f32p = C.POINTER(C.c_float)
i32p = C.POINTER(C.c_int)
f64p = C.POINTER(C.c_double)


def build(quiet: bool = True) -> None:
    """Compile liboracle.so always, and _ref/ when the reference sources exist
    (the GPU box only has the prebuilt files)."""
    targets = ["liboracle.so"]
    if REF_SRC.exists():
        targets.append("_ref/libenserve_ref.so")
        if (HERE.parent / "paper_2208_14049_b200" / "libenserve_b200.so").exists():
            targets.append("integration")
        targets.append("spec_golden")  # the reference's spec/cache units (tests/golden/spec_io.json)
    subprocess.run(["make", "-C", str(HERE), *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


# ------------------------------------------------------------------ liboracle
_orc = None


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            build()
        lib = C.CDLL(str(ORACLE_SO))
        lib.orc_mlp_create.restype = C.c_void_p
        lib.orc_mlp_create.argtypes = [C.c_int, i32p, C.c_uint64, C.c_int]
        lib.orc_mlp_destroy.argtypes = [C.c_void_p]
        lib.orc_mlp_forward.argtypes = [C.c_void_p, f32p, C.c_size_t, f32p]
        lib.orc_mlp_layer.argtypes = [C.c_void_p, C.c_int, f32p, f32p]
        lib.orc_cnn_create.restype = C.c_void_p
        lib.orc_cnn_create.argtypes = [C.c_int] * 6 + [C.c_uint64, C.c_int]
        lib.orc_cnn_destroy.argtypes = [C.c_void_p]
        lib.orc_cnn_forward.argtypes = [C.c_void_p, f32p, C.c_size_t, f32p]
        lib.orc_cnn_hidden.argtypes = [C.c_void_p, f32p, C.c_size_t, f32p]
        lib.orc_cnn_layer.argtypes = [C.c_void_p, C.c_int, f32p, f32p]
        lib.orc_softmax_rows.argtypes = [f32p, C.c_size_t, C.c_int, f32p]
        lib.orc_fold.argtypes = [C.c_int, C.c_int, C.c_size_t, C.c_int, C.POINTER(f32p), f64p,
                                 f32p, i32p]
        lib.orc_fill_features.argtypes = [C.c_uint64, C.c_size_t, C.c_size_t, f32p]
        lib.orc_weight.restype = C.c_float
        lib.orc_weight.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_int, C.c_int]
        lib.orc_bias.restype = C.c_float
        lib.orc_bias.argtypes = [C.c_uint64, C.c_int, C.c_uint64]
        lib.orc_round_bf16.restype = C.c_float
        lib.orc_round_bf16.argtypes = [C.c_float]
        _orc = lib
    return _orc


def _fp(a: np.ndarray):
    return a.ctypes.data_as(f32p)


class CpuMlp:
    """Oracle CPU member: bf16-quantised MLP forward (cpu_member.c)."""

    def __init__(self, widths, seed: int, quantize_bf16: bool = True):
        self.widths = [int(w) for w in widths]
        arr = (C.c_int * len(self.widths))(*self.widths)
        self._h = orc().orc_mlp_create(len(self.widths) - 1, arr, seed, int(quantize_bf16))
        if not self._h:
            raise ValueError("bad MLP shape")

    def forward(self, X: np.ndarray) -> np.ndarray:
        X = np.ascontiguousarray(X, dtype=np.float32)
        out = np.zeros((X.shape[0], self.widths[-1]), dtype=np.float32)
        orc().orc_mlp_forward(self._h, _fp(X), X.shape[0], _fp(out))
        return out

    def logit_scale(self, X: np.ndarray) -> np.ndarray:
        """Conditioning of every logit: |b_c| + sum_j |W[c,j]| |a_j| over the last
        layer's (bf16) inputs a — the magnitude a rounding flip in a hidden
        activation is measured against."""
        a = round_bf16(np.asarray(X, dtype=np.float32)).astype(np.float64)
        for l in range(len(self.widths) - 2):
            w, b = self.layer(l)
            a = round_bf16(np.maximum(a @ w.T.astype(np.float64) + b, 0.0).astype(np.float32))
            a = a.astype(np.float64)
        w, b = self.layer(len(self.widths) - 2)
        return (np.abs(a) @ np.abs(w.T.astype(np.float64)) + np.abs(b)).astype(np.float32)

    def layer(self, l: int):
        fi, fo = self.widths[l], self.widths[l + 1]
        w = np.zeros((fo, fi), dtype=np.float32)
        b = np.zeros(fo, dtype=np.float32)
        orc().orc_mlp_layer(self._h, l, _fp(w), _fp(b))
        return w, b

    def __del__(self):
        if getattr(self, "_h", None):
            orc().orc_mlp_destroy(self._h)
            self._h = None


class CpuCnn:
    """Oracle CPU CNN member (cpu_member.c orc_cnn_*): widths = (S, P, c1, c2,
    hidden, classes)."""

    def __init__(self, widths, seed: int, quantize_bf16: bool = True):
        self.widths = [int(w) for w in widths]
        self._h = orc().orc_cnn_create(*self.widths, seed, int(quantize_bf16))
        if not self._h:
            raise ValueError("bad CNN shape")
        S, P, c1, c2, hidden, Cn = self.widths
        G = S // P
        self.dims = [(P * P, c1), (9 * c1, c2), (G * G * c2, hidden), (hidden, Cn)]

    def forward(self, X: np.ndarray) -> np.ndarray:
        X = np.ascontiguousarray(X, dtype=np.float32)
        out = np.zeros((X.shape[0], self.widths[-1]), dtype=np.float32)
        orc().orc_cnn_forward(self._h, _fp(X), X.shape[0], _fp(out))
        return out

    def logit_scale(self, X: np.ndarray) -> np.ndarray:
        """As CpuMlp.logit_scale: |b_c| + sum_j |W[c,j]| |a_j| over the last
        layer's (bf16) inputs."""
        X = np.ascontiguousarray(X, dtype=np.float32)
        hidden = self.widths[4]
        a = np.zeros((X.shape[0], hidden), dtype=np.float32)
        orc().orc_cnn_hidden(self._h, _fp(X), X.shape[0], _fp(a))
        w, b = self.layer(3)
        return (np.abs(a.astype(np.float64)) @ np.abs(w.T.astype(np.float64))
                + np.abs(b)).astype(np.float32)

    def layer(self, l: int):
        fi, fo = self.dims[l]
        w = np.zeros((fo, fi), dtype=np.float32)
        b = np.zeros(fo, dtype=np.float32)
        orc().orc_cnn_layer(self._h, l, _fp(w), _fp(b))
        return w, b

    def __del__(self):
        if getattr(self, "_h", None):
            orc().orc_cnn_destroy(self._h)
            self._h = None


def cpu_member(arch):
    """The oracle member for a product MemberArch-like object (kind, widths,
    weight_seed)."""
    if getattr(arch, "kind", "mlp") == "cnn":
        return CpuCnn(arch.widths, arch.weight_seed)
    return CpuMlp(arch.widths, arch.weight_seed)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, kept in fp32 (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def features(seed: int, rows: int, width: int) -> np.ndarray:
    """Synthetic U[0,1) features (cpu_member.c orc_feature)."""
    X = np.zeros((rows, width), dtype=np.float32)
    orc().orc_fill_features(seed, rows, width, _fp(X))
    return X


def softmax_rows(Z: np.ndarray) -> np.ndarray:
    Z = np.ascontiguousarray(Z, dtype=np.float32)
    P = np.zeros_like(Z)
    orc().orc_softmax_rows(_fp(Z), Z.shape[0], Z.shape[1], _fp(P))
    return P


def fold(rule: int, blocks, weights=None):
    """cpu_member.c orc_fold: rule 0 avg, 1 vote, 2 wavg -> (Y, winners)."""
    arrs = [np.ascontiguousarray(b, dtype=np.float32) for b in blocks]
    rows, Cw = arrs[0].shape
    ptrs = (f32p * len(arrs))(*[_fp(a) for a in arrs])
    w = (C.c_double * len(arrs))(*(weights or [0.0] * len(arrs)))
    Y = np.zeros((rows, Cw), dtype=np.float32)
    W = np.zeros(rows, dtype=np.int32)
    orc().orc_fold(rule, len(arrs), rows, Cw, ptrs, w, _fp(Y), W.ctypes.data_as(i32p))
    return Y, W


# ------------------------------------------------------------------ reference
class _Dev(C.Structure):
    _fields_ = [("kind", C.c_int), ("memory_mib", C.c_double), ("compute_rate", C.c_double),
                ("batch_overhead_s", C.c_double)]


class _Model(C.Structure):
    _fields_ = [("name", C.c_char_p), ("weight_mib", C.c_double),
                ("act_mib_per_sample", C.c_double), ("cost_per_sample", C.c_double),
                ("output_width", C.c_int)]


class _Cluster(C.Structure):
    _fields_ = [("devices", C.POINTER(_Dev)), ("n_devices", C.c_int),
                ("models", C.POINTER(_Model)), ("n_models", C.c_int), ("menu", i32p),
                ("menu_size", C.c_int), ("segment_size", C.c_int)]


class _Roster(C.Structure):
    _fields_ = [("layers", i32p), ("widths", i32p), ("seeds", C.POINTER(C.c_uint64)),
                ("quantize_bf16", C.c_int), ("softmax", C.c_int)]


_ref = None


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            build()
        lib = C.CDLL(str(REF_SO))
        P = C.POINTER
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_validate_matrix": (C.c_int, [P(_Cluster), i32p, C.c_int, C.c_int]),
            "ref_fit_mem": (C.c_int, [P(_Cluster), i32p, f64p]),
            "ref_worst_fit_decreasing": (C.c_int, [P(_Cluster), C.c_int, i32p]),
            "ref_predict_ensemble_throughput": (C.c_double, [P(_Cluster), i32p]),
            "ref_neighborhood": (C.c_int, [P(_Cluster), i32p, i32p, C.c_int]),
            "ref_count_total_matrices": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int]),
            "ref_count_total_neighs": (C.c_longlong, [C.c_int, C.c_int, C.c_int, C.c_longlong]),
            "ref_effective_max_iter": (C.c_int, [C.c_int, C.c_int, C.c_int]),
            "ref_sample_indices": (C.c_int, [C.c_uint64, C.c_size_t, C.c_size_t,
                                             P(C.c_size_t)]),
            "ref_bounded_greedy_analytic": (C.c_int, [P(_Cluster), i32p, C.c_int, C.c_int,
                                                      C.c_uint64, i32p, f64p, i32p, f64p, i32p,
                                                      i32p, i32p, i32p]),
            "ref_bbs_analytic": (C.c_int, [P(_Cluster), i32p, i32p, i32p]),
            "ref_accumulate": (C.c_int, [C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int, f64p,
                                         i32p, i32p, C.c_int, P(f32p), f32p, i32p]),
            "ref_run_ensemble": (C.c_int, [P(_Cluster), i32p, P(_Roster), C.c_int, f64p, f32p,
                                           C.c_size_t, C.c_size_t, f32p, i32p, f64p]),
            "ref_run_synthetic": (C.c_int, [P(_Cluster), i32p, C.c_int, f64p, C.c_size_t,
                                            C.c_size_t, f32p, i32p, P(C.c_size_t),
                                            P(C.c_size_t)]),
            "ref_bench_ensemble": (C.c_int, [P(_Cluster), i32p, P(_Roster), f32p, C.c_size_t,
                                             C.c_size_t, C.c_int, f64p, f64p, f64p]),
            "ref_system_create": (C.c_int, [P(_Cluster), i32p, P(_Roster), P(C.c_void_p)]),
            "ref_system_run": (C.c_int, [C.c_void_p, f32p, C.c_size_t, C.c_size_t, f32p, f64p]),
            "ref_system_destroy": (None, [C.c_void_p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _ref = lib
    return _ref


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code  # 2 Allocation 3 Startup 4 Spec 5 Protocol 6 Baseline 7 Cap


def _chk(code: int) -> None:
    if code != 0:
        raise RefError(code, ref().ref_last_error().decode())


class RefCluster:
    def __init__(self, cluster):
        devs = cluster.devices
        mods = cluster.models
        self.d = (_Dev * max(len(devs), 1))()
        for i, d in enumerate(devs):
            self.d[i] = _Dev(0 if str(d.kind).upper() == "CPU" else 1, d.memory_mib,
                             d.compute_rate, d.batch_overhead_s)
        self.names = [m.name.encode() for m in mods]
        self.m = (_Model * max(len(mods), 1))()
        for i, m in enumerate(mods):
            self.m[i] = _Model(self.names[i], m.weight_mib, m.act_mib_per_sample,
                               m.cost_per_sample, m.output_width)
        self.menu = (C.c_int * max(len(cluster.batch_menu), 1))(*cluster.batch_menu)
        self.c = _Cluster(self.d, len(devs), self.m, len(mods), self.menu,
                          len(cluster.batch_menu), cluster.segment_size)
        self.D, self.M = len(devs), len(mods)
        # member roster for the CPU MLP backend
        layers = (C.c_int * max(self.M, 1))()
        widths = (C.c_int * (9 * max(self.M, 1)))()
        seeds = (C.c_uint64 * max(self.M, 1))()
        for i, m in enumerate(mods):
            arch = getattr(m, "arch", None)
            ws = list(getattr(arch, "widths", ()) or ())
            if ws:
                layers[i] = -1 if getattr(arch, "kind", "mlp") == "cnn" else len(ws) - 1
                for j, w in enumerate(ws):
                    widths[9 * i + j] = w
                seeds[i] = getattr(arch, "weight_seed", 0)
        self.layers, self.widths, self.seeds = layers, widths, seeds

    def roster(self, quantize=True, softmax=False):
        return _Roster(self.layers, self.widths, self.seeds, int(quantize), int(softmax))


def _mat(A) -> np.ndarray:
    a = getattr(A, "cells", A)
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def ref_wfd(cluster, default_batch: int) -> np.ndarray:
    rc = RefCluster(cluster)
    out = np.zeros((rc.D, rc.M), dtype=np.int32)
    _chk(ref().ref_worst_fit_decreasing(C.byref(rc.c), default_batch, out.ctypes.data_as(i32p)))
    return out


def ref_throughput(cluster, A) -> float:
    rc = RefCluster(cluster)
    return ref().ref_predict_ensemble_throughput(C.byref(rc.c), _mat(A).ctypes.data_as(i32p))


def ref_fit_mem(cluster, A):
    rc = RefCluster(cluster)
    used = (C.c_double * max(rc.D, 1))()
    code = ref().ref_fit_mem(C.byref(rc.c), _mat(A).ctypes.data_as(i32p), used)
    return list(used)[: rc.D], code == 0


def ref_neighborhood(cluster, A) -> np.ndarray:
    rc = RefCluster(cluster)
    cap = (len(cluster.batch_menu) + 1) * rc.D * rc.M + 1
    out = np.zeros((cap, rc.D, rc.M), dtype=np.int32)
    n = ref().ref_neighborhood(C.byref(rc.c), _mat(A).ctypes.data_as(i32p),
                               out.ctypes.data_as(i32p), cap)
    return out[:n]


def ref_count_total_matrices(B: int, D: int, M: int) -> int:
    buf = C.create_string_buffer(4096)
    _chk(ref().ref_count_total_matrices(B, D, M, buf, len(buf)))
    return int(buf.value.decode())


def ref_sample_indices(seed: int, n: int, k: int) -> list:
    out = (C.c_size_t * max(min(n, k), 1))()
    m = ref().ref_sample_indices(seed, n, k, out)
    return list(out)[:m]


def ref_greedy(cluster, A0, max_iter=10, max_neighs=100, seed=0) -> dict:
    rc = RefCluster(cluster)
    out = np.zeros((rc.D, rc.M), dtype=np.int32)
    cap = max(max_iter, rc.D - rc.M) + 1
    scores = (C.c_double * 2)()
    nbr = (C.c_int * cap)()
    best = (C.c_double * cap)()
    acc = (C.c_int * cap)()
    n_it, stop, calls = C.c_int(), C.c_int(), C.c_int()
    _chk(ref().ref_bounded_greedy_analytic(C.byref(rc.c), _mat(A0).ctypes.data_as(i32p), max_iter,
                                           max_neighs, seed, out.ctypes.data_as(i32p), scores,
                                           nbr, best, acc, C.byref(n_it), C.byref(stop),
                                           C.byref(calls)))
    k = n_it.value
    return {"matrix": out, "start": scores[0], "final": scores[1],
            "neighbors": list(nbr)[:k], "best": list(best)[:k], "accepted": list(acc)[:k],
            "stop": "local_optimum" if stop.value == 0 else "iter_cap", "calls": calls.value}


def ref_bbs(cluster) -> dict:
    rc = RefCluster(cluster)
    out = np.zeros((rc.D, rc.M), dtype=np.int32)
    chosen = (C.c_int * max(rc.M, 1))()
    calls = C.c_int()
    _chk(ref().ref_bbs_analytic(C.byref(rc.c), out.ctypes.data_as(i32p), chosen, C.byref(calls)))
    return {"matrix": out, "chosen": list(chosen)[: rc.M], "calls": calls.value}


def ref_accumulate(nb: int, N: int, rule: int, outputs, order, weights=None):
    """PredictionAccumulator fed (segment, model) blocks of full outputs in order."""
    arrs = [np.ascontiguousarray(o, dtype=np.float32) for o in outputs]
    M = len(arrs)
    Cw = arrs[0].shape[1]
    segs = (C.c_int * len(order))(*[s for s, _ in order])
    mods = (C.c_int * len(order))(*[m for _, m in order])
    ptrs = (f32p * M)(*[_fp(a) for a in arrs])
    w = (C.c_double * M)(*(weights or [0.0] * M))
    Y = np.zeros((nb, Cw), dtype=np.float32)
    W = np.zeros(nb, dtype=np.int32)
    _chk(ref().ref_accumulate(nb, Cw, M, N, rule, w, segs, mods, len(order), ptrs, _fp(Y),
                              W.ctypes.data_as(i32p)))
    return Y, W


def ref_run_ensemble(cluster, A, X: np.ndarray, rule: int = 0, weights=None,
                     quantize=True, softmax=False):
    """The reference InferenceSystem (Deploy) with the oracle CPU member."""
    rc = RefCluster(cluster)
    X = np.ascontiguousarray(X, dtype=np.float32)
    nb, width = X.shape
    Cw = cluster.models[0].output_width
    Y = np.zeros((nb, Cw), dtype=np.float32)
    W = np.zeros(nb, dtype=np.int32)
    el = C.c_double()
    w = (C.c_double * max(rc.M, 1))(*(weights or [0.0] * rc.M))
    roster = rc.roster(quantize, softmax)
    _chk(ref().ref_run_ensemble(C.byref(rc.c), _mat(A).ctypes.data_as(i32p), C.byref(roster),
                                rule, w, _fp(X), nb, width, _fp(Y), W.ctypes.data_as(i32p),
                                C.byref(el)))
    return Y, W, el.value


def ref_run_synthetic(cluster, A, nb: int, width: int = 4, rule: int = 0, weights=None):
    """The reference's run_inference with its own SyntheticBackend."""
    rc = RefCluster(cluster)
    Cw = cluster.models[0].output_width
    Y = np.zeros((nb, Cw), dtype=np.float32)
    W = np.full(nb, -1, dtype=np.int32)
    w = (C.c_double * max(rc.M, 1))(*(weights or [0.0] * rc.M))
    segs, msgs = C.c_size_t(), C.c_size_t()
    _chk(ref().ref_run_synthetic(C.byref(rc.c), _mat(A).ctypes.data_as(i32p), rule, w, nb, width,
                                 _fp(Y), W.ctypes.data_as(i32p), C.byref(segs), C.byref(msgs)))
    return Y, W, segs.value, msgs.value


class RefSystem:
    """A long-lived reference InferenceSystem with the oracle CPU member, for
    timing steady-state runs (bench.py --impl reference)."""

    def __init__(self, cluster, A, softmax=True):
        self.rc = RefCluster(cluster)
        self.roster = self.rc.roster(True, softmax)
        h = C.c_void_p()
        _chk(ref().ref_system_create(C.byref(self.rc.c), _mat(A).ctypes.data_as(i32p),
                                     C.byref(self.roster), C.byref(h)))
        self._h = h

    def run(self, X: np.ndarray, want_output: bool = False):
        X = np.ascontiguousarray(X, dtype=np.float32)
        el = C.c_double()
        Y = np.zeros((X.shape[0], self.rc.m[0].output_width), dtype=np.float32) if want_output else None
        _chk(ref().ref_system_run(self._h, _fp(X), X.shape[0], X.shape[1],
                                  _fp(Y) if want_output else None, C.byref(el)))
        return el.value, Y

    def close(self):
        if getattr(self, "_h", None):
            ref().ref_system_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
