"""ctypes binding of include/enserve_b200.h (the C ABI of libenserve_b200.so).

The library is loaded from this package directory only; there is no fallback.
If it is missing, importing the package fails with the build command to run.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libenserve_b200.so"
MAX_WIDTHS = 9

c_int_p = C.POINTER(C.c_int)
c_double_p = C.POINTER(C.c_double)
c_float_p = C.POINTER(C.c_float)
c_int32_p = C.POINTER(C.c_int32)
c_size_t_p = C.POINTER(C.c_size_t)


# include/enserve_b200.h ES_ABI_VERSION: the struct layouts below.
ABI_VERSION = 2


class DeviceDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("memory_mib", C.c_double), ("compute_rate", C.c_double),
                ("batch_overhead_s", C.c_double)]


class ModelDesc(C.Structure):
    _fields_ = [("name", C.c_char_p), ("weight_mib", C.c_double),
                ("act_mib_per_sample", C.c_double), ("cost_per_sample", C.c_double),
                ("output_width", C.c_int), ("arch", C.c_int), ("n_widths", C.c_int),
                ("widths", C.c_int * MAX_WIDTHS), ("weight_seed", C.c_uint64),
                ("b200_cost_s", C.c_double), ("b200_overhead_s", C.c_double)]


class ClusterDesc(C.Structure):
    _fields_ = [("devices", C.POINTER(DeviceDesc)), ("n_devices", C.c_int),
                ("models", C.POINTER(ModelDesc)), ("n_models", C.c_int),
                ("batch_menu", c_int_p), ("menu_size", C.c_int), ("segment_size", C.c_int)]


class RuleDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("member_softmax", C.c_int), ("weights", c_double_p)]


class PoolOpts(C.Structure):
    _fields_ = [("device_map", c_int_p), ("n_device_map", C.c_int), ("copy_outputs", C.c_int),
                ("warmup", C.c_int), ("sms_per_worker", C.c_int),
                ("overlap_colocated", C.c_int), ("e2e_chunk_rows", C.c_size_t),
                ("e2e_host_convert", C.c_int), ("e2e_convert_eighths", C.c_int),
                ("dp_equal_split", C.c_int), ("row_partials", C.c_int),
                ("no_peer_stores", C.c_int), ("row_nodes", C.c_int),
                ("dp_claim", C.c_int), ("claim_chunk", C.c_int64), ("pack_batches", C.c_int),
                ("fp32", C.c_int)]


class RunStats(C.Structure):
    _fields_ = [("nb_samples", C.c_size_t), ("segments", C.c_size_t),
                ("data_messages", C.c_size_t), ("elapsed_s", C.c_double)]


class ServiceStatsC(C.Structure):
    _fields_ = [("ready", C.c_int), ("requests_served", C.c_uint64),
                ("samples_served", C.c_uint64), ("flushes", C.c_uint64),
                ("last_flush_throughput", C.c_double), ("pending_requests", C.c_size_t),
                ("pending_samples", C.c_size_t), ("uptime_s", C.c_double)]


class BenchResultC(C.Structure):
    _fields_ = [("throughput", C.c_double), ("elapsed_s", C.c_double),
                ("nb_samples", C.c_size_t), ("n_runs", C.c_int), ("runs", C.c_double * 64),
                ("rsd", C.c_double)]


SCORE_FN = C.CFUNCTYPE(C.c_double, c_int_p, C.c_int, C.c_int, C.c_void_p)


class BenchCfg(C.Structure):
    _fields_ = [("mode", C.c_int), ("fn", SCORE_FN), ("user", C.c_void_p),
                ("calib", C.c_void_p), ("repeats", C.c_int), ("opts", C.POINTER(PoolOpts))]


class GreedyTrace(C.Structure):
    _fields_ = [("start_score", C.c_double), ("final_score", C.c_double),
                ("stop_reason", C.c_int), ("n_iters", C.c_int), ("bench_calls", C.c_int),
                ("iter_cap", C.c_int), ("iter_neighbors", c_int_p), ("iter_best", c_double_p),
                ("iter_accepted", c_int_p)]


# name -> (restype, argtypes)
_SIGS = {
    "es_fit_cost_model": (C.c_int, [c_int_p, c_int_p, c_double_p, C.c_int, C.c_int, c_double_p,
                                    c_double_p, c_double_p, c_double_p, c_double_p, c_double_p]),
    "es_calibrate_cost_model": (C.c_int, [C.POINTER(ClusterDesc), C.c_int, C.c_size_t, C.c_int,
                                          c_double_p, c_double_p, c_double_p, c_double_p,
                                          c_double_p, c_double_p, c_double_p]),
    "es_calibrated_throughput": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, c_int_p, c_double_p]),
    "es_screened_greedy": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, C.c_int, C.c_int, C.c_uint64,
                                     C.c_int, C.POINTER(BenchCfg), C.POINTER(BenchCfg), c_int_p,
                                     C.POINTER(GreedyTrace)]),
    "es_cli_main": (C.c_int, [C.c_int, C.POINTER(C.c_char_p)]),
    "es_cluster_to_json": (C.c_int, [C.POINTER(ClusterDesc), C.c_int, C.c_int, C.c_char_p,
                                     C.c_size_t, c_size_t_p]),
    "es_spec_from_json": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "es_spec_load": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "es_spec_describe": (C.c_int, [C.c_void_p, C.POINTER(ClusterDesc)]),
    "es_spec_destroy": (None, [C.c_void_p]),
    "es_save_json_file": (C.c_int, [C.c_char_p, C.c_char_p]),
    "es_matrix_to_json": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, C.c_int, C.c_char_p,
                                    C.c_size_t, c_size_t_p]),
    "es_matrix_from_json": (C.c_int, [C.POINTER(ClusterDesc), C.c_char_p, c_int_p]),
    "es_digest_hex": (C.c_int, [C.c_char_p, C.c_char_p]),
    "es_cache_key": (C.c_int, [C.POINTER(ClusterDesc), C.c_int, C.c_int, C.c_uint64, C.c_int,
                               C.c_char_p, C.c_size_t, C.c_int, C.c_char_p]),
    "es_cache_key_device": (C.c_int, [C.POINTER(ClusterDesc), C.c_int, C.c_int, C.c_uint64,
                                      C.c_int, C.c_char_p, C.c_size_t, C.c_int, C.c_char_p,
                                      C.c_char_p]),
    "es_device_identity": (C.c_int, [C.c_char_p, C.c_size_t]),
    "es_cache_lookup": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(ClusterDesc), c_int_p,
                                  c_double_p, C.POINTER(C.c_int64), c_int_p]),
    "es_cache_store": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(ClusterDesc), c_int_p,
                                 C.c_double, C.c_int64]),
    "es_abi_version": (C.c_int, []),
    "es_status_name": (C.c_char_p, [C.c_int]),
    "es_last_error": (C.c_char_p, []),
    "es_cluster_validate": (C.c_int, [C.POINTER(ClusterDesc), C.c_char_p, C.c_size_t]),
    "es_matrix_validate": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, c_int_p, c_int_p, C.c_int,
                                     c_int_p]),
    "es_num_segments": (C.c_int, [C.c_size_t, C.c_int, c_size_t_p]),
    "es_segment_bounds": (C.c_int, [C.c_int, C.c_int, C.c_size_t, c_size_t_p, c_size_t_p]),
    "es_segment_shares": (C.c_int, [c_int_p, C.c_int, C.c_int, C.c_size_t, C.c_int,
                                    C.POINTER(C.c_longlong), C.c_int, c_int_p]),
    "es_batch_rows": (C.c_int, [C.c_size_t, C.c_int, C.c_longlong, C.c_longlong, C.c_int,
                                C.POINTER(C.c_longlong), c_int_p, C.c_int, c_int_p]),
    "es_segment_shares_weighted": (C.c_int, [c_int_p, C.c_int, C.c_int, C.c_size_t, C.c_int,
                                             c_double_p, C.POINTER(C.c_longlong), C.c_int,
                                             c_int_p]),
    "es_fit_mem": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, c_double_p, c_int_p]),
    "es_more_remaining_memory": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, C.c_int, c_int_p]),
    "es_predict_ensemble_throughput": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, c_double_p]),
    "es_worst_fit_decreasing": (C.c_int, [C.POINTER(ClusterDesc), C.c_int, c_int_p]),
    "es_neighborhood": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, c_int_p, C.c_int, c_int_p]),
    "es_neighborhood_stats": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, c_size_t_p, c_size_t_p]),
    "es_count_total_matrices": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
    "es_count_total_neighs": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_longlong,
                                        C.POINTER(C.c_longlong)]),
    "es_effective_max_iter": (C.c_int, [C.c_int, C.c_int, C.c_int, c_int_p]),
    "es_enumerate_matrices": (C.c_int, [C.POINTER(ClusterDesc), C.c_char_p, c_int_p, C.c_size_t,
                                        c_size_t_p]),
    "es_sample_indices": (C.c_int, [C.c_uint64, C.c_size_t, C.c_size_t, c_size_t_p]),
    "es_bounded_greedy": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, C.c_int, C.c_int, C.c_uint64,
                                    C.POINTER(BenchCfg), c_int_p, C.POINTER(GreedyTrace)]),
    "es_bbs_baseline": (C.c_int, [C.POINTER(ClusterDesc), C.POINTER(BenchCfg), c_int_p, c_int_p,
                                  c_int_p]),
    "es_device_count": (C.c_int, [c_int_p]),
    "es_store_create": (C.c_int, [c_float_p, C.c_size_t, C.c_size_t, C.c_int,
                                  C.POINTER(C.c_void_p)]),
    "es_store_synthetic": (C.c_int, [C.c_uint64, C.c_size_t, C.c_size_t, C.c_int,
                                     C.POINTER(C.c_void_p)]),
    "es_store_destroy": (None, [C.c_void_p]),
    "es_system_create": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, C.POINTER(RuleDesc),
                                   C.POINTER(PoolOpts), C.POINTER(C.c_void_p)]),
    "es_system_begin_run": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(RuleDesc)]),
    "es_system_broadcast": (C.c_int, [C.c_void_p, c_size_t_p]),
    "es_system_await_run": (C.c_int, [C.c_void_p, c_float_p, c_int32_p, C.POINTER(RunStats)]),
    "es_system_run": (C.c_int, [C.c_void_p, C.c_void_p, c_float_p, c_int32_p,
                                C.POINTER(RunStats)]),
    "es_system_run_host": (C.c_int, [C.c_void_p, c_float_p, C.c_size_t, C.c_size_t, c_float_p,
                                     c_int32_p, c_double_p]),
    "es_host_convert_bf16": (C.c_int, [c_float_p, C.POINTER(C.c_uint16), C.c_size_t]),
    "es_system_info":(C.c_int, [C.c_void_p, c_int_p, c_int_p, c_int_p, c_int_p]),
    "es_system_timing": (C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    "es_system_last_transfer": (C.c_int, [C.c_void_p, c_size_t_p, c_size_t_p]),
    "es_system_kernel_timing": (C.c_int, [C.c_void_p, C.c_int, c_double_p, C.c_char_p,
                                          C.c_size_t, C.c_int, c_int_p]),
    "es_system_shutdown": (C.c_int, [C.c_void_p]),
    "es_system_destroy": (None, [C.c_void_p]),
    "es_run_inference": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, C.POINTER(RuleDesc),
                                   C.c_void_p, C.POINTER(PoolOpts), c_float_p, c_int32_p,
                                   C.POINTER(RunStats)]),
    "es_bench": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, C.c_void_p, C.c_int,
                           C.POINTER(PoolOpts), C.POINTER(BenchResultC)]),
    "es_member_create": (C.c_int, [C.c_int, C.POINTER(ModelDesc), C.c_int, C.c_int, C.c_double,
                                   C.c_double, C.POINTER(C.c_void_p)]),
    "es_member_predict": (C.c_int, [C.c_void_p, c_float_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                    c_float_p]),
    "es_member_destroy": (None, [C.c_void_p]),
    "es_combine": (C.c_int, [C.POINTER(RuleDesc), C.c_int, C.c_int, C.c_size_t,
                             C.POINTER(c_float_p), c_float_p, c_int32_p]),
    "es_system_shares": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), c_double_p]),
    "es_system_routes": (C.c_int, [C.c_void_p, c_int_p, c_int_p, C.c_int, c_int_p]),
    "es_system_claims": (C.c_int, [C.c_void_p, C.c_int, c_int_p, C.c_size_t, c_size_t_p]),
    "es_system_claim_models": (C.c_int, [C.c_void_p, c_int_p, C.c_int, c_int_p]),
    "es_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8), C.c_size_t]),
    "es_comm_create": (C.c_int, [C.POINTER(C.c_uint8), C.c_size_t, C.c_int, C.c_int, C.c_int,
                                 C.POINTER(C.c_void_p)]),
    "es_nccl_version": (C.c_int, [c_int_p]),
    "es_comm_destroy": (None, [C.c_void_p]),
    "es_system_set_gather": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int64), C.c_int]),
    "es_service_create": (C.c_int, [C.POINTER(ClusterDesc), c_int_p, C.POINTER(RuleDesc),
                                    C.POINTER(PoolOpts), C.c_int, C.c_size_t, C.c_longlong,
                                    C.POINTER(C.c_void_p)]),
    "es_service_wait_ready": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.c_char_p,
                                        C.c_size_t]),
    "es_service_submit": (C.c_int, [C.c_void_p, c_float_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "es_request_wait": (C.c_int, [C.c_void_p, c_float_p, c_int32_p]),
    "es_request_destroy": (None, [C.c_void_p]),
    "es_service_stats": (C.c_int, [C.c_void_p, C.POINTER(ServiceStatsC)]),
    "es_service_destroy": (None, [C.c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib() -> C.CDLL:
    """The loaded library (loads on first use; raises if it was never built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing; build it with `python -m paper_2208_14049_b200.build` "
                "(there is no CPU fallback for the enserve-b200 hot path)")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.es_abi_version() != ABI_VERSION:
            raise ImportError("libenserve_b200.so ABI version mismatch")
        _lib = handle
    return _lib
