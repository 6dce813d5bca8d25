"""enserve-b200: B200-native ensemble-inference hot path of arXiv 2208.14049.

The product is libenserve_b200.so (C++ host core + hand-written sm_100a CUDA
kernels behind the C ABI in include/enserve_b200.h).  This package is its
Python mirror of the reference's C++ API; see api.py.
"""
from ._abi import EXPORTED, LIB_PATH, lib  # noqa: F401
from .api import *  # noqa: F401,F403
from .api import (AllocationError, AllocationMatrix, BaselineError, CapExceededError,  # noqa: F401
                  ClusterSpec, CombinationRule, DeviceBench, DeviceError, DeviceSpec,
                  EnserveError, GreedyConfig, InferenceSystem, InvalidArgument, Member,
                  MemberArch, ModelSpec, ProtocolError, SampleStore, SpecError, StartupError,
                  bbs_baseline, bench, bounded_greedy, combine, count_total_matrices,
                  count_total_neighs, device_count, effective_max_iter, enumerate_all_matrices,
                  enumerated_neighborhood_stats, fit_mem, mlp_model, cnn_model, more_remaining_memory,
                  neighborhood, num_segments, predict_ensemble_throughput, run_inference,
                  sample_indices, segment_bounds, validate_matrix, worst_fit_decreasing)

__version__ = "0.1.0"
