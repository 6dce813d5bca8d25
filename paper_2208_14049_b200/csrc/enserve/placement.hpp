// Memory model, analytic cost model and worst-fit-decreasing placement.
//
// API mirror of
//   /root/reference/proj/include/enserve/memory/memory_model.hpp:10-40
//   /root/reference/proj/include/enserve/cost/cost_model.hpp:8-32
//   /root/reference/proj/include/enserve/opt/optimizer.hpp:49-54 (WFD)
// Every double is produced by the same operation sequence as the reference
// (same summation order, same association), so placements and analytic scores
// are bit-identical — tests/test_placement.py checks this against the compiled
// reference.
#pragma once

#include <optional>
#include <vector>

#include "enserve/spec.hpp"

namespace enserve {

struct DeviceLoad {
  int device_id = 0;
  double used_mib = 0.0;
  double capacity_mib = 0.0;
  double remaining_mib() const { return capacity_mib - used_mib; }
};

struct MemoryReport {
  std::vector<DeviceLoad> per_device;
  bool fits = false;
};

double worker_memory(const ModelSpec& model, int batch);
double device_load(const AllocationMatrix& A, int device_id, const ClusterSpec& cluster);
MemoryReport fit_mem(const AllocationMatrix& A, const ClusterSpec& cluster);
std::optional<int> more_remaining_memory(const AllocationMatrix& A, int default_batch,
                                         DeviceKind kind, const ClusterSpec& cluster);

struct WorkerPlacement {
  int model_id = 0;
  int device_id = 0;
  int batch = 1;
  int colocated_count = 1;
};

int colocated_count(const AllocationMatrix& A, int device_id);
double service_time(const WorkerPlacement& placement, const ClusterSpec& cluster);
double worker_throughput(const WorkerPlacement& placement, const ClusterSpec& cluster);
double predict_ensemble_throughput(const AllocationMatrix& A, const ClusterSpec& cluster);

// Algorithm 1 of the paper: heaviest model first, each onto the GPU with the
// most remaining memory (CPU only when no GPU fits), at default_batch.
AllocationMatrix worst_fit_decreasing(const ClusterSpec& cluster, int default_batch);

// Model ids sorted by weight_mib descending, ties by ascending id.
std::vector<int> models_heaviest_first(const ClusterSpec& cluster);

// Which segments each worker (nonzero cell, row-major) predicts in one run:
// a model's workers split [0, S) into contiguous, equal runs in worker order,
// so every segment is predicted exactly once per model (the property the
// reference's shared per-model FIFO gives, tests/test_runtime.cpp:282-313).
struct SegmentShare {
  int device = 0;
  int model = 0;
  long long begin = 0;  // segment ids [begin, end)
  long long end = 0;
};
std::vector<SegmentShare> segment_shares(const AllocationMatrix& A, std::size_t nb_samples,
                                         int segment_size);
// The same split with a model's runs proportional to `weight` (one entry per
// worker, row-major cell order; e.g. measured rows/s): the static fallback of
// SURVEY.md §8-E for the reference's shared FIFO, where a faster
// data-parallel worker pulls more segments.  Contiguous, exactly once; equal
// weights give segment_shares' split exactly.
std::vector<SegmentShare> segment_shares_weighted(const AllocationMatrix& A,
                                                  std::size_t nb_samples, int segment_size,
                                                  const std::vector<double>& weight);

}  // namespace enserve
