// Memory / cost models and worst-fit-decreasing.
// Behaviour: /root/reference/proj/src/memory/memory_model.cpp:7-50,
// /root/reference/proj/src/cost/cost_model.cpp:9-46,
// /root/reference/proj/src/opt/optimizer.cpp:26-64.
#include "enserve/placement.hpp"

#include <cmath>
#include <stdexcept>

#include <algorithm>
#include <limits>
#include <numeric>

namespace enserve {

double worker_memory(const ModelSpec& model, int batch) {
  if (batch < 1) throw std::invalid_argument("batch must be >= 1");
  return model.weight_mib + batch * model.act_mib_per_sample;
}

double device_load(const AllocationMatrix& A, int device_id, const ClusterSpec& cluster) {
  // Accumulate in model-id order: the order fixes the rounding of the sum.
  double total = 0.0;
  for (int m = 0; m < A.model_count(); ++m)
    if (int b = A.at(device_id, m); b > 0) total += worker_memory(cluster.models[m], b);
  return total;
}

MemoryReport fit_mem(const AllocationMatrix& A, const ClusterSpec& cluster) {
  MemoryReport rep;
  rep.fits = true;
  rep.per_device.reserve(cluster.devices.size());
  for (int d = 0; d < cluster.device_count(); ++d) {
    DeviceLoad load{d, device_load(A, d, cluster), cluster.devices[d].memory_mib};
    rep.fits = rep.fits && !(load.used_mib > load.capacity_mib);
    rep.per_device.push_back(load);
  }
  return rep;
}

std::optional<int> more_remaining_memory(const AllocationMatrix& A, int /*default_batch*/,
                                         DeviceKind kind, const ClusterSpec& cluster) {
  std::optional<int> pick;
  double pick_free = 0.0;
  for (int d = 0; d < cluster.device_count(); ++d) {
    if (cluster.devices[d].kind != kind) continue;
    double free_mib = cluster.devices[d].memory_mib - device_load(A, d, cluster);
    // Strictly larger wins, so equal headroom keeps the lower id.
    if (!pick.has_value() || free_mib > pick_free) {
      pick = d;
      pick_free = free_mib;
    }
  }
  return pick;
}

int colocated_count(const AllocationMatrix& A, int device_id) {
  return A.row_worker_count(device_id);
}

double service_time(const WorkerPlacement& p, const ClusterSpec& cluster) {
  const DeviceSpec& dev = cluster.devices[p.device_id];
  const double rate_share = dev.compute_rate / p.colocated_count;
  const double work = p.batch * cluster.models[p.model_id].cost_per_sample;
  return work / rate_share + dev.batch_overhead_s;
}

double worker_throughput(const WorkerPlacement& p, const ClusterSpec& cluster) {
  const double t = service_time(p, cluster);
  if (t <= 0.0) return std::numeric_limits<double>::infinity();
  return p.batch / t;
}

double predict_ensemble_throughput(const AllocationMatrix& A, const ClusterSpec& cluster) {
  if (!validate_matrix(A, cluster).ok || !fit_mem(A, cluster).fits) return 0.0;
  double bottleneck = std::numeric_limits<double>::infinity();
  for (int m = 0; m < A.model_count(); ++m) {
    double rate = 0.0;  // data-parallel workers of one model add up
    for (int d = 0; d < A.device_count(); ++d)
      if (int b = A.at(d, m); b != 0)
        rate += worker_throughput(WorkerPlacement{m, d, b, colocated_count(A, d)}, cluster);
    bottleneck = std::min(bottleneck, rate);
  }
  return bottleneck;
}

std::vector<int> models_heaviest_first(const ClusterSpec& cluster) {
  std::vector<int> ids(cluster.models.size());
  std::iota(ids.begin(), ids.end(), 0);
  std::stable_sort(ids.begin(), ids.end(), [&](int x, int y) {
    return cluster.models[x].weight_mib > cluster.models[y].weight_mib;
  });
  return ids;
}

std::vector<SegmentShare> segment_shares(const AllocationMatrix& A, std::size_t nb_samples,
                                         int segment_size) {
  const long long S = static_cast<long long>(num_segments(nb_samples, segment_size));
  std::vector<int> seen(A.model_count(), 0);
  std::vector<SegmentShare> out;
  for (int d = 0; d < A.device_count(); ++d)
    for (int m = 0; m < A.model_count(); ++m) {
      if (A.at(d, m) == 0) continue;
      const long long k = seen[m]++, n = A.column_worker_count(m);
      out.push_back({d, m, S * k / n, S * (k + 1) / n});
    }
  return out;
}

std::vector<SegmentShare> segment_shares_weighted(const AllocationMatrix& A,
                                                  std::size_t nb_samples, int segment_size,
                                                  const std::vector<double>& weight) {
  std::vector<SegmentShare> out = segment_shares(A, nb_samples, segment_size);
  if (weight.size() != out.size()) throw std::invalid_argument("one weight per worker");
  const long long S = static_cast<long long>(num_segments(nb_samples, segment_size));
  for (int m = 0; m < A.model_count(); ++m) {
    std::vector<std::size_t> ws;
    double total = 0.0;
    bool equal = true;
    for (std::size_t i = 0; i < out.size(); ++i)
      if (out[i].model == m) {
        if (!(weight[i] > 0.0) || !std::isfinite(weight[i]))
          throw std::invalid_argument("worker weights must be positive");
        if (!ws.empty() && weight[i] != weight[ws[0]]) equal = false;
        ws.push_back(i);
        total += weight[i];
      }
    if (ws.size() < 2 || equal) continue;  // keep the equal split bit for bit
    double cum = 0.0;
    long long prev = 0;
    for (std::size_t k = 0; k < ws.size(); ++k) {
      cum += weight[ws[k]];
      const long long end =
          k + 1 == ws.size() ? S : std::max(prev, std::llround(static_cast<double>(S) * cum / total));
      out[ws[k]].begin = prev;
      out[ws[k]].end = end;
      prev = end;
    }
  }
  return out;
}

AllocationMatrix worst_fit_decreasing(const ClusterSpec& cluster, int default_batch) {
  if (!cluster.menu_contains(default_batch))
    throw SpecError("default batch " + std::to_string(default_batch) +
                    " is not in the batch menu");
  AllocationMatrix A(cluster.device_count(), cluster.model_count());
  for (int m : models_heaviest_first(cluster)) {
    bool placed = false;
    for (DeviceKind tier : {DeviceKind::GPU, DeviceKind::CPU}) {
      std::optional<int> d = more_remaining_memory(A, default_batch, tier, cluster);
      if (!d.has_value()) continue;
      AllocationMatrix trial = A;
      trial.set(*d, m, default_batch);
      if (fit_mem(trial, cluster).fits) {
        A = std::move(trial);
        placed = true;
        break;
      }
    }
    if (!placed) {
      const std::string& name = cluster.models[m].name;
      throw AllocationError(name, "no device has enough memory for model '" + name + "'");
    }
  }
  return A;
}

}  // namespace enserve
