// Allocation-matrix search: neighbourhood, matrix-space combinatorics, the
// bounded greedy optimizer (paper Alg. 2) and the batch-size-only baseline.
//
// API mirror of /root/reference/proj/include/enserve/opt/optimizer.hpp:17-112.
// bench() is injected as a ScoreFn exactly as there (optimizer.hpp:18), so the
// same greedy drives the device-timed B200 bench (system.hpp) or the analytic
// cost model.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "enserve/bigint.hpp"
#include "enserve/spec.hpp"

namespace enserve {

using BigInt = BigUInt;
using ScoreFn = std::function<double(const AllocationMatrix&)>;
using ClusterScoreFn = std::function<double(const AllocationMatrix&, const ClusterSpec&)>;

struct GreedyConfig {
  int max_iter = 10;
  int max_neighs = 100;
  std::uint64_t rng_seed = 0;
};

enum class StopReason { local_optimum, iter_cap };
std::string to_string(StopReason reason);

struct GreedyIteration {
  int index = 0;
  int neighbors_evaluated = 0;
  double best_score = 0.0;
  bool accepted = false;
};

struct OptimizationTrace {
  std::vector<GreedyIteration> iterations;
  double start_score = 0.0;
  double final_score = 0.0;
  StopReason stop_reason = StopReason::local_optimum;
  int bench_calls() const;
};

std::vector<AllocationMatrix> neighborhood(const AllocationMatrix& A, const ClusterSpec& cluster);

struct NeighborhoodStats {
  std::size_t size = 0;
  std::size_t forbidden = 0;
};
NeighborhoodStats enumerated_neighborhood_stats(const AllocationMatrix& A,
                                                const ClusterSpec& cluster);

BigInt count_total_matrices(int menu_size, int device_count, int model_count);
long long count_total_neighs(int menu_size, int device_count, int model_count,
                             long long forbidden);

void for_each_matrix(const ClusterSpec& cluster, BigInt cap,
                     const std::function<void(const AllocationMatrix&)>& visit);
std::vector<AllocationMatrix> enumerate_all_matrices(const ClusterSpec& cluster, BigInt cap);

int effective_max_iter(int device_count, int model_count, int max_iter);

struct GreedyResult {
  AllocationMatrix matrix;
  OptimizationTrace trace;
};
GreedyResult bounded_greedy(const AllocationMatrix& A0, const ClusterSpec& cluster,
                            const ScoreFn& bench, const GreedyConfig& config);

// bounded_greedy with a pre-screen: the same start,
// neighbourhood, seeded subsample and acceptance rule (optimizer.cpp:178-227),
// but each iteration ranks its sampled neighbours by `screen` (the calibrated
// analytic model: no device time) and benches only the best `top_k` of them
// (ties keep neighbourhood order; neighbours the screen scores 0 -- invalid or
// over memory -- are never benched).  top_k >= max_neighs is bounded_greedy.
// trace.iterations[i].neighbors_evaluated counts the benched neighbours.
GreedyResult screened_greedy(const AllocationMatrix& A0, const ClusterSpec& cluster,
                             const ScoreFn& bench, const ScoreFn& screen,
                             const GreedyConfig& config, int top_k);

struct BaselineResult {
  AllocationMatrix matrix;
  int bench_calls = 0;
  std::vector<int> chosen_batches;
};
BaselineResult bbs_baseline(const ClusterSpec& cluster, const ClusterScoreFn& bench);

}  // namespace enserve
