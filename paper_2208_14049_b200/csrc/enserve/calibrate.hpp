// B200-calibrated analytic cost model.
//
// The reference's analytic bench (src/cost/cost_model.cpp:13-46) scores a
// matrix from the spec alone: a worker of model m with batch b on device d
// serves b samples every b*c_m/(R_d/n_d) + o_d seconds (n_d co-located
// workers share the device).  Its inputs -- cost_per_sample c_m, compute_rate
// R_d, batch_overhead_s o_d -- are declared numbers.  Here they are FITTED to
// this box: every member alone on one GPU is benched (device-timed bench())
// at every menu batch, and with R = 1 (costs in seconds)
//     1 / throughput(m, b) = c_m + o / b
// is solved by least squares in relative error for all c_m and one shared o
// (o >= 0).  The calibrated spec then lets `--bench-mode analytic` pre-screen
// greedy neighbourhoods at zero device cost.
#pragma once

#include <vector>

#include "enserve/spec.hpp"

namespace enserve {

struct CostSample {
  int model = 0;
  int batch = 0;
  double throughput = 0.0;  // samples/s of the model alone at this batch
};

struct CostFit {
  std::vector<double> cost_per_sample;  // seconds per sample at R = 1
  double batch_overhead_s = 0.0;
  double rms_rel_error = 0.0;           // of the fitted throughputs vs the samples
};

// Throws SpecError when a model has no usable sample.
CostFit fit_cost_model(const std::vector<CostSample>& samples, int n_models);

// Benches every model alone on CUDA device `device` at every menu batch over
// `calib_nb` synthetic samples (repeats: median), then fits.  `measured`
// receives the samples.
CostFit calibrate_cost_model(const ClusterSpec& cluster, int device, std::size_t calib_nb,
                             int repeats, std::vector<CostSample>* measured = nullptr);

// The cluster with the fit applied: GPU rows get compute_rate 1 and the fitted
// overhead, every model its fitted cost_per_sample (CPU rows untouched).
ClusterSpec apply_cost_fit(const ClusterSpec& cluster, const CostFit& fit);

}  // namespace enserve
