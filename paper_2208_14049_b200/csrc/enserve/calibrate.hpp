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
// (o >= 0) -- the reference's model form, one overhead per device.  On the
// tensor cores a b-row batch is a b-row tile whose cost depends on the member
// (an 8-row tile costs about what a 128-row one does), so a second fit gives
// every member its own pair:
//     1 / throughput(m, b) = c'_m + o_m / b           (o_m >= 0)
// stored as the spec extension ModelSpec::b200_cost_s / b200_overhead_s.
// `calibrated_throughput` scores a matrix with it the way the device runs it
// (co-located workers time-share their GPU, a data-parallel model's segments
// split in proportion to its workers' rates), and `screened_greedy` uses that
// score to pre-screen each greedy neighbourhood, device-benching only its
// top k (`--bench-mode measured --prescreen k`).
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
  // Per-member form: c'_m, o_m and its misfit.
  std::vector<double> member_cost_s;
  std::vector<double> member_overhead_s;
  double member_rms_rel_error = 0.0;
};

// Throws SpecError when a model has no usable sample.
CostFit fit_cost_model(const std::vector<CostSample>& samples, int n_models);

// Benches every model alone on CUDA device `device` at every menu batch over
// `calib_nb` synthetic samples (repeats: median), then fits.  `measured`
// receives the samples.
CostFit calibrate_cost_model(const ClusterSpec& cluster, int device, std::size_t calib_nb,
                             int repeats, std::vector<CostSample>* measured = nullptr);

// The cluster with the fit applied: GPU rows get compute_rate 1 and the fitted
// overhead, every model its fitted cost_per_sample (CPU rows untouched) and,
// when present, its per-member pair (b200_cost_s, b200_overhead_s).
ClusterSpec apply_cost_fit(const ClusterSpec& cluster, const CostFit& fit);

// Ensemble samples/s of A under the per-member model, as the device runs it:
// worker (d, m) spends t = b200_cost_s + b200_overhead_s / b per sample; a
// data-parallel model's workers take shares proportional to 1/t (the
// runtime's rate-proportional split); every device row (or every group of
// rows sharing a CUDA ordinal in `row_gpu`, when given) runs its workers one
// after another, so the ensemble rate is 1 / max over GPUs of sum(share * t).
// 0 for an invalid or over-memory matrix (cost_model.cpp:29-46's rule).
// Throws SpecError if a member of A is uncalibrated.
double calibrated_throughput(const AllocationMatrix& A, const ClusterSpec& cluster,
                             const std::vector<int>& row_gpu = {});

}  // namespace enserve
