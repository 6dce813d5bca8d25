// B200-calibrated analytic cost model (design in calibrate.hpp).
#include "enserve/calibrate.hpp"

#include <algorithm>
#include <cmath>
#include <memory>

#include "enserve/placement.hpp"
#include "enserve/runtime.hpp"

namespace enserve {

namespace {

// Solves the (n x n) normal equations in place (Gaussian elimination with
// partial pivoting); returns false when singular.
bool solve(std::vector<std::vector<double>> a, std::vector<double> b, std::vector<double>* x) {
  const std::size_t n = b.size();
  for (std::size_t c = 0; c < n; ++c) {
    std::size_t p = c;
    for (std::size_t r = c + 1; r < n; ++r)
      if (std::fabs(a[r][c]) > std::fabs(a[p][c])) p = r;
    if (std::fabs(a[p][c]) < 1e-300) return false;
    std::swap(a[p], a[c]);
    std::swap(b[p], b[c]);
    for (std::size_t r = c + 1; r < n; ++r) {
      const double f = a[r][c] / a[c][c];
      for (std::size_t k = c; k < n; ++k) a[r][k] -= f * a[c][k];
      b[r] -= f * b[c];
    }
  }
  x->assign(n, 0.0);
  for (std::size_t c = n; c-- > 0;) {
    double s = b[c];
    for (std::size_t k = c + 1; k < n; ++k) s -= a[c][k] * (*x)[k];
    (*x)[c] = s / a[c][c];
  }
  return true;
}

// Weighted least squares of  thr * (c_m + o/b) = 1  (relative error), with o
// either free or pinned to 0.
bool fit(const std::vector<CostSample>& s, int M, bool with_overhead, std::vector<double>* x) {
  const int n = M + (with_overhead ? 1 : 0);
  std::vector<std::vector<double>> ata(n, std::vector<double>(n, 0.0));
  std::vector<double> atb(n, 0.0);
  for (const CostSample& q : s) {
    std::vector<std::pair<int, double>> row = {{q.model, q.throughput}};
    if (with_overhead) row.push_back({M, q.throughput / q.batch});
    for (auto [i, vi] : row) {
      atb[i] += vi;
      for (auto [j, vj] : row) ata[i][j] += vi * vj;
    }
  }
  return solve(ata, atb, x);
}

// Per-member least squares of thr * (c + o/b) = 1 over one model's samples;
// o pinned to 0 when the free fit makes it negative.
void fit_member(const std::vector<CostSample>& s, int m, double* c, double* o) {
  double a00 = 0, a01 = 0, a11 = 0, b0 = 0, b1 = 0;
  for (const CostSample& q : s) {
    if (q.model != m) continue;
    const double u = q.throughput, v = q.throughput / q.batch;
    a00 += u * u;
    a01 += u * v;
    a11 += v * v;
    b0 += u;
    b1 += v;
  }
  const double det = a00 * a11 - a01 * a01;
  if (det > 1e-12 * a00 * a11) {
    *c = (b0 * a11 - b1 * a01) / det;
    *o = (a00 * b1 - a01 * b0) / det;
    if (*o >= 0.0 && *c > 0.0) return;
  }
  *o = 0.0;
  *c = b0 / a00;
}

}  // namespace

CostFit fit_cost_model(const std::vector<CostSample>& samples, int n_models) {
  std::vector<CostSample> s;
  std::vector<int> per_model(n_models, 0);
  for (const CostSample& q : samples) {
    if (q.model < 0 || q.model >= n_models || q.batch <= 0 || !(q.throughput > 0.0)) continue;
    s.push_back(q);
    ++per_model[q.model];
  }
  for (int m = 0; m < n_models; ++m)
    if (per_model[m] == 0)
      throw SpecError("cost fit: model " + std::to_string(m) + " has no positive throughput sample");
  std::vector<double> x;
  CostFit out;
  if (fit(s, n_models, true, &x) && x[n_models] >= 0.0) {
    out.batch_overhead_s = x[n_models];
  } else if (!fit(s, n_models, false, &x)) {
    throw SpecError("cost fit: singular system");
  }
  out.cost_per_sample.assign(x.begin(), x.begin() + n_models);
  double ss = 0.0;
  for (const CostSample& q : s) {
    const double pred = q.batch / (q.batch * out.cost_per_sample[q.model] + out.batch_overhead_s);
    ss += (pred / q.throughput - 1.0) * (pred / q.throughput - 1.0);
  }
  out.rms_rel_error = std::sqrt(ss / static_cast<double>(s.size()));
  for (double c : out.cost_per_sample)
    if (!(c > 0.0)) throw SpecError("cost fit: non-positive cost per sample");
  out.member_cost_s.assign(n_models, 0.0);
  out.member_overhead_s.assign(n_models, 0.0);
  for (int m = 0; m < n_models; ++m) fit_member(s, m, &out.member_cost_s[m], &out.member_overhead_s[m]);
  double sm = 0.0;
  for (const CostSample& q : s) {
    const double pred = q.batch / (q.batch * out.member_cost_s[q.model] + out.member_overhead_s[q.model]);
    sm += (pred / q.throughput - 1.0) * (pred / q.throughput - 1.0);
  }
  out.member_rms_rel_error = std::sqrt(sm / static_cast<double>(s.size()));
  return out;
}

CostFit calibrate_cost_model(const ClusterSpec& cluster, int device, std::size_t calib_nb,
                             int repeats, std::vector<CostSample>* measured) {
  std::vector<CostSample> samples;
  for (int m = 0; m < cluster.model_count(); ++m) {
    ClusterSpec solo;
    DeviceSpec d;
    d.id = 0;
    d.kind = DeviceKind::GPU;
    d.memory_mib = 1e12;  // the fit measures speed, not capacity
    d.compute_rate = 1.0;
    solo.devices = {d};
    ModelSpec mm = cluster.models[m];
    mm.id = 0;
    solo.models = {mm};
    solo.batch_menu = cluster.batch_menu;
    solo.segment_size = cluster.segment_size;
    const int width = mm.arch.kind == MemberArch::Kind::Synthetic ? 16 : mm.arch.input_width();
    auto calib = SampleStore::synthetic(7, calib_nb, static_cast<std::size_t>(width), device);
    PoolOptions opts;
    opts.device_map = {device};
    for (int b : cluster.batch_menu) {
      AllocationMatrix A(1, 1);
      A.set(0, 0, b);
      samples.push_back({m, b, bench(A, calib, solo, repeats, opts).throughput});
    }
  }
  if (measured) *measured = samples;
  return fit_cost_model(samples, cluster.model_count());
}

ClusterSpec apply_cost_fit(const ClusterSpec& cluster, const CostFit& fit) {
  ClusterSpec out = cluster;
  for (DeviceSpec& d : out.devices)
    if (d.kind == DeviceKind::GPU) {
      d.compute_rate = 1.0;
      d.batch_overhead_s = fit.batch_overhead_s;
    }
  for (int m = 0; m < out.model_count(); ++m) {
    out.models[m].cost_per_sample = fit.cost_per_sample.at(m);
    if (m < static_cast<int>(fit.member_cost_s.size())) {
      out.models[m].b200_cost_s = fit.member_cost_s[m];
      out.models[m].b200_overhead_s = fit.member_overhead_s[m];
    }
  }
  return out;
}

double calibrated_throughput(const AllocationMatrix& A, const ClusterSpec& cluster,
                             const std::vector<int>& row_gpu) {
  try {
    if (!validate_matrix(A, cluster).ok) return 0.0;
  } catch (const SpecError&) {
    return 0.0;
  }
  if (!fit_mem(A, cluster).fits) return 0.0;
  const int D = A.device_count(), M = A.model_count();
  if (!row_gpu.empty() && static_cast<int>(row_gpu.size()) != D)
    throw SpecError("calibrated_throughput: row_gpu needs one entry per device row");
  auto t = [&](int d, int m) {
    const ModelSpec& mm = cluster.models[m];
    return mm.b200_cost_s + mm.b200_overhead_s / A.at(d, m);
  };
  std::vector<double> rate_sum(M, 0.0);
  for (int m = 0; m < M; ++m) {
    if (!(cluster.models[m].b200_cost_s > 0.0))
      throw SpecError("calibrated_throughput: model " + cluster.models[m].name +
                      " has no B200 calibration (run calibrate first)");
    for (int d = 0; d < D; ++d)
      if (A.at(d, m) > 0) rate_sum[m] += 1.0 / t(d, m);
  }
  std::vector<double> busy;  // seconds per ensemble sample, per GPU
  for (int d = 0; d < D; ++d) {
    const int g = row_gpu.empty() ? d : row_gpu[d];
    if (g < 0) throw SpecError("calibrated_throughput: negative GPU index");
    if (static_cast<int>(busy.size()) <= g) busy.resize(g + 1, 0.0);
    for (int m = 0; m < M; ++m)
      if (A.at(d, m) > 0) busy[g] += (1.0 / t(d, m)) / rate_sum[m] * t(d, m);
  }
  double worst = 0.0;
  for (double b : busy) worst = std::max(worst, b);
  return worst > 0.0 ? 1.0 / worst : 0.0;
}

}  // namespace enserve
