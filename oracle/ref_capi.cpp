// ORACLE — test infrastructure only.  A flat C ABI over the UNMODIFIED
// reference (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libenserve_ref.so) so pytest and bench.py can drive it through
// ctypes.  Nothing here is reference source: it only calls the reference's
// public API (include/enserve/**) and plugs the oracle's CPU member
// (cpu_member.c) into the reference's PredictorFactory seam
// (/root/reference/proj/include/enserve/runtime/backend.hpp:25-41).
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "cpu_member.h"
#include "enserve/cost/cost_model.hpp"
#include "enserve/memory/memory_model.hpp"
#include "enserve/opt/optimizer.hpp"
#include "enserve/runtime/backend.hpp"
#include "enserve/runtime/combine.hpp"
#include "enserve/runtime/pipeline.hpp"
#include "enserve/util/rng.hpp"

using namespace enserve;

extern "C" {

struct ref_device {
  int kind;  // 0 = CPU, 1 = GPU
  double memory_mib;
  double compute_rate;
  double batch_overhead_s;
};

struct ref_model {
  const char* name;
  double weight_mib;
  double act_mib_per_sample;
  double cost_per_sample;
  int output_width;
};

struct ref_cluster {
  const ref_device* devices;
  int n_devices;
  const ref_model* models;
  int n_models;
  const int* menu;
  int menu_size;
  int segment_size;
};

// Member architecture for the CPU backend: layers[m] dense layers with
// widths[m*9 .. m*9+layers[m]] (input, hidden..., classes), or layers[m] = -1
// for a CNN member with widths[m*9 .. m*9+5] = {S, P, c1, c2, hidden, classes}.
struct ref_roster {
  const int* layers;
  const int* widths;
  const std::uint64_t* seeds;
  int quantize_bf16;
  int softmax;  // predictor emits softmax(logits) instead of logits
};

}  // extern "C"

namespace {

thread_local std::string g_error;

ClusterSpec to_cluster(const ref_cluster* c) {
  ClusterSpec s;
  for (int d = 0; d < c->n_devices; ++d) {
    const ref_device& x = c->devices[d];
    s.devices.push_back({d, x.kind == 0 ? DeviceKind::CPU : DeviceKind::GPU,
                         x.memory_mib, x.compute_rate, x.batch_overhead_s});
  }
  for (int m = 0; m < c->n_models; ++m) {
    const ref_model& x = c->models[m];
    s.models.push_back({m, x.name ? std::string(x.name) : "m" + std::to_string(m),
                        x.weight_mib, x.act_mib_per_sample, x.cost_per_sample,
                        x.output_width});
  }
  s.batch_menu.assign(c->menu, c->menu + c->menu_size);
  s.segment_size = c->segment_size;
  return s;
}

AllocationMatrix to_matrix(const int* a, int D, int M) {
  AllocationMatrix A(D, M);
  for (int d = 0; d < D; ++d)
    for (int m = 0; m < M; ++m) A.set(d, m, a[d * M + m]);
  return A;
}

void from_matrix(const AllocationMatrix& A, int* out) {
  for (int d = 0; d < A.device_count(); ++d)
    for (int m = 0; m < A.model_count(); ++m) out[d * A.model_count() + m] = A.at(d, m);
}

// The oracle member behind the reference's own Predictor seam.
class CpuMlpBackend : public PredictorFactory {
 public:
  CpuMlpBackend(const ref_roster* r, int n_models) : softmax_(r->softmax != 0) {
    for (int m = 0; m < n_models; ++m) {
      Member mem;
      const int* w = r->widths + 9 * m;
      if (r->layers[m] < 0)
        mem.cnn.reset(orc_cnn_create(w[0], w[1], w[2], w[3], w[4], w[5], r->seeds[m],
                                     r->quantize_bf16));
      else
        mem.mlp.reset(orc_mlp_create(r->layers[m], w, r->seeds[m], r->quantize_bf16));
      members_.push_back(std::move(mem));
    }
  }
  std::unique_ptr<Predictor> make(const WorkerContext& ctx) const override {
    return std::make_unique<CpuMemberPredictor>(ctx, &members_.at(ctx.model.id), softmax_);
  }
  std::string name() const override { return "oracle-cpu-member"; }

 private:
  struct Member {
    std::unique_ptr<orc_mlp, void (*)(orc_mlp*)> mlp{nullptr, &orc_mlp_destroy};
    std::unique_ptr<orc_cnn, void (*)(orc_cnn*)> cnn{nullptr, &orc_cnn_destroy};
  };
  class CpuMemberPredictor : public Predictor {
   public:
    CpuMemberPredictor(const WorkerContext& ctx, const Member* m, bool softmax)
        : ctx_(ctx), m_(m), softmax_(softmax) {}
    // Same capacity rule as SyntheticPredictor::load (backend.cpp:41).
    bool load() override { return ctx_.device_load_mib <= ctx_.device.memory_mib; }
    void predict(const SampleView& in, std::span<float> out) override {
      int C;
      if (m_->cnn) {
        orc_cnn_forward(m_->cnn.get(), in.features.data(), in.rows, out.data());
        C = orc_cnn_classes(m_->cnn.get());
      } else {
        orc_mlp_forward(m_->mlp.get(), in.features.data(), in.rows, out.data());
        C = orc_mlp_classes(m_->mlp.get());
      }
      if (softmax_) {
        std::vector<float> z(out.begin(), out.end());
        orc_softmax_rows(z.data(), in.rows, C, out.data());
      }
    }

   private:
    WorkerContext ctx_;
    const Member* m_;
    bool softmax_;
  };
  std::vector<Member> members_;
  bool softmax_;
};

CombinationRule make_rule(int rule, const double* weights, int M) {
  if (rule == 1) return CombinationRule::majority_vote();
  if (rule == 2) return CombinationRule::weighted(std::vector<double>(weights, weights + M));
  return CombinationRule::averaging();
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const AllocationError& e) {
    g_error = e.what();
    return 2;
  } catch (const StartupError& e) {
    g_error = e.what();
    return 3;
  } catch (const SpecError& e) {
    g_error = e.what();
    return 4;
  } catch (const ProtocolError& e) {
    g_error = e.what();
    return 5;
  } catch (const BaselineError& e) {
    g_error = e.what();
    return 6;
  } catch (const CapExceededError& e) {
    g_error = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

int ref_validate_matrix(const ref_cluster* c, const int* a, int D, int M) {
  return guarded([&] { return validate_matrix(to_matrix(a, D, M), to_cluster(c)).ok ? 0 : 8; });
}

int ref_fit_mem(const ref_cluster* c, const int* a, double* used) {
  return guarded([&] {
    ClusterSpec s = to_cluster(c);
    MemoryReport r = fit_mem(to_matrix(a, s.device_count(), s.model_count()), s);
    for (std::size_t d = 0; d < r.per_device.size(); ++d) used[d] = r.per_device[d].used_mib;
    return r.fits ? 0 : 9;
  });
}

int ref_worst_fit_decreasing(const ref_cluster* c, int default_batch, int* out) {
  return guarded([&] {
    from_matrix(worst_fit_decreasing(to_cluster(c), default_batch), out);
    return 0;
  });
}

double ref_predict_ensemble_throughput(const ref_cluster* c, const int* a) {
  ClusterSpec s = to_cluster(c);
  return predict_ensemble_throughput(to_matrix(a, s.device_count(), s.model_count()), s);
}

// Returns the neighbour count; writes at most cap matrices.
int ref_neighborhood(const ref_cluster* c, const int* a, int* out, int cap) {
  ClusterSpec s = to_cluster(c);
  int D = s.device_count(), M = s.model_count();
  std::vector<AllocationMatrix> n = neighborhood(to_matrix(a, D, M), s);
  for (int i = 0; i < static_cast<int>(n.size()) && i < cap; ++i) from_matrix(n[i], out + i * D * M);
  return static_cast<int>(n.size());
}

int ref_count_total_matrices(int B, int D, int M, char* buf, int buflen) {
  return guarded([&] {
    std::string s = count_total_matrices(B, D, M).str();
    std::snprintf(buf, buflen, "%s", s.c_str());
    return 0;
  });
}

long long ref_count_total_neighs(int B, int D, int M, long long forbidden) {
  return count_total_neighs(B, D, M, forbidden);
}

int ref_effective_max_iter(int D, int M, int max_iter) { return effective_max_iter(D, M, max_iter); }

// Reference rng stream (include/enserve/util/rng.hpp:13-38).
int ref_sample_indices(std::uint64_t seed, std::size_t n, std::size_t k, std::size_t* out) {
  std::mt19937_64 rng(seed);
  std::vector<std::size_t> v = sample_indices(rng, n, k);
  std::memcpy(out, v.data(), v.size() * sizeof(std::size_t));
  return static_cast<int>(v.size());
}

// bounded_greedy (src/opt/optimizer.cpp:178-227) with the analytic bench the
// reference's own optimizer tests use (tests/test_optimizer.cpp:15-19).
int ref_bounded_greedy_analytic(const ref_cluster* c, const int* a0, int max_iter,
                                int max_neighs, std::uint64_t seed, int* out,
                                double* scores /* start, final */, int* iter_neighbors,
                                double* iter_best, int* iter_accepted, int* n_iters,
                                int* stop_reason, int* calls) {
  return guarded([&] {
    ClusterSpec s = to_cluster(c);
    int D = s.device_count(), M = s.model_count();
    int n_calls = 0;
    ScoreFn f = [&](const AllocationMatrix& A) {
      ++n_calls;
      return predict_ensemble_throughput(A, s);
    };
    GreedyResult r = bounded_greedy(to_matrix(a0, D, M), s, f,
                                    {max_iter, max_neighs, seed});
    from_matrix(r.matrix, out);
    scores[0] = r.trace.start_score;
    scores[1] = r.trace.final_score;
    *n_iters = static_cast<int>(r.trace.iterations.size());
    for (std::size_t i = 0; i < r.trace.iterations.size(); ++i) {
      iter_neighbors[i] = r.trace.iterations[i].neighbors_evaluated;
      iter_best[i] = r.trace.iterations[i].best_score;
      iter_accepted[i] = r.trace.iterations[i].accepted ? 1 : 0;
    }
    *stop_reason = r.trace.stop_reason == StopReason::local_optimum ? 0 : 1;
    *calls = n_calls;
    return 0;
  });
}

int ref_bbs_analytic(const ref_cluster* c, int* out, int* chosen, int* calls) {
  return guarded([&] {
    ClusterSpec s = to_cluster(c);
    BaselineResult r = bbs_baseline(s, [](const AllocationMatrix& A, const ClusterSpec& cl) {
      return predict_ensemble_throughput(A, cl);
    });
    from_matrix(r.matrix, out);
    for (std::size_t m = 0; m < r.chosen_batches.size(); ++m) chosen[m] = r.chosen_batches[m];
    *calls = r.bench_calls;
    return 0;
  });
}

// Feeds PredictionAccumulator (src/runtime/combine.cpp:60-136) the segment
// blocks of full per-model outputs in the given arrival order.
int ref_accumulate(std::size_t nb, int C, int M, int N, int rule, const double* weights,
                   const int* order_seg, const int* order_model, int n_msgs,
                   const float* const* outputs, float* y, int* winners) {
  return guarded([&] {
    PredictionAccumulator acc(nb, C, M, N, make_rule(rule, weights, M));
    for (int i = 0; i < n_msgs; ++i) {
      Segment seg = segment_bounds(order_seg[i], N, nb);
      const float* src = outputs[order_model[i]] + seg.start * C;
      acc.add(PredictionMessage::data(order_seg[i], order_model[i], seg.size(),
                                      std::vector<float>(src, src + seg.size() * C)));
    }
    if (!acc.complete()) return 10;
    std::memcpy(y, acc.combined().data(), nb * C * sizeof(float));
    if (rule == 1) std::memcpy(winners, acc.winners().data(), nb * sizeof(int));
    return 0;
  });
}

// run_inference in Deploy mode (src/runtime/pipeline.cpp:418-444) with the
// oracle CPU member behind the reference's InferenceSystem.
int ref_run_ensemble(const ref_cluster* c, const int* a, const ref_roster* roster, int rule,
                     const double* weights, const float* X, std::size_t nb, std::size_t width,
                     float* Y, int* winners, double* elapsed_s) {
  return guarded([&] {
    ClusterSpec s = to_cluster(c);
    int D = s.device_count(), M = s.model_count();
    CpuMlpBackend backend(roster, M);
    auto store = std::make_shared<SampleStore>(std::vector<float>(X, X + nb * width), nb, width);
    InferenceResult r = run_inference(store, to_matrix(a, D, M), s, backend,
                                      make_rule(rule, weights, M), Mode::Deploy);
    const RunOutput& out = *r.output;
    std::memcpy(Y, out.combined.data(), out.combined.size() * sizeof(float));
    if (winners && !out.winners.empty())
      std::memcpy(winners, out.winners.data(), out.winners.size() * sizeof(int));
    *elapsed_s = out.stats.elapsed_s;
    return 0;
  });
}

// run_inference (Deploy) with the reference's OWN SyntheticBackend
// (src/runtime/backend.cpp:33-60): the plumbing-parity oracle.
int ref_run_synthetic(const ref_cluster* c, const int* a, int rule, const double* weights,
                      std::size_t nb, std::size_t width, float* Y, int* winners,
                      std::size_t* segments, std::size_t* messages) {
  return guarded([&] {
    ClusterSpec s = to_cluster(c);
    int D = s.device_count(), M = s.model_count();
    SyntheticBackend backend;
    auto store = std::make_shared<SampleStore>(std::vector<float>(nb * width, 0.0f), nb, width);
    InferenceResult r = run_inference(store, to_matrix(a, D, M), s, backend,
                                      make_rule(rule, weights, M), Mode::Deploy);
    const RunOutput& out = *r.output;
    if (!out.combined.empty()) std::memcpy(Y, out.combined.data(), out.combined.size() * sizeof(float));
    if (winners && !out.winners.empty())
      std::memcpy(winners, out.winners.data(), out.winners.size() * sizeof(int));
    *segments = out.stats.segments;
    *messages = out.stats.data_messages;
    return 0;
  });
}

// bench (src/runtime/pipeline.cpp:465-501) with the oracle CPU member.
int ref_bench_ensemble(const ref_cluster* c, const int* a, const ref_roster* roster,
                       const float* X, std::size_t nb, std::size_t width, int repeats,
                       double* throughput, double* rsd, double* runs) {
  return guarded([&] {
    ClusterSpec s = to_cluster(c);
    int D = s.device_count(), M = s.model_count();
    CpuMlpBackend backend(roster, M);
    auto store = std::make_shared<SampleStore>(std::vector<float>(X, X + nb * width), nb, width);
    BenchResult r = bench(to_matrix(a, D, M), store, s, backend, repeats);
    *throughput = r.throughput;
    *rsd = r.rsd;
    for (std::size_t i = 0; i < r.runs.size(); ++i) runs[i] = r.runs[i];
    return 0;
  });
}

// InferenceSystem kept alive across runs so a caller can time steady-state
// runs the way bench() does, without rebuilding the pool per step.
struct ref_system {
  ClusterSpec cluster;
  std::unique_ptr<CpuMlpBackend> backend;
  std::unique_ptr<InferenceSystem> system;
  std::shared_ptr<const SampleStore> store;
};

int ref_system_create(const ref_cluster* c, const int* a, const ref_roster* roster,
                      ref_system** out) {
  return guarded([&] {
    auto sys = std::make_unique<ref_system>();
    sys->cluster = to_cluster(c);
    int D = sys->cluster.device_count(), M = sys->cluster.model_count();
    sys->backend = std::make_unique<CpuMlpBackend>(roster, M);
    sys->system = std::make_unique<InferenceSystem>(to_matrix(a, D, M), sys->cluster,
                                                    *sys->backend, CombinationRule::averaging());
    *out = sys.release();
    return 0;
  });
}

int ref_system_run(ref_system* sys, const float* X, std::size_t nb, std::size_t width,
                   float* Y, double* elapsed_s) {
  return guarded([&] {
    if (!sys->store || sys->store->nb_samples() != nb)
      sys->store = std::make_shared<SampleStore>(std::vector<float>(X, X + nb * width), nb, width);
    RunOutput out = sys->system->run(sys->store);
    if (Y) std::memcpy(Y, out.combined.data(), out.combined.size() * sizeof(float));
    *elapsed_s = out.stats.elapsed_s;
    return 0;
  });
}

void ref_system_destroy(ref_system* sys) {
  if (!sys) return;
  try {
    sys->system->shutdown();
  } catch (...) {
  }
  delete sys;
}

}  // extern "C"
