// Reference-side binding (see enserve_b200_backend.hpp), plus a small C entry
// the integration test drives through ctypes.
#include "enserve_b200_backend.hpp"

#include <cstring>
#include <stdexcept>

#include "enserve/opt/optimizer.hpp"
#include "enserve/runtime/pipeline.hpp"

namespace enserve {

namespace {

class B200Predictor final : public Predictor {
 public:
  B200Predictor(const WorkerContext& ctx, const es_model_desc& desc, int gpu)
      : ctx_(ctx), desc_(desc), gpu_(gpu) {}
  ~B200Predictor() override { es_member_destroy(handle_); }

  // Predictor::load (backend.hpp:29-30): false means out of memory.
  bool load() override {
    es_status s = es_member_create(gpu_, &desc_, ctx_.model.id, ctx_.batch, ctx_.device_load_mib,
                                   ctx_.device.memory_mib, &handle_);
    if (s == ES_ERR_STARTUP) return false;
    if (s != ES_OK) throw Error(std::string("b200 load: ") + es_last_error());
    return true;
  }

  // Predictor::predict (backend.hpp:32-33).
  void predict(const SampleView& in, std::span<float> out) override {
    es_status s = es_member_predict(handle_, in.features.data(), in.first_index, in.rows,
                                    in.width, out.data());
    if (s != ES_OK) throw Error(std::string("b200 predict: ") + es_last_error());
  }

 private:
  WorkerContext ctx_;
  es_model_desc desc_;
  int gpu_;
  es_member* handle_ = nullptr;
};

void fill_cluster(const ClusterSpec& c, const std::vector<es_model_desc>& members,
                  std::vector<es_device_desc>& devs, std::vector<es_model_desc>& mods,
                  es_cluster_desc& out) {
  devs.clear();
  mods.clear();
  for (const DeviceSpec& d : c.devices)
    devs.push_back({d.kind == DeviceKind::CPU ? 0 : 1, d.memory_mib, d.compute_rate,
                    d.batch_overhead_s});
  for (std::size_t m = 0; m < c.models.size(); ++m) {
    es_model_desc md = members.at(m);
    md.name = c.models[m].name.c_str();
    md.weight_mib = c.models[m].weight_mib;
    md.act_mib_per_sample = c.models[m].act_mib_per_sample;
    md.cost_per_sample = c.models[m].cost_per_sample;
    md.output_width = c.models[m].output_width;
    mods.push_back(md);
  }
  out = {devs.data(), static_cast<int>(devs.size()), mods.data(), static_cast<int>(mods.size()),
         c.batch_menu.data(), static_cast<int>(c.batch_menu.size()), c.segment_size};
}

}  // namespace

B200Backend::B200Backend(std::vector<es_model_desc> members) : members_(std::move(members)) {
  if (es_device_count(&gpus_) != ES_OK || gpus_ < 1)
    throw Error("b200 backend: no CUDA device");
}

std::unique_ptr<Predictor> B200Backend::make(const WorkerContext& ctx) const {
  return std::make_unique<B200Predictor>(ctx, members_.at(ctx.model.id), ctx.device.id % gpus_);
}

ScoreFn make_b200_score(const ClusterSpec& cluster, std::vector<es_model_desc> members,
                        std::shared_ptr<const SampleStore> calib, int repeats) {
  // The reference SampleStore keeps its data private; re-materialise rows once.
  std::vector<float> rows(calib->nb_samples() * calib->width());
  auto all = calib->rows(0, calib->nb_samples());
  std::memcpy(rows.data(), all.data(), rows.size() * sizeof(float));
  auto data = std::make_shared<std::vector<float>>(std::move(rows));
  es_store* store = nullptr;
  if (es_store_create(data->data(), calib->nb_samples(), calib->width(), 1, &store) != ES_OK)
    throw Error(std::string("b200 score: ") + es_last_error());
  std::shared_ptr<es_store> keep(store, es_store_destroy);
  return [cluster, members, keep, repeats](const AllocationMatrix& A) {
    std::vector<es_device_desc> devs;
    std::vector<es_model_desc> mods;
    es_cluster_desc c;
    fill_cluster(cluster, members, devs, mods, c);
    std::vector<int> cells(static_cast<std::size_t>(A.device_count()) * A.model_count());
    for (int d = 0; d < A.device_count(); ++d)
      for (int m = 0; m < A.model_count(); ++m) cells[d * A.model_count() + m] = A.at(d, m);
    es_bench_result r;
    if (es_bench(&c, cells.data(), keep.get(), repeats, nullptr, &r) != ES_OK)
      throw Error(std::string("b200 bench: ") + es_last_error());
    return r.throughput;
  };
}

}  // namespace enserve

// ---------------------------------------------------------------------------
// Test entries (ctypes): the reference's own run_inference and bounded_greedy
// with the b200 backend / score.  The cluster arrives as the es_cluster_desc
// of include/enserve_b200.h.
namespace {

enserve::ClusterSpec cluster_of(const es_cluster_desc* c) {
  using namespace enserve;
  ClusterSpec cluster;
  for (int d = 0; d < c->n_devices; ++d)
    cluster.devices.push_back({d, c->devices[d].kind == 0 ? DeviceKind::CPU : DeviceKind::GPU,
                               c->devices[d].memory_mib, c->devices[d].compute_rate,
                               c->devices[d].batch_overhead_s});
  for (int m = 0; m < c->n_models; ++m) {
    const es_model_desc& md = c->models[m];
    cluster.models.push_back({m, md.name ? md.name : "m", md.weight_mib, md.act_mib_per_sample,
                              md.cost_per_sample, md.output_width});
  }
  cluster.batch_menu.assign(c->batch_menu, c->batch_menu + c->menu_size);
  cluster.segment_size = c->segment_size;
  return cluster;
}

enserve::AllocationMatrix matrix_of(const int* cells, int D, int M) {
  enserve::AllocationMatrix A(D, M);
  for (int d = 0; d < D; ++d)
    for (int m = 0; m < M; ++m) A.set(d, m, cells[d * M + m]);
  return A;
}

}  // namespace

// run_inference (pipeline.cpp:418-444) through B200Backend; *elapsed_s (may be
// NULL) = the reference's own timing window (broadcast -> last fold).
extern "C" int ref_b200_run(const es_cluster_desc* c, const int* cells, int rule,
                            const float* X, std::size_t nb, std::size_t width, float* Y,
                            int* winners, double* elapsed_s) {
  using namespace enserve;
  try {
    ClusterSpec cluster = cluster_of(c);
    const AllocationMatrix A = matrix_of(cells, cluster.device_count(), cluster.model_count());
    B200Backend backend(std::vector<es_model_desc>(c->models, c->models + c->n_models));
    auto store = std::make_shared<SampleStore>(std::vector<float>(X, X + nb * width), nb, width);
    CombinationRule r = rule == 1 ? CombinationRule::majority_vote() : CombinationRule::averaging();
    InferenceResult out = run_inference(store, A, cluster, backend, r, Mode::Deploy);
    std::memcpy(Y, out.output->combined.data(), out.output->combined.size() * sizeof(float));
    if (winners && !out.output->winners.empty())
      std::memcpy(winners, out.output->winners.data(), out.output->winners.size() * sizeof(int));
    if (elapsed_s) *elapsed_s = out.output->stats.elapsed_s;
    return 0;
  } catch (const StartupError&) {
    return 3;
  } catch (const std::exception&) {
    return 1;
  }
}

// The reference's bounded_greedy (optimizer.cpp:178-227) scoring every matrix
// with make_b200_score (the device-timed bench behind the C ABI) over calib
// rows X[nb][width]: A_out[D*M], *final_score, *calls (bench calls).
extern "C" int ref_b200_greedy(const es_cluster_desc* c, const int* A0_cells, int max_iter,
                               int max_neighs, std::uint64_t seed, const float* X, std::size_t nb,
                               std::size_t width, int repeats, int* A_out, double* final_score,
                               int* calls) {
  using namespace enserve;
  try {
    ClusterSpec cluster = cluster_of(c);
    const int D = cluster.device_count(), M = cluster.model_count();
    auto calib = std::make_shared<SampleStore>(std::vector<float>(X, X + nb * width), nb, width);
    ScoreFn inner = make_b200_score(cluster, std::vector<es_model_desc>(c->models, c->models + M),
                                    calib, repeats);
    int n = 0;
    ScoreFn counted = [&](const AllocationMatrix& A) {
      ++n;
      return inner(A);
    };
    GreedyConfig cfg;
    cfg.max_iter = max_iter;
    cfg.max_neighs = max_neighs;
    cfg.rng_seed = seed;
    GreedyResult g = bounded_greedy(matrix_of(A0_cells, D, M), cluster, counted, cfg);
    for (int d = 0; d < D; ++d)
      for (int m = 0; m < M; ++m) A_out[d * M + m] = g.matrix.at(d, m);
    *final_score = g.trace.final_score;
    *calls = n;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}
