// The C ABI (include/enserve_b200.h) over the enserve-b200 C++ host core and
// GPU runtime.  Exceptions never cross the boundary: each one maps to the
// es_status of its reference error class, with the message kept per thread.
#include "enserve_b200.h"

#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "enserve/host_convert.hpp"
#include "enserve/spec_io.hpp"
#include "enserve/commands.hpp"
#include "enserve/calibrate.hpp"
#include "enserve/collective.hpp"
#include "enserve/service.hpp"
#include "cuda/batching.cuh"
#include "enserve/placement.hpp"
#include "enserve/rng.hpp"
#include "enserve/runtime.hpp"
#include "enserve/search.hpp"

using namespace enserve;

struct es_store {
  std::shared_ptr<SampleStore> store;
};

struct es_system {
  std::unique_ptr<InferenceSystem> sys;
  int models = 0;
};

struct es_comm {
  std::shared_ptr<enserve::Comm> comm;
};

struct es_member {
  std::unique_ptr<B200Predictor> predictor;
};

struct es_service {
  std::unique_ptr<enserve::PredictionService> svc;
  int C = 0;
};

struct es_request {
  std::future<enserve::RunOutput> fut;
  std::size_t rows = 0;
};

// A parsed spec document: the ClusterSpec plus the C views es_spec_describe
// hands out (valid while the handle lives).
struct es_spec {
  enserve::ClusterSpec cluster;
  std::vector<es_device_desc> devices;
  std::vector<es_model_desc> models;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
es_status guard(F&& body) {
  try {
    return body();
  } catch (const AllocationError& e) {
    g_last_error = e.what();
    return ES_ERR_ALLOCATION;
  } catch (const StartupError& e) {
    g_last_error = e.what();
    return ES_ERR_STARTUP;
  } catch (const SpecError& e) {
    g_last_error = e.what();
    return ES_ERR_SPEC;
  } catch (const BaselineError& e) {
    g_last_error = e.what();
    return ES_ERR_BASELINE;
  } catch (const CapExceededError& e) {
    g_last_error = e.what();
    return ES_ERR_CAP_EXCEEDED;
  } catch (const ProtocolError& e) {
    g_last_error = e.what();
    return ES_ERR_PROTOCOL;
  } catch (const NotReadyError& e) {
    g_last_error = e.what();
    return ES_ERR_NOT_READY;
  } catch (const DeviceError& e) {
    g_last_error = e.what();
    return ES_ERR_CUDA;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return ES_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return ES_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ES_ERR_INTERNAL;
  } catch (...) {
    g_last_error = "unknown exception";
    return ES_ERR_INTERNAL;
  }
}

void need(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}

ModelSpec to_model(const es_model_desc& d, int id) {
  ModelSpec m;
  m.id = id;
  m.name = d.name ? d.name : "m" + std::to_string(id);
  m.weight_mib = d.weight_mib;
  m.act_mib_per_sample = d.act_mib_per_sample;
  m.cost_per_sample = d.cost_per_sample;
  m.output_width = d.output_width;
  m.b200_cost_s = d.b200_cost_s;
  m.b200_overhead_s = d.b200_overhead_s;
  if (d.arch == 1) {
    need(d.n_widths >= 2 && d.n_widths <= ES_MAX_WIDTHS, "MLP needs 2..9 widths");
    m.arch.kind = MemberArch::Kind::MLP;
    m.arch.widths.assign(d.widths, d.widths + d.n_widths);
    m.arch.weight_seed = d.weight_seed;
  } else if (d.arch == 2) {
    need(d.n_widths == 6, "CNN needs widths {S, P, c1, c2, hidden, classes}");
    m.arch.kind = MemberArch::Kind::CNN;
    m.arch.widths.assign(d.widths, d.widths + d.n_widths);
    m.arch.weight_seed = d.weight_seed;
  } else {
    m.arch.kind = MemberArch::Kind::Synthetic;
  }
  return m;
}

ClusterSpec to_cluster(const es_cluster_desc* c) {
  need(c != nullptr, "cluster descriptor is NULL");
  ClusterSpec s;
  for (int d = 0; d < c->n_devices; ++d) {
    const es_device_desc& x = c->devices[d];
    s.devices.push_back({d, x.kind == 0 ? DeviceKind::CPU : DeviceKind::GPU, x.memory_mib,
                         x.compute_rate, x.batch_overhead_s});
  }
  for (int m = 0; m < c->n_models; ++m) s.models.push_back(to_model(c->models[m], m));
  if (c->menu_size > 0) s.batch_menu.assign(c->batch_menu, c->batch_menu + c->menu_size);
  s.segment_size = c->segment_size;
  return s;
}

AllocationMatrix to_matrix(const int* A, int D, int M) {
  need(A != nullptr || D * M == 0, "matrix is NULL");
  AllocationMatrix out(D, M);
  for (int d = 0; d < D; ++d)
    for (int m = 0; m < M; ++m) out.set(d, m, A[d * M + m]);
  return out;
}

void write_matrix(const AllocationMatrix& A, int* out) {
  std::memcpy(out, A.cells().data(), A.cells().size() * sizeof(int));
}

CombinationRule to_rule(const es_rule_desc* r, int M) {
  if (!r) return CombinationRule::averaging();
  const bool sm = r->member_softmax != 0;
  switch (r->kind) {
    case 1: return CombinationRule::majority_vote(sm);
    case 2:
      need(r->weights != nullptr, "weighted averaging needs weights");
      return CombinationRule::weighted(std::vector<double>(r->weights, r->weights + M), sm);
    default: return CombinationRule::averaging(sm);
  }
}

PoolOptions to_opts(const es_pool_opts* o) {
  PoolOptions p;
  if (!o) return p;
  if (o->device_map && o->n_device_map > 0)
    p.device_map.assign(o->device_map, o->device_map + o->n_device_map);
  p.copy_outputs = o->copy_outputs != 0;
  p.warmup = o->warmup != 0;
  p.sms_per_worker = o->sms_per_worker;
  p.overlap_colocated = o->overlap_colocated != 0;
  if (o->e2e_chunk_rows > 0) p.e2e_chunk_rows = o->e2e_chunk_rows;
  p.e2e_host_convert = o->e2e_host_convert != 0;
  if (o->e2e_convert_eighths > 0) p.e2e_convert_eighths = o->e2e_convert_eighths;
  p.dp_equal_split = o->dp_equal_split != 0;
  p.row_partials = o->row_partials != 0;
  p.peer_stores = o->no_peer_stores == 0;
  p.row_nodes = o->row_nodes != 0;
  p.dp_claim = o->dp_claim < 0 ? PoolOptions::kClaimOff
               : o->dp_claim > 0 ? PoolOptions::kClaimAlways : PoolOptions::kClaimAuto;
  p.claim_chunk = o->claim_chunk;
  p.pack_batches = o->pack_batches != 0;
  p.fp32 = o->fp32 != 0;
  return p;
}

ScoreFn make_score(const ClusterSpec& cluster, const es_bench_cfg* cfg) {
  const int mode = cfg ? cfg->mode : ES_BENCH_ANALYTIC;
  if (mode == ES_BENCH_ANALYTIC)
    return [&cluster](const AllocationMatrix& A) { return predict_ensemble_throughput(A, cluster); };
  if (mode == ES_BENCH_CALLBACK) {
    need(cfg->fn != nullptr, "callback bench needs fn");
    return [cfg](const AllocationMatrix& A) {
      return cfg->fn(A.cells().data(), A.device_count(), A.model_count(), cfg->user);
    };
  }
  if (mode == ES_BENCH_CALIBRATED) {
    const std::vector<int> row_gpu = to_opts(cfg->opts).device_map;
    return [&cluster, row_gpu](const AllocationMatrix& A) {
      return calibrated_throughput(A, cluster, row_gpu);
    };
  }
  need(cfg->calib != nullptr, "device bench needs a calibration store");
  PoolOptions opts = to_opts(cfg->opts);
  std::shared_ptr<const SampleStore> calib = cfg->calib->store;
  const int repeats = cfg->repeats > 0 ? cfg->repeats : 1;
  return [&cluster, calib, repeats, opts](const AllocationMatrix& A) {
    return bench(A, calib, cluster, repeats, opts).throughput;
  };
}

void export_trace(const GreedyResult& r, int calls, es_greedy_trace* trace) {
  if (!trace) return;
  trace->start_score = r.trace.start_score;
  trace->final_score = r.trace.final_score;
  trace->stop_reason = r.trace.stop_reason == StopReason::local_optimum ? 0 : 1;
  trace->n_iters = static_cast<int>(r.trace.iterations.size());
  trace->bench_calls = calls;
  for (int i = 0; i < trace->n_iters && i < trace->iter_cap; ++i) {
    const GreedyIteration& it = r.trace.iterations[i];
    if (trace->iter_neighbors) trace->iter_neighbors[i] = it.neighbors_evaluated;
    if (trace->iter_best) trace->iter_best[i] = it.best_score;
    if (trace->iter_accepted) trace->iter_accepted[i] = it.accepted ? 1 : 0;
  }
}

}  // namespace

extern "C" {

int es_abi_version(void) { return ES_ABI_VERSION; }

const char* es_status_name(es_status s) {
  switch (s) {
    case ES_OK: return "ES_OK";
    case ES_ERR_INVALID_ARGUMENT: return "ES_ERR_INVALID_ARGUMENT";
    case ES_ERR_SPEC: return "ES_ERR_SPEC";
    case ES_ERR_ALLOCATION: return "ES_ERR_ALLOCATION";
    case ES_ERR_STARTUP: return "ES_ERR_STARTUP";
    case ES_ERR_BASELINE: return "ES_ERR_BASELINE";
    case ES_ERR_CAP_EXCEEDED: return "ES_ERR_CAP_EXCEEDED";
    case ES_ERR_PROTOCOL: return "ES_ERR_PROTOCOL";
    case ES_ERR_CUDA: return "ES_ERR_CUDA";
    case ES_ERR_INTERNAL: return "ES_ERR_INTERNAL";
    case ES_ERR_BUFFER: return "ES_ERR_BUFFER";
  }
  return "ES_ERR_UNKNOWN";
}

const char* es_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------ host core
es_status es_cluster_validate(const es_cluster_desc* c, char* warnings, size_t len) {
  return guard([&] {
    std::vector<std::string> w;
    to_cluster(c).validate(&w);
    std::string all;
    for (const std::string& s : w) all += s + "\n";
    if (warnings && len) std::snprintf(warnings, len, "%s", all.c_str());
    return ES_OK;
  });
}

es_status es_matrix_validate(const es_cluster_desc* c, const int* A, int* ok, int* violations,
                             int cap, int* n) {
  return guard([&] {
    ClusterSpec s = to_cluster(c);
    MatrixValidation v = validate_matrix(to_matrix(A, c->n_devices, c->n_models), s);
    *ok = v.ok ? 1 : 0;
    if (n) *n = static_cast<int>(v.violations.size());
    for (int i = 0; violations && i < static_cast<int>(v.violations.size()) && i < cap; ++i) {
      const MatrixViolation& x = v.violations[i];
      violations[4 * i + 0] = x.kind == MatrixViolation::Kind::EmptyColumn ? 1 : 0;
      violations[4 * i + 1] = x.device;
      violations[4 * i + 2] = x.model;
      violations[4 * i + 3] = x.value;
    }
    return ES_OK;
  });
}

es_status es_num_segments(size_t nb, int segment_size, size_t* out) {
  return guard([&] {
    *out = num_segments(nb, segment_size);
    return ES_OK;
  });
}

es_status es_segment_bounds(int segment_id, int segment_size, size_t nb, size_t* start,
                            size_t* end) {
  return guard([&] {
    Segment s = segment_bounds(segment_id, segment_size, nb);
    *start = s.start;
    *end = s.end;
    return ES_OK;
  });
}

es_status es_segment_shares(const int* A, int devices, int models, size_t nb, int segment_size,
                            long long* out, int cap, int* n) {
  return guard([&] {
    std::vector<SegmentShare> s = segment_shares(to_matrix(A, devices, models), nb, segment_size);
    *n = static_cast<int>(s.size());
    for (int i = 0; out && i < *n && i < cap; ++i) {
      out[4 * i + 0] = s[i].device;
      out[4 * i + 1] = s[i].model;
      out[4 * i + 2] = s[i].begin;
      out[4 * i + 3] = s[i].end;
    }
    return ES_OK;
  });
}

es_status es_batch_rows(size_t nb, int segment_size, long long seg_begin, long long seg_end,
                        int batch, long long* row0, int* rows, int cap, int* n) {
  return guard([&] {
    need(n != nullptr && segment_size > 0 && batch > 0 && seg_begin >= 0 && seg_end >= seg_begin,
         "invalid batching arguments");
    const long long S = static_cast<long long>(num_segments(nb, segment_size));
    need(seg_end <= S, "segment range past the store");
    const es::BatchTiles ts =
        es::batch_tiles(seg_begin, seg_end, segment_size, static_cast<long long>(nb), batch);
    *n = static_cast<int>(ts.total);
    for (long long t = 0; t < ts.total && t < cap; ++t) {
      int r = 0;
      const long long r0 =
          es::batch_tile(ts, t, seg_begin, segment_size, static_cast<long long>(nb), batch, &r);
      if (row0) row0[t] = r0;
      if (rows) rows[t] = r;
    }
    return ES_OK;
  });
}

es_status es_segment_shares_weighted(const int* A, int devices, int models, size_t nb,
                                     int segment_size, const double* weight, long long* out,
                                     int cap, int* n) {
  return guard([&] {
    need(weight != nullptr, "NULL weights");
    const AllocationMatrix M = to_matrix(A, devices, models);
    std::vector<double> w(weight, weight + M.worker_count());
    std::vector<SegmentShare> s = segment_shares_weighted(M, nb, segment_size, w);
    *n = static_cast<int>(s.size());
    for (int i = 0; out && i < *n && i < cap; ++i) {
      out[4 * i + 0] = s[i].device;
      out[4 * i + 1] = s[i].model;
      out[4 * i + 2] = s[i].begin;
      out[4 * i + 3] = s[i].end;
    }
    return ES_OK;
  });
}

es_status es_fit_mem(const es_cluster_desc* c, const int* A, double* used_mib, int* fits) {
  return guard([&] {
    MemoryReport r = fit_mem(to_matrix(A, c->n_devices, c->n_models), to_cluster(c));
    for (std::size_t d = 0; used_mib && d < r.per_device.size(); ++d) used_mib[d] = r.per_device[d].used_mib;
    *fits = r.fits ? 1 : 0;
    return ES_OK;
  });
}

es_status es_more_remaining_memory(const es_cluster_desc* c, const int* A, int kind, int* device) {
  return guard([&] {
    ClusterSpec s = to_cluster(c);
    std::optional<int> d = more_remaining_memory(to_matrix(A, c->n_devices, c->n_models), 0,
                                                 kind == 0 ? DeviceKind::CPU : DeviceKind::GPU, s);
    *device = d.value_or(-1);
    return ES_OK;
  });
}

es_status es_predict_ensemble_throughput(const es_cluster_desc* c, const int* A, double* out) {
  return guard([&] {
    *out = predict_ensemble_throughput(to_matrix(A, c->n_devices, c->n_models), to_cluster(c));
    return ES_OK;
  });
}

es_status es_worst_fit_decreasing(const es_cluster_desc* c, int default_batch, int* A_out) {
  return guard([&] {
    write_matrix(worst_fit_decreasing(to_cluster(c), default_batch), A_out);
    return ES_OK;
  });
}

es_status es_neighborhood(const es_cluster_desc* c, const int* A, int* out, int cap, int* count) {
  return guard([&] {
    std::vector<AllocationMatrix> n =
        neighborhood(to_matrix(A, c->n_devices, c->n_models), to_cluster(c));
    *count = static_cast<int>(n.size());
    const int cells = c->n_devices * c->n_models;
    for (int i = 0; out && i < *count && i < cap; ++i) write_matrix(n[i], out + i * cells);
    return ES_OK;
  });
}

es_status es_neighborhood_stats(const es_cluster_desc* c, const int* A, size_t* size,
                                size_t* forbidden) {
  return guard([&] {
    NeighborhoodStats s =
        enumerated_neighborhood_stats(to_matrix(A, c->n_devices, c->n_models), to_cluster(c));
    *size = s.size;
    *forbidden = s.forbidden;
    return ES_OK;
  });
}

es_status es_count_total_matrices(int menu_size, int devices, int models, char* buf, size_t len) {
  return guard([&] {
    std::string s = count_total_matrices(menu_size, devices, models).str();
    if (s.size() + 1 > len) return ES_ERR_BUFFER;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return ES_OK;
  });
}

es_status es_count_total_neighs(int menu_size, int devices, int models, long long forbidden,
                                long long* out) {
  return guard([&] {
    *out = count_total_neighs(menu_size, devices, models, forbidden);
    return ES_OK;
  });
}

es_status es_effective_max_iter(int devices, int models, int max_iter, int* out) {
  return guard([&] {
    *out = effective_max_iter(devices, models, max_iter);
    return ES_OK;
  });
}

es_status es_enumerate_matrices(const es_cluster_desc* c, const char* cap, int* out,
                                size_t out_cap, size_t* count) {
  return guard([&] {
    ClusterSpec s = to_cluster(c);
    const std::size_t cells = static_cast<std::size_t>(c->n_devices) * c->n_models;
    std::size_t i = 0;
    for_each_matrix(s, BigUInt::parse(cap ? cap : "0"), [&](const AllocationMatrix& A) {
      if (out && i < out_cap) write_matrix(A, out + i * cells);
      ++i;
    });
    *count = i;
    return ES_OK;
  });
}

es_status es_sample_indices(uint64_t seed, size_t n, size_t k, size_t* out) {
  return guard([&] {
    std::mt19937_64 gen(seed);
    std::vector<std::size_t> v = sample_indices(gen, n, k);
    std::memcpy(out, v.data(), v.size() * sizeof(std::size_t));
    return ES_OK;
  });
}

es_status es_bounded_greedy(const es_cluster_desc* c, const int* A0, int max_iter, int max_neighs,
                            uint64_t seed, const es_bench_cfg* bcfg, int* A_out,
                            es_greedy_trace* trace) {
  return guard([&] {
    ClusterSpec s = to_cluster(c);
    int calls = 0;
    ScoreFn inner = make_score(s, bcfg);
    ScoreFn counted = [&](const AllocationMatrix& A) {
      ++calls;
      return inner(A);
    };
    GreedyResult r = bounded_greedy(to_matrix(A0, c->n_devices, c->n_models), s, counted,
                                    {max_iter, max_neighs, seed});
    write_matrix(r.matrix, A_out);
    export_trace(r, calls, trace);
    return ES_OK;
  });
}

es_status es_screened_greedy(const es_cluster_desc* c, const int* A0, int max_iter,
                             int max_neighs, uint64_t seed, int top_k, const es_bench_cfg* bcfg,
                             const es_bench_cfg* scfg, int* A_out, es_greedy_trace* trace) {
  return guard([&] {
    ClusterSpec s = to_cluster(c);
    int calls = 0;
    ScoreFn inner = make_score(s, bcfg);
    ScoreFn counted = [&](const AllocationMatrix& A) {
      ++calls;
      return inner(A);
    };
    ScoreFn screen = make_score(s, scfg);
    GreedyResult r = screened_greedy(to_matrix(A0, c->n_devices, c->n_models), s, counted, screen,
                                     {max_iter, max_neighs, seed}, top_k);
    write_matrix(r.matrix, A_out);
    export_trace(r, calls, trace);
    return ES_OK;
  });
}

es_status es_bbs_baseline(const es_cluster_desc* c, const es_bench_cfg* bcfg, int* A_out,
                          int* chosen, int* calls) {
  return guard([&] {
    ClusterSpec s = to_cluster(c);
    ClusterScoreFn fn;
    const int mode = bcfg ? bcfg->mode : ES_BENCH_ANALYTIC;
    if (mode == ES_BENCH_ANALYTIC) {
      fn = [](const AllocationMatrix& A, const ClusterSpec& cl) {
        return predict_ensemble_throughput(A, cl);
      };
    } else if (mode == ES_BENCH_CALLBACK) {
      need(bcfg->fn != nullptr, "callback bench needs fn");
      fn = [bcfg](const AllocationMatrix& A, const ClusterSpec&) {
        return bcfg->fn(A.cells().data(), A.device_count(), A.model_count(), bcfg->user);
      };
    } else {
      need(bcfg->calib != nullptr, "device bench needs a calibration store");
      PoolOptions opts = to_opts(bcfg->opts);
      auto calib = bcfg->calib->store;
      const int repeats = bcfg->repeats > 0 ? bcfg->repeats : 1;
      fn = [calib, repeats, opts](const AllocationMatrix& A, const ClusterSpec& cl) {
        return bench(A, calib, cl, repeats, opts).throughput;
      };
    }
    BaselineResult r = bbs_baseline(s, fn);
    write_matrix(r.matrix, A_out);
    for (std::size_t m = 0; chosen && m < r.chosen_batches.size(); ++m) chosen[m] = r.chosen_batches[m];
    *calls = r.bench_calls;
    return ES_OK;
  });
}

// ------------------------------------------------------------ device runtime
es_status es_device_count(int* n) {
  return guard([&] {
    *n = 0;
    if (cudaGetDeviceCount(n) != cudaSuccess) {
      cudaGetLastError();
      *n = 0;
    }
    return ES_OK;
  });
}

es_status es_store_create(const float* X, size_t nb, size_t width, int copy, es_store** out) {
  return guard([&] {
    need(X != nullptr || nb * width == 0, "features are NULL");
    auto h = std::make_unique<es_store>();
    if (copy)
      h->store = std::make_shared<SampleStore>(std::vector<float>(X, X + nb * width), nb, width);
    else
      h->store = SampleStore::borrow(X, nb, width);
    *out = h.release();
    return ES_OK;
  });
}

es_status es_store_synthetic(uint64_t seed, size_t nb, size_t width, int device, es_store** out) {
  return guard([&] {
    auto h = std::make_unique<es_store>();
    h->store = SampleStore::synthetic(seed, nb, width, device);
    *out = h.release();
    return ES_OK;
  });
}

void es_store_destroy(es_store* s) { delete s; }

es_status es_system_create(const es_cluster_desc* c, const int* A, const es_rule_desc* rule,
                           const es_pool_opts* opts, es_system** out) {
  return guard([&] {
    ClusterSpec s = to_cluster(c);
    auto h = std::make_unique<es_system>();
    h->models = c->n_models;
    h->sys = std::make_unique<InferenceSystem>(to_matrix(A, c->n_devices, c->n_models), s,
                                               to_rule(rule, c->n_models), to_opts(opts));
    *out = h.release();
    return ES_OK;
  });
}

es_status es_system_begin_run(es_system* s, es_store* X, const es_rule_desc* rule) {
  return guard([&] {
    need(s && X, "NULL handle");
    if (rule)
      s->sys->begin_run(X->store, to_rule(rule, s->models));
    else
      s->sys->begin_run(X->store);
    return ES_OK;
  });
}

es_status es_system_broadcast(es_system* s, size_t* segments) {
  return guard([&] {
    need(s != nullptr, "NULL handle");
    std::size_t n = s->sys->broadcast();
    if (segments) *segments = n;
    return ES_OK;
  });
}

namespace {
void export_run(const RunOutput& out, float* Y, int32_t* winners, es_run_stats* stats) {
  if (Y && !out.combined.empty()) std::memcpy(Y, out.combined.data(), out.combined.size() * sizeof(float));
  if (winners && !out.winners.empty())
    std::memcpy(winners, out.winners.data(), out.winners.size() * sizeof(int32_t));
  if (stats) {
    stats->nb_samples = out.stats.nb_samples;
    stats->segments = out.stats.segments;
    stats->data_messages = out.stats.data_messages;
    stats->elapsed_s = out.stats.elapsed_s;
  }
}
}  // namespace

es_status es_system_await_run(es_system* s, float* Y, int32_t* winners, es_run_stats* stats) {
  return guard([&] {
    need(s != nullptr, "NULL handle");
    export_run(s->sys->await_run(), Y, winners, stats);
    return ES_OK;
  });
}

es_status es_system_run(es_system* s, es_store* X, float* Y, int32_t* winners,
                        es_run_stats* stats) {
  return guard([&] {
    need(s && X, "NULL handle");
    export_run(s->sys->run(X->store), Y, winners, stats);
    return ES_OK;
  });
}

es_status es_system_run_host(es_system* s, const float* X, size_t nb, size_t width, float* Y,
                             int32_t* labels, double* elapsed_s) {
  return guard([&] {
    need(s && X, "NULL handle");
    double t = s->sys->run_host(X, nb, width, Y, labels);
    if (elapsed_s) *elapsed_s = t;
    return ES_OK;
  });
}

es_status es_host_convert_bf16(const float* x, uint16_t* y, size_t n) {
  return guard([&] {
    static ThreadPool pool(0);
    convert_f32_to_bf16_host(x, y, n, pool);
    return ES_OK;
  });
}

es_status es_system_info(es_system* s, int* workers, int* workers_per_model, int* launches,
                         int* combine_device) {
  return guard([&] {
    need(s != nullptr, "NULL handle");
    if (workers) *workers = s->sys->worker_count();
    if (workers_per_model) {
      std::vector<int> w = s->sys->workers_per_model();
      std::memcpy(workers_per_model, w.data(), w.size() * sizeof(int));
    }
    if (launches) *launches = s->sys->launches_last_run();
    if (combine_device) *combine_device = s->sys->combine_device();
    return ES_OK;
  });
}

es_status es_system_shares(es_system* s, int64_t* shares, double* rates) {
  return guard([&] {
    need(s != nullptr, "NULL handle");
    const auto sh = s->sys->last_shares();
    const auto& r = s->sys->worker_rates();
    for (std::size_t w = 0; w < sh.size(); ++w) {
      if (shares) {
        shares[2 * w] = sh[w].first;
        shares[2 * w + 1] = sh[w].second;
      }
      if (rates) rates[w] = r.empty() ? 1.0 : r[w];
    }
    return ES_OK;
  });
}

es_status es_system_timing(es_system* s, double* member_ms, double* combine_ms) {
  return guard([&] {
    need(s != nullptr, "NULL handle");
    for (int w = 0; member_ms && w < s->sys->worker_count(); ++w) member_ms[w] = s->sys->last_member_ms(w);
    if (combine_ms) *combine_ms = s->sys->last_combine_ms();
    return ES_OK;
  });
}

es_status es_system_last_transfer(es_system* s, size_t* h2d_bytes, size_t* d2h_bytes) {
  return guard([&] {
    need(s != nullptr, "NULL handle");
    if (h2d_bytes) *h2d_bytes = s->sys->h2d_bytes_last();
    if (d2h_bytes) *d2h_bytes = s->sys->d2h_bytes_last();
    return ES_OK;
  });
}

es_status es_system_kernel_timing(es_system* s, int worker, double* ms, char* names,
                                  size_t names_len, int cap, int* count) {
  return guard([&] {
    need(s != nullptr, "NULL handle");
    need(worker >= 0 && worker < s->sys->worker_count(), "worker out of range");
    const std::vector<double> t = s->sys->last_kernel_ms(worker);
    const std::vector<std::string> n = s->sys->kernel_names(worker);
    if (count) *count = static_cast<int>(n.size());
    for (int i = 0; ms && i < cap && i < static_cast<int>(n.size()); ++i)
      ms[i] = i < static_cast<int>(t.size()) ? t[i] : -1.0;
    if (names && names_len) {
      std::string joined;
      for (std::size_t i = 0; i < n.size(); ++i) joined += (i ? ";" : "") + n[i];
      std::snprintf(names, names_len, "%s", joined.c_str());
    }
    return ES_OK;
  });
}

es_status es_system_routes(es_system* s, int* routes, int* peers, int cap, int* n_peers) {
  return guard([&] {
    need(s != nullptr, "NULL handle");
    const std::vector<int> r = s->sys->worker_routes();
    for (std::size_t w = 0; routes && w < r.size(); ++w) routes[w] = r[w];
    const std::vector<int>& p = s->sys->peer_devices();
    for (int i = 0; peers && i < cap && i < static_cast<int>(p.size()); ++i) peers[i] = p[i];
    if (n_peers) *n_peers = static_cast<int>(p.size());
    return ES_OK;
  });
}

es_status es_system_claims(es_system* s, int model, int* owner, size_t cap, size_t* n) {
  return guard([&] {
    need(s != nullptr && n != nullptr, "NULL argument");
    const auto all = s->sys->last_claims();
    need(model >= 0 && model < static_cast<int>(all.size()), "model out of range");
    const std::vector<int>& o = all[model];
    *n = o.size();
    if (owner) std::memcpy(owner, o.data(), std::min(cap, o.size()) * sizeof(int));
    return ES_OK;
  });
}

es_status es_system_claim_models(es_system* s, int* models, int cap, int* n) {
  return guard([&] {
    need(s != nullptr && n != nullptr, "NULL argument");
    const std::vector<int> m = s->sys->claim_models();
    *n = static_cast<int>(m.size());
    for (int i = 0; models && i < cap && i < *n; ++i) models[i] = m[i];
    return ES_OK;
  });
}

es_status es_comm_unique_id(uint8_t* id, size_t len) {
  return guard([&] {
    need(id != nullptr, "NULL id buffer");
    const std::string u = enserve::Comm::unique_id();
    need(len >= u.size(), "id buffer smaller than an NCCL unique id (128 bytes)");
    std::memcpy(id, u.data(), u.size());
    return ES_OK;
  });
}

es_status es_comm_create(const uint8_t* id, size_t len, int nranks, int rank, int device,
                         es_comm** out) {
  return guard([&] {
    need(id != nullptr && out != nullptr, "NULL argument");
    auto h = std::make_unique<es_comm>();
    h->comm = std::make_shared<enserve::Comm>(
        std::string(reinterpret_cast<const char*>(id), len), nranks, rank, device);
    *out = h.release();
    return ES_OK;
  });
}

es_status es_nccl_version(int* version) {
  return guard([&] {
    need(version != nullptr, "NULL argument");
    *version = enserve::Comm::version();
    return ES_OK;
  });
}

void es_comm_destroy(es_comm* c) { delete c; }

es_status es_system_set_gather(es_system* s, es_comm* comm, int root, const int64_t* first_rows,
                               const int64_t* rows, int nranks) {
  return guard([&] {
    need(s != nullptr, "NULL handle");
    if (!comm) {
      s->sys->set_gather(nullptr, 0, {}, {});
      return ES_OK;
    }
    need(first_rows && rows && nranks == comm->comm->size(), "gather plan needs one entry per rank");
    s->sys->set_gather(comm->comm, root, std::vector<long long>(first_rows, first_rows + nranks),
                       std::vector<long long>(rows, rows + nranks));
    return ES_OK;
  });
}

es_status es_system_shutdown(es_system* s) {
  return guard([&] {
    need(s != nullptr, "NULL handle");
    s->sys->shutdown();
    return ES_OK;
  });
}

void es_system_destroy(es_system* s) { delete s; }

es_status es_run_inference(const es_cluster_desc* c, const int* A, const es_rule_desc* rule,
                           es_store* X, const es_pool_opts* opts, float* Y, int32_t* winners,
                           es_run_stats* stats) {
  return guard([&] {
    need(X != nullptr, "no sample store");
    ClusterSpec s = to_cluster(c);
    InferenceResult r = run_inference(X->store, to_matrix(A, c->n_devices, c->n_models), s,
                                      to_rule(rule, c->n_models), Mode::Deploy, to_opts(opts));
    export_run(*r.output, Y, winners, stats);
    return ES_OK;
  });
}

es_status es_bench(const es_cluster_desc* c, const int* A, es_store* calib, int repeats,
                   const es_pool_opts* opts, es_bench_result* out) {
  return guard([&] {
    ClusterSpec s = to_cluster(c);
    BenchResult r = bench(to_matrix(A, c->n_devices, c->n_models), calib ? calib->store : nullptr,
                          s, repeats, to_opts(opts));
    out->throughput = r.throughput;
    out->elapsed_s = r.elapsed_s;
    out->nb_samples = r.nb_samples;
    out->n_runs = static_cast<int>(std::min<std::size_t>(r.runs.size(), 64));
    for (int i = 0; i < out->n_runs; ++i) out->runs[i] = r.runs[i];
    out->rsd = r.rsd;
    return ES_OK;
  });
}

// ------------------------------------------------------------ Predictor seam
es_status es_member_create(int device, const es_model_desc* model, int model_id, int batch,
                           double device_load_mib, double capacity_mib, es_member** out) {
  return guard([&] {
    need(model != nullptr, "model descriptor is NULL");
    auto h = std::make_unique<es_member>();
    h->predictor = std::make_unique<B200Predictor>(device, to_model(*model, model_id), batch,
                                                   device_load_mib, capacity_mib);
    if (!h->predictor->load()) throw StartupError("member load() reported out-of-memory");
    *out = h.release();
    return ES_OK;
  });
}

es_status es_member_predict(es_member* m, const float* features, size_t first_index, size_t rows,
                            size_t width, float* out) {
  return guard([&] {
    need(m != nullptr, "NULL handle");
    m->predictor->predict(features, first_index, rows, width, out);
    return ES_OK;
  });
}

void es_member_destroy(es_member* m) { delete m; }

es_status es_combine(const es_rule_desc* rule, int M, int C, size_t rows,
                     const float* const* blocks, float* Y, int32_t* winners) {
  return guard([&] {
    combine_blocks(to_rule(rule, M), M, C, rows, blocks, Y, winners);
    return ES_OK;
  });
}


// ------------------------------------------------------------ spec / matrix / cache documents
namespace {

es_status put_text(const std::string& text, char* buf, size_t len, size_t* needed) {
  if (needed) *needed = text.size() + 1;
  if (!buf) return ES_OK;
  if (len < text.size() + 1) {
    g_last_error = "buffer too small";
    return ES_ERR_BUFFER;
  }
  std::memcpy(buf, text.c_str(), text.size() + 1);
  return ES_OK;
}

es_spec* make_spec(ClusterSpec c) {
  auto* s = new es_spec();
  s->cluster = std::move(c);
  for (const DeviceSpec& d : s->cluster.devices)
    s->devices.push_back({d.kind == DeviceKind::CPU ? 0 : 1, d.memory_mib, d.compute_rate,
                          d.batch_overhead_s});
  for (const ModelSpec& m : s->cluster.models) {
    es_model_desc x{};
    x.name = m.name.c_str();
    x.weight_mib = m.weight_mib;
    x.act_mib_per_sample = m.act_mib_per_sample;
    x.cost_per_sample = m.cost_per_sample;
    x.output_width = m.output_width;
    x.arch = m.arch.kind == MemberArch::Kind::MLP ? 1 : m.arch.kind == MemberArch::Kind::CNN ? 2 : 0;
    x.n_widths = static_cast<int>(std::min<std::size_t>(m.arch.widths.size(), ES_MAX_WIDTHS));
    for (int i = 0; i < x.n_widths; ++i) x.widths[i] = m.arch.widths[i];
    x.weight_seed = m.arch.weight_seed;
    x.b200_cost_s = m.b200_cost_s;
    x.b200_overhead_s = m.b200_overhead_s;
    s->models.push_back(x);
  }
  return s;
}

OptimizerKey opt_key(int max_iter, int max_neighs, uint64_t seed, int default_batch,
                     const char* bench_mode, size_t calib_samples, int repeats) {
  OptimizerKey k;
  k.greedy.max_iter = max_iter;
  k.greedy.max_neighs = max_neighs;
  k.greedy.rng_seed = seed;
  k.default_batch = default_batch;
  k.bench_mode = bench_mode ? bench_mode : "";
  k.calib_samples = calib_samples;
  k.repeats = repeats;
  return k;
}

js::Value parse_text(const char* text, const char* what) {
  need(text != nullptr, what);
  try {
    return js::parse(text);
  } catch (const std::exception& e) {
    throw SpecError(e.what());
  }
}

}  // namespace

es_status es_cluster_to_json(const es_cluster_desc* c, int indent, int with_arch, char* buf,
                             size_t len, size_t* needed) {
  return guard([&] {
    return put_text(js::dump(cluster_to_json(to_cluster(c), with_arch != 0), indent), buf, len,
                    needed);
  });
}

es_status es_spec_from_json(const char* base_json, const char* overlay_json, es_spec** out) {
  return guard([&] {
    need(out != nullptr, "out is NULL");
    const js::Value base = parse_text(base_json, "spec text is NULL");
    const js::Value overlay = overlay_json ? parse_text(overlay_json, "") : js::Value();
    *out = make_spec(cluster_from_documents(base, overlay));
    return ES_OK;
  });
}

es_status es_spec_load(const char* path, const char* overlay_path, es_spec** out) {
  return guard([&] {
    need(path != nullptr && out != nullptr, "path or out is NULL");
    const js::Value base = load_json_file(path);
    const js::Value overlay = overlay_path ? load_json_file(overlay_path) : js::Value();
    *out = make_spec(cluster_from_documents(base, overlay));
    return ES_OK;
  });
}

es_status es_spec_describe(es_spec* s, es_cluster_desc* out) {
  return guard([&] {
    need(s != nullptr && out != nullptr, "NULL handle");
    out->devices = s->devices.data();
    out->n_devices = static_cast<int>(s->devices.size());
    out->models = s->models.data();
    out->n_models = static_cast<int>(s->models.size());
    out->batch_menu = s->cluster.batch_menu.data();
    out->menu_size = static_cast<int>(s->cluster.batch_menu.size());
    out->segment_size = s->cluster.segment_size;
    return ES_OK;
  });
}

void es_spec_destroy(es_spec* s) { delete s; }

es_status es_save_json_file(const char* path, const char* json_text) {
  return guard([&] {
    need(path != nullptr, "path is NULL");
    save_json_file(path, parse_text(json_text, "text is NULL"));
    return ES_OK;
  });
}

es_status es_matrix_to_json(const es_cluster_desc* c, const int* A, int indent, char* buf,
                            size_t len, size_t* needed) {
  return guard([&] {
    const ClusterSpec s = to_cluster(c);
    return put_text(js::dump(matrix_to_json(to_matrix(A, c->n_devices, c->n_models), s), indent),
                    buf, len, needed);
  });
}

es_status es_matrix_from_json(const es_cluster_desc* c, const char* json_text, int* A_out) {
  return guard([&] {
    need(A_out != nullptr, "A_out is NULL");
    write_matrix(matrix_from_json(parse_text(json_text, "text is NULL"), to_cluster(c)), A_out);
    return ES_OK;
  });
}

es_status es_digest_hex(const char* text, char out[17]) {
  return guard([&] {
    need(text != nullptr && out != nullptr, "NULL argument");
    std::memcpy(out, digest_hex(text).c_str(), 17);
    return ES_OK;
  });
}

es_status es_cache_key(const es_cluster_desc* c, int max_iter, int max_neighs, uint64_t rng_seed,
                       int default_batch, const char* bench_mode, size_t calib_samples,
                       int repeats, char out[17]) {
  return guard([&] {
    need(out != nullptr, "out is NULL");
    const std::string k = cache_key(to_cluster(c), opt_key(max_iter, max_neighs, rng_seed,
                                                           default_batch, bench_mode,
                                                           calib_samples, repeats));
    std::memcpy(out, k.c_str(), 17);
    return ES_OK;
  });
}

es_status es_cache_key_device(const es_cluster_desc* c, int max_iter, int max_neighs,
                              uint64_t rng_seed, int default_batch, const char* bench_mode,
                              size_t calib_samples, int repeats, const char* device,
                              char out[17]) {
  return guard([&] {
    need(out != nullptr, "out is NULL");
    OptimizerKey k = opt_key(max_iter, max_neighs, rng_seed, default_batch, bench_mode,
                             calib_samples, repeats);
    k.device = device ? device : "";
    const std::string d = cache_key(to_cluster(c), k);
    std::memcpy(out, d.c_str(), 17);
    return ES_OK;
  });
}

es_status es_device_identity(char* out, size_t len) {
  return guard([&] {
    need(out != nullptr && len > 0, "out is NULL");
    std::snprintf(out, len, "%s", enserve::device_identity().c_str());
    return ES_OK;
  });
}

es_status es_cache_lookup(const char* directory, const char* key, const es_cluster_desc* c,
                          int* A_out, double* score, int64_t* created_at, int* hit) {
  return guard([&] {
    need(directory != nullptr && key != nullptr && hit != nullptr, "NULL argument");
    MatrixCache cache(directory);
    auto e = cache.lookup(key, to_cluster(c));
    *hit = e ? 1 : 0;
    if (e) {
      if (A_out) write_matrix(e->matrix, A_out);
      if (score) *score = e->score;
      if (created_at) *created_at = e->created_at;
    }
    return ES_OK;
  });
}

es_status es_cache_store(const char* directory, const char* key, const es_cluster_desc* c,
                         const int* A, double score, int64_t created_at) {
  return guard([&] {
    need(directory != nullptr && key != nullptr, "NULL argument");
    MatrixCache cache(directory);
    MatrixCacheEntry e;
    e.key = key;
    e.matrix = to_matrix(A, c->n_devices, c->n_models);
    e.score = score;
    e.created_at = created_at;
    cache.store(e, to_cluster(c));
    return ES_OK;
  });
}


// ------------------------------------------------------------ operator commands
int es_cli_main(int argc, const char* const* argv) {
  try {
    std::vector<std::string> args;
    for (int i = 1; i < argc; ++i) args.emplace_back(argv[i] ? argv[i] : "");
    return cli_main(args);
  } catch (...) {
    return 1;
  }
}


// ------------------------------------------------------------ calibrated cost model
namespace {
void export_member_fit(const CostFit& f, int M, double* c, double* o, double* rms) {
  for (int m = 0; c && m < M; ++m) c[m] = f.member_cost_s[m];
  for (int m = 0; o && m < M; ++m) o[m] = f.member_overhead_s[m];
  if (rms) *rms = f.member_rms_rel_error;
}
}  // namespace

es_status es_fit_cost_model(const int* model, const int* batch, const double* throughput, int n,
                            int n_models, double* cost_out, double* overhead_out, double* rms_out,
                            double* member_cost_out, double* member_overhead_out,
                            double* member_rms_out) {
  return guard([&] {
    need(n >= 0 && n_models > 0 && cost_out != nullptr, "bad arguments");
    std::vector<CostSample> s;
    for (int i = 0; i < n; ++i) s.push_back({model[i], batch[i], throughput[i]});
    const CostFit f = fit_cost_model(s, n_models);
    for (int m = 0; m < n_models; ++m) cost_out[m] = f.cost_per_sample[m];
    if (overhead_out) *overhead_out = f.batch_overhead_s;
    if (rms_out) *rms_out = f.rms_rel_error;
    export_member_fit(f, n_models, member_cost_out, member_overhead_out, member_rms_out);
    return ES_OK;
  });
}

es_status es_calibrate_cost_model(const es_cluster_desc* c, int device, size_t calib_nb,
                                  int repeats, double* cost_out, double* overhead_out,
                                  double* rms_out, double* measured_out, double* member_cost_out,
                                  double* member_overhead_out, double* member_rms_out) {
  return guard([&] {
    need(cost_out != nullptr, "cost_out is NULL");
    const ClusterSpec s = to_cluster(c);
    std::vector<CostSample> meas;
    const CostFit f = calibrate_cost_model(s, device, calib_nb, repeats, &meas);
    for (int m = 0; m < s.model_count(); ++m) cost_out[m] = f.cost_per_sample[m];
    if (overhead_out) *overhead_out = f.batch_overhead_s;
    if (rms_out) *rms_out = f.rms_rel_error;
    if (measured_out)
      for (std::size_t i = 0; i < meas.size(); ++i) measured_out[i] = meas[i].throughput;
    export_member_fit(f, s.model_count(), member_cost_out, member_overhead_out, member_rms_out);
    return ES_OK;
  });
}

es_status es_calibrated_throughput(const es_cluster_desc* c, const int* A, const int* row_gpu,
                                   double* out) {
  return guard([&] {
    need(c != nullptr && out != nullptr, "NULL argument");
    std::vector<int> rg;
    if (row_gpu) rg.assign(row_gpu, row_gpu + c->n_devices);
    *out = calibrated_throughput(to_matrix(A, c->n_devices, c->n_models), to_cluster(c), rg);
    return ES_OK;
  });
}


// ------------------------------------------------------------ deploy-mode service
es_status es_service_create(const es_cluster_desc* c, const int* A, const es_rule_desc* rule,
                            const es_pool_opts* opts, int flush_timeout_ms, size_t input_width,
                            long long arena_rows, es_service** out) {
  return guard([&] {
    need(out != nullptr, "out is NULL");
    ClusterSpec cl = to_cluster(c);
    ServiceConfig cfg;
    cfg.flush_timeout_ms = flush_timeout_ms;
    cfg.input_width = input_width;
    cfg.rule = to_rule(rule, cl.model_count());
    cfg.pool = to_opts(opts);
    if (arena_rows >= 0) cfg.arena_rows = static_cast<std::size_t>(arena_rows);
    auto* s = new es_service();
    s->C = cl.models.empty() ? 0 : cl.models[0].output_width;
    try {
      s->svc = std::make_unique<PredictionService>(cl, to_matrix(A, c->n_devices, c->n_models), cfg);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
    return ES_OK;
  });
}

es_status es_service_wait_ready(es_service* s, int timeout_ms, int* ready, char* error, size_t len) {
  return guard([&] {
    need(s != nullptr && ready != nullptr, "NULL argument");
    *ready = s->svc->wait_ready(std::chrono::milliseconds(timeout_ms)) ? 1 : 0;
    if (error && len) std::snprintf(error, len, "%s", s->svc->startup_error().c_str());
    return ES_OK;
  });
}

es_status es_service_submit(es_service* s, const float* X, size_t rows, es_request** out) {
  return guard([&] {
    need(s != nullptr && out != nullptr && (X != nullptr || rows == 0), "NULL argument");
    auto* r = new es_request();
    r->rows = rows;
    r->fut = s->svc->submit(X, rows);
    *out = r;
    return ES_OK;
  });
}

es_status es_request_wait(es_request* r, float* Y, int32_t* winners) {
  return guard([&] {
    need(r != nullptr, "NULL handle");
    RunOutput out = r->fut.get();  // rethrows StartupError / Error
    if (Y) std::memcpy(Y, out.combined.data(), out.combined.size() * sizeof(float));
    if (winners)
      for (std::size_t i = 0; i < out.winners.size(); ++i) winners[i] = out.winners[i];
    return ES_OK;
  });
}

void es_request_destroy(es_request* r) { delete r; }

es_status es_service_stats(es_service* s, es_service_info* out) {
  return guard([&] {
    need(s != nullptr && out != nullptr, "NULL argument");
    const ServiceStats st = s->svc->stats();
    out->ready = st.ready ? 1 : 0;
    out->requests_served = st.requests_served;
    out->samples_served = st.samples_served;
    out->flushes = st.flushes;
    out->last_flush_throughput = st.last_flush_throughput;
    out->pending_requests = st.pending_requests;
    out->pending_samples = st.pending_samples;
    out->uptime_s = st.uptime_s;
    return ES_OK;
  });
}

void es_service_destroy(es_service* s) {
  if (!s) return;
  try {
    s->svc->stop();
  } catch (...) {
  }
  delete s;
}

}  // extern "C"
