// enserve-b200 runtime: device members, sample stores, the GPU InferenceSystem
// and bench().  See runtime.hpp for the mapping onto the reference pipeline.
#include "enserve/runtime.hpp"

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>

#include "../cuda/aux_kernels.cuh"
#include "../cuda/fp32_kernels.cuh"
#include "../cuda/mlp_kernel.cuh"
#include "enserve/collective.hpp"
#include "enserve/member.hpp"
#include "enserve/host_convert.hpp"
#include "enserve/placement.hpp"

#include <chrono>

namespace enserve {

namespace {

[[noreturn]] void throw_cuda(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear a sticky launch error so later calls report fresh state
  throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

#define ES_CUDA(call)                                  \
  do {                                                 \
    cudaError_t es_err_ = (call);                      \
    if (es_err_ != cudaSuccess) throw_cuda(es_err_, #call); \
  } while (0)

#define ES_LAUNCH(call)                                                       \
  do {                                                                        \
    if ((call) != 0) throw_cuda(cudaGetLastError(), "kernel launch " #call); \
  } while (0)

int visible_devices() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1)
    throw DeviceError("no CUDA device visible to the enserve-b200 runtime");
  return n;
}

// NVTX range over the host code that enqueues one worker's (or the combine's)
// work: a profiler shows each worker's segments next to its kernels.  No cost
// without an attached tool (nvtx3 is header-only, the injection is dlopen'd).
struct Nvtx {
  explicit Nvtx(const std::string& what) { nvtxRangePushA(what.c_str()); }
  ~Nvtx() { nvtxRangePop(); }
};

// RAII device selection.
struct OnDevice {
  int prev = 0;
  explicit OnDevice(int dev) {
    cudaGetDevice(&prev);
    ES_CUDA(cudaSetDevice(dev));
  }
  ~OnDevice() { cudaSetDevice(prev); }
};

// `from` may access `to`'s memory (idempotent: an already enabled pair is fine).
void enable_peer(int from, int to) {
  OnDevice on(from);
  const cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return;
  }
  ES_CUDA(e);
}

// K3 arguments for M per-model logit buffers of `rows` rows.
es::CombineArgs combine_args(const CombinationRule& rule, const std::vector<float*>& logits,
                             std::size_t rows, int C, float* y, int32_t* labels) {
  es::CombineArgs ca;
  ca.M = static_cast<int>(logits.size());
  ca.C = C;
  ca.rows = static_cast<long long>(rows);
  ca.y = y;
  ca.argmax = labels;
  ca.softmax = rule.member_softmax ? 1 : 0;
  ca.rule = rule.kind == CombinationRule::Kind::majority_vote        ? es::kVote
            : rule.kind == CombinationRule::Kind::weighted_averaging ? es::kWeighted
                                                                       : es::kAverage;
  const float inv = 1.0f / static_cast<float>(ca.M);  // combine.cpp:101
  for (int m = 0; m < ca.M; ++m) {
    ca.logits[m] = logits[m];
    ca.weight[m] = rule.kind == CombinationRule::Kind::weighted_averaging
                       ? static_cast<float>(rule.weights[m])
                       : inv;
  }
  return ca;
}

}  // namespace

// ---------------------------------------------------------------- rule
CombinationRule CombinationRule::weighted(std::vector<double> weights, bool softmax) {
  double total = 0.0;
  for (double w : weights) {
    if (w < 0) throw SpecError("combination weights must be nonnegative");
    total += w;
  }
  if (std::abs(total - 1.0) > 1e-9)
    throw SpecError("combination weights must sum to 1, got " + std::to_string(total));
  return {Kind::weighted_averaging, std::move(weights), softmax};
}

std::string CombinationRule::name() const {
  switch (kind) {
    case Kind::majority_vote: return "vote";
    case Kind::weighted_averaging: return "wavg";
    default: return "avg";
  }
}

CombinationRule CombinationRule::from_name(const std::string& name, int model_count) {
  if (name == "avg") return averaging();
  if (name == "vote") return majority_vote();
  if (name == "wavg") return weighted(std::vector<double>(model_count, 1.0 / model_count));
  throw SpecError("unknown combination rule '" + name + "'");
}

// ---------------------------------------------------------------- store
SampleStore::SampleStore(std::vector<float> data, std::size_t nb, std::size_t width)
    : owned_(std::move(data)), nb_(nb), width_(width) {
  if (owned_.size() != nb * width)
    throw SpecError("sample store size does not match nb_samples * width");
  host_ = owned_.data();
}

std::shared_ptr<SampleStore> SampleStore::borrow(const float* data, std::size_t nb,
                                                 std::size_t width) {
  std::shared_ptr<SampleStore> s(new SampleStore());
  s->host_ = data;
  s->nb_ = nb;
  s->width_ = width;
  return s;
}

std::shared_ptr<SampleStore> SampleStore::synthetic(std::uint64_t seed, std::size_t nb,
                                                    std::size_t width, int device) {
  std::shared_ptr<SampleStore> s(new SampleStore());
  s->nb_ = nb;
  s->width_ = width;
  s->synthetic_ = true;
  s->synthetic_seed_ = seed;
  s->device_replica(device);
  return s;
}

SampleStore::~SampleStore() {
  for (std::size_t d = 0; d < replicas_.size(); ++d)
    if (replicas_[d]) {
      cudaSetDevice(static_cast<int>(d));
      cudaFree(replicas_[d]);
    }
  for (std::size_t d = 0; d < replicas32_.size(); ++d)
    if (replicas32_[d]) {
      cudaSetDevice(static_cast<int>(d));
      cudaFree(replicas32_[d]);
    }
}

const float* SampleStore::device_replica_f32(int device) const {
  if (replicas32_.size() <= static_cast<std::size_t>(device)) replicas32_.resize(device + 1, nullptr);
  if (replicas32_[device]) return replicas32_[device];
  OnDevice on(device);
  const std::size_t n = nb_ * width_;
  float* x = nullptr;
  ES_CUDA(cudaMalloc(&x, std::max<std::size_t>(n, 1) * sizeof(float)));
  if (synthetic_)
    ES_LAUNCH(es::generate_features_f32(synthetic_seed_, n, x, 0));
  else if (n > 0)
    ES_CUDA(cudaMemcpy(x, host_, n * sizeof(float), cudaMemcpyHostToDevice));
  ES_CUDA(cudaDeviceSynchronize());
  replicas32_[device] = x;
  return x;
}

const void* SampleStore::device_replica(int device) const {
  if (replicas_.size() <= static_cast<std::size_t>(device)) replicas_.resize(device + 1, nullptr);
  if (replicas_[device]) return replicas_[device];
  OnDevice on(device);
  const std::size_t n = nb_ * width_;
  void* bf = nullptr;
  ES_CUDA(cudaMalloc(&bf, std::max<std::size_t>(n, 1) * sizeof(__nv_bfloat16)));
  if (synthetic_) {
    ES_LAUNCH(es::generate_features_bf16(synthetic_seed_, n, static_cast<__nv_bfloat16*>(bf), 0));
  } else if (n > 0) {
    // Stage through fp32 in bounded chunks, convert on device.
    const std::size_t chunk = std::min<std::size_t>(n, std::size_t(1) << 26);
    float* stage = nullptr;
    ES_CUDA(cudaMalloc(&stage, chunk * sizeof(float)));
    for (std::size_t off = 0; off < n; off += chunk) {
      const std::size_t len = std::min(chunk, n - off);
      ES_CUDA(cudaMemcpy(stage, host_ + off, len * sizeof(float), cudaMemcpyHostToDevice));
      ES_LAUNCH(es::convert_f32_to_bf16(stage, static_cast<__nv_bfloat16*>(bf) + off, len, 0));
    }
    ES_CUDA(cudaDeviceSynchronize());
    cudaFree(stage);
  }
  ES_CUDA(cudaDeviceSynchronize());
  replicas_[device] = bf;
  return bf;
}

// ---------------------------------------------------------------- system
struct InferenceSystem::Worker {
  int model = 0;
  int row = 0;   // cluster device id
  int phys = 0;  // CUDA ordinal
  int batch = 1;
  int colocated = 1;
  std::unique_ptr<DeviceMember> member;
  cudaStream_t stream = nullptr;
  bool owns_stream = true;
  cudaEvent_t ev_begin = nullptr, ev_done = nullptr;
  std::vector<cudaEvent_t> marks;  // one per member launch (DeviceMember::forward)
  long long seg_begin = 0, seg_end = 0;  // this run's share
  float* staging = nullptr;              // remote worker: local logits [nb][C]
  std::size_t staging_rows = 0;
  bool remote = false;  // on another node than the combining one
  bool peer = false;    // may access the combining GPU's memory (same GPU or peer access)
  es::ClaimedRun* claim = nullptr;  // device FIFO: this worker's claimed run (on its GPU)
  bool direct = false;  // remote, storing its logits straight into the combining GPU's buffers
  // Logits go to the worker's own staging buffer: a remote worker without
  // direct peer stores, or any remote worker in row_partials mode (its row's
  // partial fold runs on its own GPU).
  bool staged(bool partial_mode) const { return remote && (!direct || partial_mode); }
};

struct InferenceSystem::Impl {
  cudaStream_t main = nullptr;
  cudaEvent_t start = nullptr, combine_begin = nullptr, end = nullptr;
  std::vector<float*> logits;  // per model, on combine device
  float* y = nullptr;
  int32_t* labels = nullptr;
  std::size_t cap_rows = 0;
  // row_partials: per device row, its partial on its GPU and (remote rows)
  // the copy on the combining GPU; rows without workers stay empty.
  struct RowPartial {
    int phys = 0;
    float* local = nullptr;
    float* at_combine = nullptr;  // == local when phys is the combining GPU
    std::size_t rows = 0;
    cudaEvent_t done = nullptr;
  };
  std::vector<RowPartial> partials;
  bool partial_mode = false;
  // Device FIFO per data-parallel model (PoolOptions::dp_claim).
  struct Queue {
    bool on = false;
    unsigned long long* counter = nullptr;  // on the combining GPU
    int* owner = nullptr;                   // [segments] claiming worker (evidence)
    std::size_t owner_cap = 0;
    long long segments = 0, chunk = 1, rounds = 0;
  };
  std::vector<Queue> queues;
  // run_host pipeline (slots of whole-segment chunks).  A slot's host side
  // and combining-node buffers:
  struct Slot {
    void* pinned = nullptr;      // bf16 chunk staged by the host pool (portable)
    std::vector<float*> logits;  // per model, on the combining GPU
    float* y = nullptr;
    int32_t* labels = nullptr;
    cudaEvent_t combined = nullptr, d2h_done = nullptr;
  };
  // Every node hosting workers is a lane (lane 0 = the combining node): its
  // copy stream brings the rows its workers predict over its own PCIe link,
  // its compute stream runs them, remote logits reach the combining GPU by
  // direct peer stores or staging + peer copy.
  struct Lane {
    int phys = 0;
    cudaStream_t copy = nullptr, comp = nullptr;
    std::vector<int> workers;  // indices into workers_
    struct LSlot {
      float* x32 = nullptr;
      void* x16 = nullptr;
      std::vector<float*> staging;  // per model (staged workers only)
      cudaEvent_t h2d_done = nullptr, comp_done = nullptr;
      bool used = false;  // the lane had rows in the chunk last held by this slot
    } s[3];
  };
  Slot slots[3];
  std::vector<Lane> lanes;
  cudaStream_t d2h = nullptr;
  std::unique_ptr<ThreadPool> pool;
  std::size_t e2e_chunk_elems = 0;
  void free_e2e() {
    int prev = 0;
    cudaGetDevice(&prev);
    for (Slot& sl : slots) {
      if (sl.pinned) cudaFreeHost(sl.pinned);
      cudaSetDevice(lanes.empty() ? 0 : lanes[0].phys);
      for (float* p : sl.logits) cudaFree(p);
      cudaFree(sl.y);
      cudaFree(sl.labels);
      if (sl.combined) cudaEventDestroy(sl.combined);
      if (sl.d2h_done) cudaEventDestroy(sl.d2h_done);
      sl = Slot{};
    }
    for (std::size_t l = 0; l < lanes.size(); ++l) {
      Lane& ln = lanes[l];
      cudaSetDevice(ln.phys);
      if (ln.copy) cudaStreamSynchronize(ln.copy);
      if (ln.comp) cudaStreamSynchronize(ln.comp);
      for (Lane::LSlot& ls : ln.s) {
        cudaFree(ls.x32);
        cudaFree(ls.x16);
        for (float* p : ls.staging) cudaFree(p);
        if (ls.h2d_done) cudaEventDestroy(ls.h2d_done);
        if (ls.comp_done) cudaEventDestroy(ls.comp_done);
      }
      if (ln.copy) cudaStreamDestroy(ln.copy);
      if (l > 0 && ln.comp) cudaStreamDestroy(ln.comp);  // lane 0 computes on `main`
    }
    lanes.clear();
    if (d2h) cudaStreamDestroy(d2h);
    d2h = nullptr;
    e2e_chunk_elems = 0;
    cudaSetDevice(prev);
  }
  // NCCL prediction gather (set_gather).
  std::shared_ptr<Comm> comm;
  int root = 0;
  std::vector<long long> g_first, g_rows;
  float* gy = nullptr;
  int32_t* glabels = nullptr;
  std::size_t g_cap = 0;
  std::shared_ptr<const SampleStore> store;
  CombinationRule rule;
  std::size_t segments = 0;
};

InferenceSystem::InferenceSystem(const AllocationMatrix& A, const ClusterSpec& cluster,
                                 CombinationRule rule, PoolOptions options)
    : matrix_(A), cluster_(cluster), rule_(std::move(rule)), options_(std::move(options)),
      impl_(std::make_unique<Impl>()) {
  MatrixValidation verdict = validate_matrix(A, cluster);
  if (!verdict.ok) {
    std::string what = "allocation matrix is invalid:";
    for (const MatrixViolation& v : verdict.violations) what += " " + v.describe() + ";";
    throw SpecError(what);
  }
  output_width_ = cluster.models.front().output_width;
  for (const ModelSpec& m : cluster.models)
    if (m.output_width != output_width_) throw SpecError("ensemble models disagree on output width");
  if (output_width_ > es::kMaxClasses)
    throw SpecError("output width above " + std::to_string(es::kMaxClasses) + " classes");
  if (cluster.model_count() > es::kMaxMembers)
    throw SpecError("more than " + std::to_string(es::kMaxMembers) + " ensemble members");
  if (rule_.kind == CombinationRule::Kind::weighted_averaging &&
      rule_.weights.size() != static_cast<std::size_t>(cluster.model_count()))
    throw SpecError("weighted averaging needs one weight per model");

  const int gpus = visible_devices();
  auto phys_of = [&](int row) {
    if (!options_.device_map.empty()) {
      if (row >= static_cast<int>(options_.device_map.size()) || options_.device_map[row] >= gpus)
        throw SpecError("device_map has no valid CUDA ordinal for " + cluster.devices[row].label());
      return options_.device_map[row];
    }
    return row % gpus;
  };

  // One worker per nonzero cell, row-major (pipeline.cpp:106-124).
  bool oom = false;
  for (int d = 0; d < A.device_count() && !oom; ++d) {
    const double load = device_load(A, d, cluster_);
    for (int m = 0; m < A.model_count(); ++m) {
      const int b = A.at(d, m);
      if (b == 0) continue;
      auto w = std::make_unique<Worker>();
      w->model = m;
      w->row = d;
      w->phys = phys_of(d);
      w->batch = b;
      w->colocated = A.row_worker_count(d);
      // Predictor::load(): the declared footprint must fit (the reference
      // backend's rule, backend.cpp:41), and the real device must host it.
      w->member = std::make_unique<DeviceMember>();
      if (load > cluster_.devices[d].memory_mib ||
          !w->member->load(w->phys, cluster_.models[m],
                           options_.pack_batches ? std::max(b, cluster_.segment_size) : b,
                           options_.fp32)) {
        oom = true;
        break;
      }
      OnDevice on(w->phys);
      // Co-located workers time-share their GPU (cost_model.cpp:17): each
      // member kernel is a persistent full-device grid, so they queue on one
      // stream per GPU in worker order (unless asked to overlap).
      cudaStream_t shared = nullptr;
      if (!options_.overlap_colocated)
        for (const auto& o : workers_)
          if (o->phys == w->phys && (!options_.row_nodes || o->row == w->row)) shared = o->stream;
      if (shared) {
        w->stream = shared;
        w->owns_stream = false;
      } else {
        ES_CUDA(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking));
      }
      ES_CUDA(cudaEventCreate(&w->ev_begin));
      ES_CUDA(cudaEventCreate(&w->ev_done));
      w->marks.resize(w->member->max_launches());
      for (auto& e : w->marks) ES_CUDA(cudaEventCreate(&e));
      workers_.push_back(std::move(w));
    }
  }
  if (oom) {
    shutdown();
    throw StartupError("a worker reported out-of-memory during startup");
  }
  combine_dev_ = workers_.front()->phys;
  combine_row_ = workers_.front()->row;
  // Remote workers and NVLink peer access (both directions: the worker's GPU
  // stores into the combining GPU's buffers, the combining GPU's copies may
  // read a staging buffer).  Without peer access a remote worker stages.
  for (auto& w : workers_) {
    w->remote = w->phys != combine_dev_ || (options_.row_nodes && w->row != combine_row_);
    if (!w->remote) continue;
    bool peer = w->phys == combine_dev_;
    if (!peer) {
      if (std::find(peers_.begin(), peers_.end(), w->phys) == peers_.end()) {
        int fwd = 0, back = 0;
        ES_CUDA(cudaDeviceCanAccessPeer(&fwd, w->phys, combine_dev_));
        ES_CUDA(cudaDeviceCanAccessPeer(&back, combine_dev_, w->phys));
        if (fwd && back) {
          enable_peer(w->phys, combine_dev_);
          enable_peer(combine_dev_, w->phys);
          peers_.push_back(w->phys);
        }
      }
      peer = std::find(peers_.begin(), peers_.end(), w->phys) != peers_.end();
    }
    w->direct = peer && options_.peer_stores;
    w->peer = peer;
  }
  for (auto& w : workers_)
    if (!w->remote) w->peer = true;
  // Device FIFO: models with several workers that can all follow a claim and
  // store straight into the combining GPU's logits.
  impl_->queues.assign(cluster.model_count(), Impl::Queue{});
  if (options_.dp_claim != PoolOptions::kClaimOff) {
    const std::vector<int> per_model = workers_per_model();
    for (int m = 0; m < cluster.model_count(); ++m) {
      if (per_model[m] < 2) continue;
      bool ok = true;
      std::vector<int> gpus;
      for (const auto& w : workers_)
        if (w->model == m) {
          ok = ok && w->member->supports_claim() && w->peer && (!w->remote || w->direct);
          ok = ok && (options_.dp_claim == PoolOptions::kClaimAlways ||
                      std::find(gpus.begin(), gpus.end(), w->phys) == gpus.end());
          gpus.push_back(w->phys);
        }
      if (!ok) continue;
      Impl::Queue& q = impl_->queues[m];
      {
        OnDevice oc(combine_dev_);
        ES_CUDA(cudaMalloc(&q.counter, sizeof(unsigned long long)));
      }
      for (auto& w : workers_)
        if (w->model == m) {
          OnDevice ow(w->phys);
          ES_CUDA(cudaMalloc(&w->claim, sizeof(es::ClaimedRun)));
        }
      q.on = true;
    }
  }
  OnDevice on(combine_dev_);
  ES_CUDA(cudaStreamCreateWithFlags(&impl_->main, cudaStreamNonBlocking));
  ES_CUDA(cudaEventCreate(&impl_->start));
  ES_CUDA(cudaEventCreate(&impl_->combine_begin));
  ES_CUDA(cudaEventCreate(&impl_->end));
  impl_->logits.assign(cluster.model_count(), nullptr);
}

InferenceSystem::~InferenceSystem() {
  try {
    shutdown();
  } catch (...) {
  }
}

void InferenceSystem::shutdown() {
  if (shut_down_) return;
  shut_down_ = true;
  for (auto& w : workers_) {  // drain every stream before any is destroyed
    cudaSetDevice(w->phys);
    if (w->stream) cudaStreamSynchronize(w->stream);
  }
  for (auto& w : workers_) {
    cudaSetDevice(w->phys);
    if (w->staging) cudaFree(w->staging);
    if (w->claim) cudaFree(w->claim);
    if (w->stream && w->owns_stream) cudaStreamDestroy(w->stream);
    if (w->ev_begin) cudaEventDestroy(w->ev_begin);
    if (w->ev_done) cudaEventDestroy(w->ev_done);
    for (auto e : w->marks) cudaEventDestroy(e);
    w->member.reset();
  }
  if (impl_ && impl_->main) {
    cudaSetDevice(combine_dev_);
    cudaStreamSynchronize(impl_->main);
    for (float* p : impl_->logits) cudaFree(p);
    cudaFree(impl_->y);
    cudaFree(impl_->labels);
    cudaFree(impl_->gy);
    cudaFree(impl_->glabels);
    for (Impl::Queue& q : impl_->queues) {
      cudaFree(q.counter);
      cudaFree(q.owner);
    }
    impl_->queues.clear();
    impl_->comm.reset();
    impl_->free_e2e();
    for (Impl::RowPartial& p : impl_->partials) {
      if (p.at_combine != p.local) cudaFree(p.at_combine);
      cudaSetDevice(p.phys);
      cudaFree(p.local);
      if (p.done) cudaEventDestroy(p.done);
      cudaSetDevice(combine_dev_);
    }
    cudaEventDestroy(impl_->start);
    cudaEventDestroy(impl_->combine_begin);
    cudaEventDestroy(impl_->end);
    cudaStreamDestroy(impl_->main);
    impl_->main = nullptr;
  }
}

void InferenceSystem::assign_shares(std::size_t nb) {
  std::vector<SegmentShare> shares =
      rates_.empty() ? segment_shares(matrix_, nb, cluster_.segment_size)
                     : segment_shares_weighted(matrix_, nb, cluster_.segment_size, rates_);
  for (std::size_t i = 0; i < workers_.size(); ++i) {  // both in row-major cell order
    workers_[i]->seg_begin = shares[i].begin;
    workers_[i]->seg_end = shares[i].end;
  }
}

std::vector<std::pair<long long, long long>> InferenceSystem::last_shares() const {
  std::vector<std::pair<long long, long long>> out;
  for (const auto& w : workers_) out.emplace_back(w->seg_begin, w->seg_end);
  return out;
}

// Rows/s of every data-parallel worker running alone over one wave of its
// tiles (grid x batch rows, whole segments) of this run's store: untimed, like
// the upload in begin_run.  The second of two launches counts.
void InferenceSystem::probe_rates(const SampleStore& X) {
  const std::vector<int> per_model = workers_per_model();
  bool any = false;
  for (const auto& w : workers_) any = any || per_model[w->model] > 1;
  if (!any) return;
  const long long nb = static_cast<long long>(X.nb_samples());
  const long long S = static_cast<long long>(num_segments(X.nb_samples(), cluster_.segment_size));
  std::vector<double> rates(workers_.size(), 1.0);
  for (std::size_t i = 0; i < workers_.size(); ++i) {
    Worker& w = *workers_[i];
    if (per_model[w.model] < 2) continue;
    OnDevice on(w.phys);
    int grid = es::num_sms(w.phys);
    if (options_.sms_per_worker > 0) grid = std::min(grid, options_.sms_per_worker);
    const long long want = (static_cast<long long>(grid) * w.batch + cluster_.segment_size - 1) /
                           cluster_.segment_size;
    const long long segs = std::max<long long>(1, std::min(S, want));
    float* out = w.staged(false) ? w.staging : impl_->logits[w.model];
    float ms = 0.0f;
    for (int rep = 0; rep < 2; ++rep) {
      ES_CUDA(cudaEventRecord(w.ev_begin, w.stream));
      w.member->forward(x_on(X, w.phys), nb, cluster_.segment_size, 0, segs, out, grid,
                        w.stream, nullptr);
      ES_CUDA(cudaEventRecord(w.ev_done, w.stream));
      ES_CUDA(cudaEventSynchronize(w.ev_done));
      ES_CUDA(cudaEventElapsedTime(&ms, w.ev_begin, w.ev_done));
    }
    const double rows = static_cast<double>(std::min(nb, segs * cluster_.segment_size));
    rates[i] = rows / std::max(static_cast<double>(ms) * 1e-3, 1e-9);
  }
  rates_ = std::move(rates);
}

const void* InferenceSystem::x_on(const SampleStore& X, int phys) const {
  if (options_.fp32) return X.device_replica_f32(phys);
  return X.device_replica(phys);
}

bool InferenceSystem::single_device() const {
  for (const auto& w : workers_)
    if (w->remote) return false;
  return true;
}

std::vector<std::vector<int>> InferenceSystem::last_claims() const {
  std::vector<std::vector<int>> out(impl_->queues.size());
  OnDevice on(combine_dev_);
  ES_CUDA(cudaStreamSynchronize(impl_->main));
  for (std::size_t m = 0; m < impl_->queues.size(); ++m) {
    const Impl::Queue& q = impl_->queues[m];
    if (!q.on || q.segments == 0) continue;
    out[m].resize(static_cast<std::size_t>(q.segments));
    ES_CUDA(cudaMemcpy(out[m].data(), q.owner, out[m].size() * sizeof(int), cudaMemcpyDeviceToHost));
  }
  return out;
}

std::vector<int> InferenceSystem::claim_models() const {
  std::vector<int> out;
  for (std::size_t m = 0; m < impl_->queues.size(); ++m)
    if (impl_->queues[m].on) out.push_back(static_cast<int>(m));
  return out;
}

std::vector<int> InferenceSystem::worker_routes() const {
  std::vector<int> r;
  for (const auto& w : workers_) r.push_back(!w->remote ? 0 : w->direct ? 1 : 2);
  return r;
}

std::vector<int> InferenceSystem::workers_per_model() const {
  std::vector<int> n(cluster_.model_count(), 0);
  for (const auto& w : workers_) ++n[w->model];
  return n;
}

void InferenceSystem::begin_run(std::shared_ptr<const SampleStore> X) { begin_run(std::move(X), rule_); }

void InferenceSystem::begin_run(std::shared_ptr<const SampleStore> X, CombinationRule rule) {
  if (!X) throw SpecError("no sample store");
  if (shut_down_) throw Error("inference system is shut down");
  if (run_open_) throw Error("previous run still open");
  if (rule.kind == CombinationRule::Kind::weighted_averaging &&
      rule.weights.size() != static_cast<std::size_t>(cluster_.model_count()))
    throw SpecError("weighted averaging needs one weight per model");
  for (const ModelSpec& m : cluster_.models)
    if (m.arch.kind != MemberArch::Kind::Synthetic &&
        static_cast<std::size_t>(m.arch.input_width()) != X->width())
      throw SpecError(m.name + ": input width " + std::to_string(m.arch.input_width()) +
                      " differs from the store's " + std::to_string(X->width()));
  const std::size_t nb = X->nb_samples();
  const int C = output_width_;
  // Device replicas (untimed, like the reference's begin_run).
  for (const auto& w : workers_) x_on(*X, w->phys);
  {
    OnDevice on(combine_dev_);
    if (nb > impl_->cap_rows) {
      for (float*& p : impl_->logits) {
        cudaFree(p);
        p = nullptr;
      }
      cudaFree(impl_->y);
      cudaFree(impl_->labels);
      const std::size_t rows = std::max<std::size_t>(nb, 1);
      for (float*& p : impl_->logits) ES_CUDA(cudaMalloc(&p, rows * C * sizeof(float)));
      ES_CUDA(cudaMalloc(&impl_->y, rows * C * sizeof(float)));
      ES_CUDA(cudaMalloc(&impl_->labels, rows * sizeof(int32_t)));
      impl_->cap_rows = rows;
    }
  }
  const std::size_t S = num_segments(nb, cluster_.segment_size);
  for (auto& w : workers_) {
    if (w->remote && w->staging_rows < nb) {
      OnDevice on(w->phys);
      cudaFree(w->staging);
      ES_CUDA(cudaMalloc(&w->staging, std::max<std::size_t>(nb, 1) * C * sizeof(float)));
      w->staging_rows = nb;
    }
  }
  if (!options_.dp_equal_split && rates_.empty() && nb > 0) probe_rates(*X);
  assign_shares(nb);
  // Device FIFO sizing: chunks of about S / (4 W) segments, at least two
  // waves of 128-row tiles on the smallest worker GPU, so every claimed round
  // still fills the machine; enough rounds per worker to drain the queue alone.
  {
    const std::vector<int> per_model = workers_per_model();
    for (int m = 0; m < cluster_.model_count(); ++m) {
      Impl::Queue& q = impl_->queues[m];
      if (!q.on) continue;
      q.segments = static_cast<long long>(S);
      int sms = 1 << 30;
      for (const auto& w : workers_)
        if (w->model == m) sms = std::min(sms, es::num_sms(w->phys));
      long long chunk = options_.claim_chunk;
      if (chunk <= 0)
        chunk = std::max<long long>(2LL * sms, (q.segments + 4LL * per_model[m] - 1) /
                                                   (4LL * per_model[m]));
      q.chunk = std::max<long long>(1, chunk);
      q.rounds = q.segments > 0 ? (q.segments + q.chunk - 1) / q.chunk : 0;
      if (static_cast<std::size_t>(q.segments) > q.owner_cap) {
        OnDevice oc(combine_dev_);
        cudaFree(q.owner);
        q.owner = nullptr;
        ES_CUDA(cudaMalloc(&q.owner, std::max<std::size_t>(S, 1) * sizeof(int)));
        q.owner_cap = S;
      }
    }
  }
  // Fast gather: one partial per device row (pure model placement only).
  impl_->partial_mode = false;
  if (options_.row_partials) {
    const std::vector<int> per_model = workers_per_model();
    bool single = true;
    for (int n : per_model) single = single && n == 1;
    impl_->partial_mode = single;
  }
  if (impl_->partial_mode) {
    impl_->partials.resize(static_cast<std::size_t>(cluster_.device_count()));
    for (auto& w : workers_) {
      Impl::RowPartial& p = impl_->partials[static_cast<std::size_t>(w->row)];
      p.phys = w->phys;
      if (p.rows < nb) {
        OnDevice on(p.phys);
        if (p.at_combine != p.local) {
          OnDevice oc(combine_dev_);
          cudaFree(p.at_combine);
        }
        cudaFree(p.local);
        ES_CUDA(cudaMalloc(&p.local, std::max<std::size_t>(nb, 1) * C * sizeof(float)));
        p.at_combine = p.local;
        if (p.phys != combine_dev_) {
          OnDevice oc(combine_dev_);
          ES_CUDA(cudaMalloc(&p.at_combine, std::max<std::size_t>(nb, 1) * C * sizeof(float)));
        }
        p.rows = nb;
      }
      if (!p.done) {
        OnDevice on(p.phys);
        ES_CUDA(cudaEventCreateWithFlags(&p.done, cudaEventDisableTiming));
      }
    }
  }
  if (impl_->comm) {
    const int r = impl_->comm->rank();
    if (static_cast<long long>(nb) != impl_->g_rows[r])
      throw SpecError("gather plan gives rank " + std::to_string(r) + " " +
                      std::to_string(impl_->g_rows[r]) + " rows, the store holds " +
                      std::to_string(nb));
    if (r == impl_->root) {
      std::size_t total = 0;
      for (long long n : impl_->g_rows) total += static_cast<std::size_t>(n);
      if (total > impl_->g_cap) {
        OnDevice on(combine_dev_);
        cudaFree(impl_->gy);
        cudaFree(impl_->glabels);
        impl_->gy = nullptr;
        impl_->glabels = nullptr;
        ES_CUDA(cudaMalloc(&impl_->gy, total * C * sizeof(float)));
        ES_CUDA(cudaMalloc(&impl_->glabels, total * sizeof(int32_t)));
        impl_->g_cap = total;
      }
    }
  }
  impl_->store = std::move(X);
  impl_->rule = std::move(rule);
  impl_->segments = S;
  run_open_ = true;
}

std::size_t InferenceSystem::broadcast() {
  if (!run_open_) throw Error("broadcast without begin_run");
  const SampleStore& X = *impl_->store;
  const long long nb = static_cast<long long>(X.nb_samples());
  const int C = output_width_;
  launches_ = 0;
  {
    OnDevice on(combine_dev_);
    // Fresh queues: every segment of a data-parallel model once more.
    for (const Impl::Queue& q : impl_->queues)
      if (q.on && q.segments > 0) {
        ES_CUDA(cudaMemsetAsync(q.counter, 0, sizeof(unsigned long long), impl_->main));
        ES_CUDA(cudaMemsetAsync(q.owner, 0xff, static_cast<std::size_t>(q.segments) * sizeof(int),
                                impl_->main));
      }
    ES_CUDA(cudaEventRecord(impl_->start, impl_->main));
  }
  for (auto& w : workers_) {
    OnDevice on(w->phys);
    ES_CUDA(cudaStreamWaitEvent(w->stream, impl_->start, 0));
    ES_CUDA(cudaEventRecord(w->ev_begin, w->stream));
    const bool staged = w->staged(impl_->partial_mode);
    float* out = staged ? w->staging : impl_->logits[w->model];
    int grid = es::num_sms(w->phys);
    if (options_.sms_per_worker > 0) grid = std::min(grid, options_.sms_per_worker);
    Nvtx range("worker row " + std::to_string(w->row) + " model " + std::to_string(w->model) +
               " b=" + std::to_string(w->batch) + " segments [" + std::to_string(w->seg_begin) +
               "," + std::to_string(w->seg_end) + ")");
    const Impl::Queue& q = impl_->queues[w->model];
    if (q.on) {
      // Device FIFO: pop a chunk, run the member chain over it, repeat; a
      // round after the queue ran dry claims an empty run and its launches
      // exit at once.  The worker's launch marks all land after its rounds.
      const int index = static_cast<int>(&w - workers_.data());
      for (long long r = 0; r < q.rounds; ++r) {
        ES_LAUNCH(es::claim_launch(q.counter, q.segments, q.chunk, cluster_.segment_size, nb,
                                   w->claim, q.owner, index, w->stream));
        launches_ += 1 + w->member->forward(x_on(X, w->phys), nb, cluster_.segment_size,
                                            0, q.segments, out, grid, w->stream, nullptr, w->claim);
      }
      for (cudaEvent_t e : w->marks) ES_CUDA(cudaEventRecord(e, w->stream));
    } else {
      launches_ += w->member->forward(x_on(X, w->phys), nb, cluster_.segment_size,
                                      w->seg_begin, w->seg_end, out, grid, w->stream,
                                      w->marks.empty() ? nullptr : w->marks.data());
    }
    if (!q.on && staged && w->seg_end > w->seg_begin && !impl_->partial_mode) {
      const long long r0 = w->seg_begin * cluster_.segment_size;
      const long long r1 = std::min<long long>(w->seg_end * cluster_.segment_size, nb);
      ES_CUDA(cudaMemcpyPeerAsync(impl_->logits[w->model] + r0 * C, combine_dev_,
                                  w->staging + r0 * C, w->phys,
                                  static_cast<std::size_t>(r1 - r0) * C * sizeof(float), w->stream));
    }
    ES_CUDA(cudaEventRecord(w->ev_done, w->stream));
  }
  if (impl_->partial_mode && nb > 0) return broadcast_partials(nb);
  OnDevice on(combine_dev_);
  for (auto& w : workers_) ES_CUDA(cudaStreamWaitEvent(impl_->main, w->ev_done, 0));
  ES_CUDA(cudaEventRecord(impl_->combine_begin, impl_->main));
  Nvtx range("combine " + impl_->rule.name());
  es::CombineArgs ca = combine_args(impl_->rule, impl_->logits, static_cast<std::size_t>(nb),
                                    C, impl_->y, impl_->labels);
  if (nb > 0) {
    ES_LAUNCH(es::combine_launch(ca, impl_->main));
    ++launches_;
  }
  finish_broadcast();
  return impl_->segments;
}

void InferenceSystem::finish_broadcast() {
  if (impl_->comm) {
    ES_CUDA(cudaGetLastError());
    impl_->comm->gather_rows(impl_->y, impl_->labels, output_width_, impl_->g_first,
                             impl_->g_rows, impl_->root, impl_->gy, impl_->glabels, impl_->main);
  }
  ES_CUDA(cudaEventRecord(impl_->end, impl_->main));
}

void InferenceSystem::set_gather(std::shared_ptr<Comm> comm, int root,
                                 std::vector<long long> first_rows, std::vector<long long> rows) {
  if (run_open_) throw Error("set_gather while a run is open");
  if (!comm) {
    impl_->comm.reset();
    return;
  }
  if (comm->device() != combine_dev_)
    throw SpecError("the gather communicator must live on the combining GPU (CUDA ordinal " +
                    std::to_string(combine_dev_) + ")");
  const int n = comm->size();
  if (static_cast<int>(first_rows.size()) != n || static_cast<int>(rows.size()) != n)
    throw SpecError("gather plan needs one (first row, rows) pair per rank");
  if (root < 0 || root >= n) throw SpecError("gather root out of range");
  // The ranks' row ranges tile [0, total) exactly once.
  std::vector<std::pair<long long, long long>> r;
  for (int i = 0; i < n; ++i) {
    if (first_rows[i] < 0 || rows[i] < 0) throw SpecError("negative gather row range");
    r.emplace_back(first_rows[i], rows[i]);
  }
  std::sort(r.begin(), r.end());
  long long next = 0;
  for (const auto& [f, k] : r) {
    if (k == 0) continue;
    if (f != next) throw SpecError("gather row ranges must tile the result exactly once");
    next = f + k;
  }
  impl_->comm = std::move(comm);
  impl_->root = root;
  impl_->g_first = std::move(first_rows);
  impl_->g_rows = std::move(rows);
}

// Fast gather (PoolOptions::row_partials): every device row folds its own
// members on its GPU -- the same K3 kernel over the row's members with the
// rule's per-member factor (avg: 1/M of the whole ensemble, wavg: w_m; vote:
// tallies) -- and the combining GPU sums the partials in row order with factor
// 1 (exact for tallies) and takes the argmax.
std::size_t InferenceSystem::broadcast_partials(long long nb) {
  const int C = output_width_;
  const int M = cluster_.model_count();
  const CombinationRule& rule = impl_->rule;
  const bool vote = rule.kind == CombinationRule::Kind::majority_vote;
  std::vector<float*> finals;
  for (std::size_t d = 0; d < impl_->partials.size(); ++d) {
    Impl::RowPartial& p = impl_->partials[d];
    es::CombineArgs ca;
    ca.C = C;
    ca.rows = nb;
    ca.y = p.local;
    ca.argmax = nullptr;
    ca.softmax = rule.member_softmax ? 1 : 0;
    ca.rule = vote ? es::kVote : es::kWeighted;
    Worker* last = nullptr;
    for (auto& w : workers_) {
      if (w->row != static_cast<int>(d)) continue;
      ca.logits[ca.M] = w->staged(true) ? w->staging : impl_->logits[w->model];
      ca.weight[ca.M] = rule.kind == CombinationRule::Kind::weighted_averaging
                            ? static_cast<float>(rule.weights[w->model])
                            : 1.0f / static_cast<float>(M);
      ++ca.M;
      last = w.get();
    }
    if (!last) continue;
    OnDevice on(p.phys);
    for (auto& w : workers_)  // the row's workers may run on other streams
      if (w->row == static_cast<int>(d) && w.get() != last)
        ES_CUDA(cudaStreamWaitEvent(last->stream, w->ev_done, 0));
    ES_LAUNCH(es::combine_launch(ca, last->stream));
    ++launches_;
    if (p.at_combine != p.local)
      ES_CUDA(cudaMemcpyPeerAsync(p.at_combine, combine_dev_, p.local, p.phys,
                                  static_cast<std::size_t>(nb) * C * sizeof(float), last->stream));
    ES_CUDA(cudaEventRecord(p.done, last->stream));
    finals.push_back(p.at_combine);
  }
  OnDevice on(combine_dev_);
  for (auto& w : workers_) ES_CUDA(cudaStreamWaitEvent(impl_->main, w->ev_done, 0));
  for (const Impl::RowPartial& p : impl_->partials)
    if (p.done && p.rows) ES_CUDA(cudaStreamWaitEvent(impl_->main, p.done, 0));
  ES_CUDA(cudaEventRecord(impl_->combine_begin, impl_->main));
  es::CombineArgs fa;
  fa.M = static_cast<int>(finals.size());
  fa.C = C;
  fa.rows = nb;
  fa.y = impl_->y;
  fa.argmax = impl_->labels;
  fa.softmax = 0;
  fa.rule = es::kWeighted;
  for (int i = 0; i < fa.M; ++i) {
    fa.logits[i] = finals[static_cast<std::size_t>(i)];
    fa.weight[i] = 1.0f;
  }
  ES_LAUNCH(es::combine_launch(fa, impl_->main));
  ++launches_;
  finish_broadcast();
  return impl_->segments;
}

RunOutput InferenceSystem::await_run() {
  if (!run_open_) throw Error("await without begin_run");
  run_open_ = false;
  OnDevice on(combine_dev_);
  cudaError_t e = cudaEventSynchronize(impl_->end);
  if (e != cudaSuccess) throw_cuda(e, "run failed on device");
  for (auto& w : workers_) {
    OnDevice wd(w->phys);
    ES_CUDA(cudaStreamSynchronize(w->stream));
  }
  float ms = 0.0f;
  ES_CUDA(cudaEventElapsedTime(&ms, impl_->start, impl_->end));
  const SampleStore& X = *impl_->store;
  const std::size_t nb = X.nb_samples();
  RunOutput out;
  out.output_width = output_width_;
  out.stats.nb_samples = nb;
  out.stats.segments = impl_->segments;
  out.stats.data_messages = impl_->segments * static_cast<std::size_t>(cluster_.model_count());
  out.stats.segment_rows.resize(impl_->segments);
  for (std::size_t s = 0; s < impl_->segments; ++s)
    out.stats.segment_rows[s] = segment_bounds(static_cast<int>(s), cluster_.segment_size, nb).size();
  out.stats.elapsed_s = ms * 1e-3;
  // The gather root returns every rank's rows.
  const bool gathered = impl_->comm && impl_->comm->rank() == impl_->root;
  std::size_t rows = nb;
  if (gathered) {
    rows = 0;
    for (long long n : impl_->g_rows) rows += static_cast<std::size_t>(n);
  }
  if (options_.copy_outputs && rows > 0) {
    out.combined.resize(rows * output_width_);
    out.winners.resize(rows);
    ES_CUDA(cudaMemcpy(out.combined.data(), gathered ? impl_->gy : impl_->y,
                       out.combined.size() * sizeof(float), cudaMemcpyDeviceToHost));
    ES_CUDA(cudaMemcpy(out.winners.data(), gathered ? impl_->glabels : impl_->labels,
                       rows * sizeof(int32_t), cudaMemcpyDeviceToHost));
  }
  return out;
}

RunOutput InferenceSystem::run(std::shared_ptr<const SampleStore> X) { return run(std::move(X), rule_); }

RunOutput InferenceSystem::run(std::shared_ptr<const SampleStore> X, CombinationRule rule) {
  begin_run(std::move(X), std::move(rule));
  broadcast();
  return await_run();
}

double InferenceSystem::last_member_ms(int worker) const {
  const Worker& w = *workers_.at(worker);
  OnDevice on(w.phys);
  float ms = 0.0f;
  if (cudaEventElapsedTime(&ms, w.ev_begin, w.ev_done) != cudaSuccess) return -1.0;
  return ms;
}

std::vector<double> InferenceSystem::last_kernel_ms(int worker) const {
  const Worker& w = *workers_.at(worker);
  OnDevice on(w.phys);
  std::vector<double> out;
  cudaEvent_t prev = w.ev_begin;
  for (cudaEvent_t e : w.marks) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, prev, e) != cudaSuccess) {
      cudaGetLastError();
      return {};
    }
    out.push_back(ms);
    prev = e;
  }
  return out;
}

std::vector<std::string> InferenceSystem::kernel_names(int worker) const {
  return workers_.at(worker)->member->kernel_names();
}

double InferenceSystem::last_combine_ms() const {
  OnDevice on(combine_dev_);
  float ms = 0.0f;
  if (cudaEventElapsedTime(&ms, impl_->combine_begin, impl_->end) != cudaSuccess) return -1.0;
  return ms;
}

// End to end from host memory, pipelined over chunks of whole segments:
//   host threads: fp32 -> bf16 of chunk i into a pinned slot (2 B/feature on
//                 the wire) — or, with e2e_host_convert off, the fp32 chunk
//                 itself is copied and converted on the device;
//   copy stream:  H2D of chunk i while chunk i-1 computes;
//   main stream:  member kernels + combine of chunk i into slot buffers;
//   d2h stream:   combined probabilities + labels of chunk i back to the caller.
// The returned time is host wall-clock around the whole call (it includes the
// host conversion, which no CUDA event can see).
double InferenceSystem::run_host(const float* X, std::size_t nb, std::size_t width, float* Y_out,
                                 std::int32_t* labels_out) {
  // Chunk routes: "convert" = host threads write bf16 into a
  // pinned slot, 2 B/feature cross PCIe; "direct" = DMA straight from the
  // caller's pinned fp32 buffer, converted on the device (no host-memory
  // pass).  Alternating them balances host-memory bandwidth against PCIe.
  cudaPointerAttributes pa{};
  const bool pinned_input =
      cudaPointerGetAttributes(&pa, X) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  // fp32 members read fp32 rows: every chunk is DMA'd as is (mode 3).
  const int mode = options_.fp32 ? 3
                   : options_.e2e_host_convert ? (pinned_input ? 0 : 1)
                                               : (pinned_input ? 2 : 1);
  const std::size_t k8 = static_cast<std::size_t>(std::clamp(options_.e2e_convert_eighths, 0, 8));
  return run_host_core(nb, width, Y_out, labels_out,
                       [&](std::size_t i, std::uint16_t* pinned, std::size_t r0,
                           std::size_t rows) -> HostChunk {
                         const bool convert = mode != 3 && (mode == 1 || (mode == 0 && (i + 1) * k8 / 8 > i * k8 / 8));
                         if (!convert) return {X + r0 * width, true};
                         convert_f32_to_bf16_host(X + r0 * width, pinned, rows * width,
                                                  *impl_->pool);
                         return {};
                       });
}

double InferenceSystem::run_host_blocks(const std::vector<HostRowBlock>& blocks, std::size_t width,
                                        float* Y_out, std::int32_t* labels_out) {
  if (options_.fp32)
    throw SpecError("fp32 members read fp32 rows; host row blocks carry bf16 (use run_host)");
  std::size_t nb = 0;
  for (const HostRowBlock& b : blocks) nb += b.rows;
  std::vector<std::size_t> first(blocks.size() + 1, 0);  // first row of every block
  for (std::size_t k = 0; k < blocks.size(); ++k) first[k + 1] = first[k] + blocks[k].rows;
  return run_host_core(nb, width, Y_out, labels_out,
                       [&](std::size_t, std::uint16_t* pinned, std::size_t r0,
                           std::size_t rows) -> HostChunk {
                         // A chunk inside one page-locked block goes straight to the DMA.
                         const std::size_t k0 =
                             std::upper_bound(first.begin(), first.end(), r0) - first.begin() - 1;
                         if (blocks[k0].pinned && r0 + rows <= first[k0 + 1])
                           return {blocks[k0].bf16 + (r0 - first[k0]) * width, false};
                         // Gather rows [r0, r0 + rows) from the blocks, split over the pool.
                         const std::function<void(int, int)> job = [&](int part, int parts) {
                           const std::size_t per = (rows + parts - 1) / parts;
                           const std::size_t a = r0 + std::min(rows, part * per);
                           const std::size_t e = r0 + std::min(rows, (part + 1) * per);
                           std::size_t k = std::upper_bound(first.begin(), first.end(), a) -
                                           first.begin() - 1;
                           for (std::size_t r = a; r < e; ++k) {
                             const std::size_t take = std::min(e, first[k + 1]) - r;
                             std::memcpy(pinned + (r - r0) * width,
                                         blocks[k].bf16 + (r - first[k]) * width,
                                         take * width * sizeof(std::uint16_t));
                             r += take;
                           }
                         };
                         impl_->pool->run(job);
                         return {};
                       });
}

// End to end from host memory, pipelined over chunks of whole segments:
//   host threads: fill(i) puts chunk i into a pinned slot as bf16 (2 B/feature
//                 on the wire) — or returns a pinned fp32 source that is DMA'd
//                 as is and converted on the device;
//   copy stream:  H2D of chunk i while chunk i-1 computes;
//   main stream:  member kernels + combine of chunk i into slot buffers;
//   d2h stream:   combined probabilities + labels of chunk i back to the caller.
// The returned time is host wall-clock around the whole call (it includes the
// host conversion, which no CUDA event can see).
double InferenceSystem::run_host_core(std::size_t nb, std::size_t width, float* Y_out,
                                      std::int32_t* labels_out, const HostFill& fill) {
  if (run_open_) throw Error("previous run still open");
  for (const ModelSpec& m : cluster_.models)
    if (m.arch.kind != MemberArch::Kind::Synthetic &&
        static_cast<std::size_t>(m.arch.input_width()) != width)
      throw SpecError(m.name + ": input width differs from the samples'");
  OnDevice on(combine_dev_);
  Impl& I = *impl_;
  const int C = output_width_;
  const int M = cluster_.model_count();
  const std::size_t seg = static_cast<std::size_t>(cluster_.segment_size);
  const std::size_t chunk = std::max<std::size_t>(seg, (options_.e2e_chunk_rows / seg) * seg);
  constexpr int kSlots = 3;
  if (chunk * width > I.e2e_chunk_elems) {
    I.free_e2e();
    I.e2e_chunk_elems = chunk * width;
    // Lanes: the combining node first, then every other node in worker order.
    auto node_of = [&](const Worker& w) {
      return w.remote ? (options_.row_nodes ? 1000000 + w.row : w.phys) : -1;
    };
    std::vector<int> keys;
    for (std::size_t i = 0; i < workers_.size(); ++i) {
      const int key = node_of(*workers_[i]);
      auto it = std::find(keys.begin(), keys.end(), key);
      std::size_t l = static_cast<std::size_t>(it - keys.begin());
      if (it == keys.end()) {
        if (key == -1) {  // keep the combining node at lane 0
          keys.insert(keys.begin(), key);
          I.lanes.insert(I.lanes.begin(), Impl::Lane{});
          l = 0;
        } else {
          keys.push_back(key);
          I.lanes.emplace_back();
        }
        I.lanes[l].phys = workers_[i]->phys;
      }
      I.lanes[l].workers.push_back(static_cast<int>(i));
    }
    if (keys.empty() || keys.front() != -1) {  // no worker on the combining node
      keys.insert(keys.begin(), -1);
      I.lanes.insert(I.lanes.begin(), Impl::Lane{});
      I.lanes[0].phys = combine_dev_;
    }
    for (std::size_t l = 0; l < I.lanes.size(); ++l) {
      Impl::Lane& ln = I.lanes[l];
      OnDevice od(ln.phys);
      ES_CUDA(cudaStreamCreateWithFlags(&ln.copy, cudaStreamNonBlocking));
      if (l == 0)
        ln.comp = I.main;
      else
        ES_CUDA(cudaStreamCreateWithFlags(&ln.comp, cudaStreamNonBlocking));
      for (Impl::Lane::LSlot& ls : ln.s) {
        ES_CUDA(cudaMalloc(&ls.x32, chunk * width * sizeof(float)));
        ES_CUDA(cudaMalloc(&ls.x16, chunk * width * 2));
        ls.staging.assign(M, nullptr);
        for (int wi : ln.workers)
          if (workers_[wi]->staged(false) && !ls.staging[workers_[wi]->model])
            ES_CUDA(cudaMalloc(&ls.staging[workers_[wi]->model], chunk * C * sizeof(float)));
        ES_CUDA(cudaEventCreateWithFlags(&ls.h2d_done, cudaEventDisableTiming));
        ES_CUDA(cudaEventCreateWithFlags(&ls.comp_done, cudaEventDisableTiming));
      }
    }
    for (int s = 0; s < kSlots; ++s) {
      Impl::Slot& sl = I.slots[s];
      // Portable: every lane's GPU DMAs from it.
      ES_CUDA(cudaHostAlloc(&sl.pinned, chunk * width * 2, cudaHostAllocPortable));
      sl.logits.assign(M, nullptr);
      for (float*& p : sl.logits) ES_CUDA(cudaMalloc(&p, chunk * C * sizeof(float)));
      ES_CUDA(cudaMalloc(&sl.y, chunk * C * sizeof(float)));
      ES_CUDA(cudaMalloc(&sl.labels, chunk * sizeof(int32_t)));
      ES_CUDA(cudaEventCreateWithFlags(&sl.combined, cudaEventDisableTiming));
      ES_CUDA(cudaEventCreateWithFlags(&sl.d2h_done, cudaEventDisableTiming));
    }
    ES_CUDA(cudaStreamCreateWithFlags(&I.d2h, cudaStreamNonBlocking));
  }
  if (!I.pool) I.pool = std::make_unique<ThreadPool>(0);
  for (const Impl::Lane& ln : I.lanes) {
    OnDevice od(ln.phys);
    ES_CUDA(cudaDeviceSynchronize());
  }
  for (Impl::Lane& ln : I.lanes)
    for (Impl::Lane::LSlot& ls : ln.s) ls.used = false;
  const auto t0 = std::chrono::steady_clock::now();
  launches_ = 0;
  h2d_bytes_ = d2h_bytes_ = 0;
  const std::size_t nchunks = (nb + chunk - 1) / chunk;
  for (std::size_t i = 0; i < nchunks; ++i) {
    const int si = static_cast<int>(i % kSlots);
    Impl::Slot& sl = I.slots[si];
    Nvtx range("run_host chunk " + std::to_string(i));
    const std::size_t r0 = i * chunk;
    const std::size_t rows = std::min(chunk, nb - r0);
    if (i >= kSlots)  // the pinned slot is reusable once every lane's H2D of chunk i-3 is done
      for (Impl::Lane& ln : I.lanes)
        if (ln.s[si].used) ES_CUDA(cudaEventSynchronize(ln.s[si].h2d_done));
    const HostChunk src = fill(i, static_cast<std::uint16_t*>(sl.pinned), r0, rows);
    const float* direct = src.fp32 ? static_cast<const float*>(src.src) : nullptr;
    const std::uint16_t* bf = static_cast<const std::uint16_t*>(src.src ? src.src : sl.pinned);
    std::vector<SegmentShare> shares =
        rates_.empty() ? segment_shares(matrix_, rows, cluster_.segment_size)
                       : segment_shares_weighted(matrix_, rows, cluster_.segment_size, rates_);
    for (std::size_t l = 0; l < I.lanes.size(); ++l) {
      Impl::Lane& ln = I.lanes[l];
      Impl::Lane::LSlot& ls = ln.s[si];
      // Rows this lane's workers predict in the chunk (their segment runs are
      // contiguous; a lane with a whole member needs the whole chunk).
      long long sb = -1, se = -1;
      for (int wi : ln.workers)
        if (shares[wi].end > shares[wi].begin) {
          sb = sb < 0 ? shares[wi].begin : std::min<long long>(sb, shares[wi].begin);
          se = std::max<long long>(se, shares[wi].end);
        }
      ls.used = sb >= 0;
      if (!ls.used) continue;
      const std::size_t g0 = static_cast<std::size_t>(sb) * seg;
      const std::size_t g1 = std::min(static_cast<std::size_t>(se) * seg, rows);
      const std::size_t elems = (g1 - g0) * width;
      OnDevice od(ln.phys);
      // x16/x32 of this slot are free once the lane's compute of chunk i-3 is done.
      if (i >= kSlots) ES_CUDA(cudaStreamWaitEvent(ln.copy, ls.comp_done, 0));
      h2d_bytes_ += elems * (direct ? sizeof(float) : 2);
      if (!direct)
        ES_CUDA(cudaMemcpyAsync(static_cast<std::uint16_t*>(ls.x16) + g0 * width, bf + g0 * width,
                                elems * 2, cudaMemcpyHostToDevice, ln.copy));
      else
        ES_CUDA(cudaMemcpyAsync(ls.x32 + g0 * width, direct + g0 * width, elems * sizeof(float),
                                cudaMemcpyHostToDevice, ln.copy));
      ES_CUDA(cudaEventRecord(ls.h2d_done, ln.copy));
      ES_CUDA(cudaStreamWaitEvent(ln.comp, ls.h2d_done, 0));
      if (direct && !options_.fp32) {
        ES_LAUNCH(es::convert_f32_to_bf16(ls.x32 + g0 * width,
                                          static_cast<__nv_bfloat16*>(ls.x16) + g0 * width, elems,
                                          ln.comp));
        ++launches_;
      }
      const void* xin = options_.fp32 ? static_cast<const void*>(ls.x32) : ls.x16;
      // The combining slot's logits are free once its combine of chunk i-3 ran.
      if (i >= kSlots) ES_CUDA(cudaStreamWaitEvent(ln.comp, sl.combined, 0));
      const int grid = es::num_sms(ln.phys);
      for (int wi : ln.workers) {
        Worker& w = *workers_[wi];
        const SegmentShare& sh = shares[wi];
        if (sh.end <= sh.begin) continue;
        const bool staged = w.staged(false);
        float* out = staged ? ls.staging[w.model] : sl.logits[w.model];
        launches_ += w.member->forward(xin, static_cast<long long>(rows), cluster_.segment_size,
                                       sh.begin, sh.end, out, grid, ln.comp);
        if (staged) {
          const std::size_t a = static_cast<std::size_t>(sh.begin) * seg;
          const std::size_t e = std::min(static_cast<std::size_t>(sh.end) * seg, rows);
          ES_CUDA(cudaMemcpyPeerAsync(sl.logits[w.model] + a * C, combine_dev_, out + a * C,
                                      ln.phys, (e - a) * C * sizeof(float), ln.comp));
        }
      }
      ES_CUDA(cudaEventRecord(ls.comp_done, ln.comp));
    }
    for (std::size_t l = 1; l < I.lanes.size(); ++l)
      if (I.lanes[l].s[si].used) ES_CUDA(cudaStreamWaitEvent(I.main, I.lanes[l].s[si].comp_done, 0));
    if (i >= kSlots) ES_CUDA(cudaStreamWaitEvent(I.main, sl.d2h_done, 0));  // y/labels free
    d2h_bytes_ += (Y_out ? rows * C * sizeof(float) : 0) + (labels_out ? rows * sizeof(int32_t) : 0);
    es::CombineArgs ca = combine_args(rule_, sl.logits, rows, C, sl.y, sl.labels);
    ES_LAUNCH(es::combine_launch(ca, I.main));
    ++launches_;
    ES_CUDA(cudaEventRecord(sl.combined, I.main));
    ES_CUDA(cudaStreamWaitEvent(I.d2h, sl.combined, 0));
    if (Y_out)
      ES_CUDA(cudaMemcpyAsync(Y_out + r0 * C, sl.y, rows * C * sizeof(float),
                              cudaMemcpyDeviceToHost, I.d2h));
    if (labels_out)
      ES_CUDA(cudaMemcpyAsync(labels_out + r0, sl.labels, rows * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, I.d2h));
    ES_CUDA(cudaEventRecord(sl.d2h_done, I.d2h));
  }
  ES_CUDA(cudaStreamSynchronize(I.d2h));
  for (const Impl::Lane& ln : I.lanes) {
    OnDevice od(ln.phys);
    ES_CUDA(cudaStreamSynchronize(ln.comp));
  }
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

// ---------------------------------------------------------------- free functions
InferenceResult run_inference(std::shared_ptr<const SampleStore> X, const AllocationMatrix& A,
                              const ClusterSpec& cluster, CombinationRule rule, Mode mode,
                              PoolOptions options) {
  if (!X) throw SpecError("no sample store");
  if (mode == Mode::Benchmark && X->nb_samples() == 0)
    throw SpecError("benchmark mode needs a nonempty sample store");
  InferenceSystem system(A, cluster, std::move(rule), options);
  RunOutput out = system.run(X);
  system.shutdown();
  InferenceResult result;
  if (mode == Mode::Deploy) {
    result.output = std::move(out);
  } else {
    BenchResult s;
    s.nb_samples = out.stats.nb_samples;
    s.elapsed_s = std::max(out.stats.elapsed_s, 1e-9);
    s.throughput = static_cast<double>(s.nb_samples) / s.elapsed_s;
    s.runs = {s.throughput};
    result.score = s;
  }
  return result;
}

double median(std::vector<double> values) {
  if (values.empty()) return 0.0;
  std::sort(values.begin(), values.end());
  const std::size_t h = values.size() / 2;
  return values.size() % 2 ? values[h] : 0.5 * (values[h - 1] + values[h]);
}

double relative_standard_deviation(const std::vector<double>& values) {
  if (values.size() < 2) return 0.0;
  double mean = 0.0;
  for (double v : values) mean += v;
  mean /= static_cast<double>(values.size());
  if (mean == 0.0) return 0.0;
  double ss = 0.0;
  for (double v : values) ss += (v - mean) * (v - mean);
  return std::sqrt(ss / static_cast<double>(values.size() - 1)) / mean;
}

BenchResult bench(const AllocationMatrix& A, std::shared_ptr<const SampleStore> calib,
                  const ClusterSpec& cluster, int repeats, PoolOptions options) {
  if (repeats < 1) throw std::invalid_argument("repeats must be >= 1");
  if (!calib || calib->nb_samples() == 0) throw SpecError("empty calibration set");
  BenchResult result;
  result.nb_samples = calib->nb_samples();
  try {
    if (!validate_matrix(A, cluster).ok) return result;
  } catch (const SpecError&) {
    return result;
  }
  if (!fit_mem(A, cluster).fits) return result;
  options.copy_outputs = false;
  try {
    InferenceSystem system(A, cluster, CombinationRule::averaging(true), options);
    if (options.warmup) system.run(calib);
    std::vector<double> elapsed;
    for (int r = 0; r < repeats; ++r) {
      RunOutput out = system.run(calib);
      elapsed.push_back(std::max(out.stats.elapsed_s, 1e-9));
      result.runs.push_back(static_cast<double>(calib->nb_samples()) / elapsed.back());
    }
    system.shutdown();
    result.elapsed_s = median(elapsed);
    result.throughput = median(result.runs);
    result.rsd = relative_standard_deviation(result.runs);
  } catch (const StartupError&) {
    result.runs.clear();
    result.throughput = 0.0;
  }
  return result;
}

// ---------------------------------------------------------------- compat seams
struct B200Predictor::State {
  int device = 0;
  ModelSpec model;
  int batch = 1;
  double load_mib = 0.0, capacity_mib = 0.0;
  std::unique_ptr<DeviceMember> member;
  cudaStream_t stream = nullptr;
  float* x32 = nullptr;
  __nv_bfloat16* x16 = nullptr;
  float* out = nullptr;
  std::size_t cap = 0, cap_out = 0;
};

B200Predictor::B200Predictor(int device, ModelSpec model, int batch, double device_load_mib,
                             double capacity_mib)
    : s_(std::make_unique<State>()) {
  s_->device = device;
  s_->model = std::move(model);
  s_->batch = batch;
  s_->load_mib = device_load_mib;
  s_->capacity_mib = capacity_mib;
}

B200Predictor::~B200Predictor() {
  if (!s_) return;
  cudaSetDevice(s_->device);
  if (s_->stream) cudaStreamSynchronize(s_->stream);
  cudaFree(s_->x32);
  cudaFree(s_->x16);
  cudaFree(s_->out);
  if (s_->stream) cudaStreamDestroy(s_->stream);
  s_->member.reset();
}

bool B200Predictor::load() {
  if (s_->load_mib > s_->capacity_mib) return false;
  auto m = std::make_unique<DeviceMember>();
  if (!m->load(s_->device, s_->model, s_->batch)) return false;
  OnDevice on(s_->device);
  ES_CUDA(cudaStreamCreateWithFlags(&s_->stream, cudaStreamNonBlocking));
  s_->member = std::move(m);
  return true;
}

void B200Predictor::predict(const float* features, std::size_t first_index, std::size_t rows,
                            std::size_t width, float* out) {
  if (!s_->member) throw Error("predict before a successful load()");
  const int C = s_->model.output_width;
  // The member kernels' TMA maps are [rows][input_width]: a narrower row
  // would make them read past the staging buffer (begin_run checks the same).
  if (s_->model.arch.kind != MemberArch::Kind::Synthetic &&
      width != static_cast<std::size_t>(s_->model.arch.input_width()))
    throw SpecError(s_->model.name + ": input width " + std::to_string(s_->model.arch.input_width()) +
                    " differs from the batch's " + std::to_string(width));
  if (rows == 0) return;
  OnDevice on(s_->device);
  const std::size_t n = rows * width;
  if (n > s_->cap) {
    cudaFree(s_->x32);
    cudaFree(s_->x16);
    ES_CUDA(cudaMalloc(&s_->x32, n * sizeof(float)));
    ES_CUDA(cudaMalloc(&s_->x16, n * sizeof(__nv_bfloat16)));
    s_->cap = n;
  }
  if (rows > s_->cap_out) {
    cudaFree(s_->out);
    ES_CUDA(cudaMalloc(&s_->out, rows * C * sizeof(float)));
    s_->cap_out = rows;
  }
  ES_CUDA(cudaMemcpyAsync(s_->x32, features, n * sizeof(float), cudaMemcpyHostToDevice, s_->stream));
  ES_LAUNCH(es::convert_f32_to_bf16(s_->x32, s_->x16, n, s_->stream));
  if (s_->model.arch.kind == MemberArch::Kind::Synthetic) {
    // Keyed on absolute sample indices (backend.hpp:43-45): write the rows at
    // their global offset into a shifted view of the output buffer.
    const long long first = static_cast<long long>(first_index);
    ES_LAUNCH(es::synthetic_member_launch(s_->model.id, C, 1, first, first + static_cast<long long>(rows),
                                          first + static_cast<long long>(rows),
                                          s_->out - first * C, s_->stream));
  } else {
    s_->member->forward(s_->x16, static_cast<long long>(rows), static_cast<int>(rows), 0, 1, s_->out,
                        es::num_sms(s_->device), s_->stream);
  }
  ES_CUDA(cudaMemcpyAsync(out, s_->out, rows * C * sizeof(float), cudaMemcpyDeviceToHost, s_->stream));
  ES_CUDA(cudaStreamSynchronize(s_->stream));
}

void combine_blocks(const CombinationRule& rule, int M, int C, std::size_t rows,
                    const float* const* blocks, float* y, std::int32_t* winners) {
  if (M < 1 || M > es::kMaxMembers || C < 1 || C > es::kMaxClasses)
    throw SpecError("combine: unsupported member or class count");
  if (rule.kind == CombinationRule::Kind::weighted_averaging &&
      rule.weights.size() != static_cast<std::size_t>(M))
    throw SpecError("weighted averaging needs one weight per model");
  if (rows == 0) return;
  visible_devices();
  const std::size_t n = rows * C;
  std::vector<float*> dev(M, nullptr);
  float* dy = nullptr;
  int32_t* dl = nullptr;
  try {
    for (int m = 0; m < M; ++m) {
      ES_CUDA(cudaMalloc(&dev[m], n * sizeof(float)));
      ES_CUDA(cudaMemcpy(dev[m], blocks[m], n * sizeof(float), cudaMemcpyHostToDevice));
    }
    ES_CUDA(cudaMalloc(&dy, n * sizeof(float)));
    ES_CUDA(cudaMalloc(&dl, rows * sizeof(int32_t)));
    es::CombineArgs ca;
    ca.M = M;
    ca.C = C;
    ca.rows = static_cast<long long>(rows);
    ca.y = dy;
    ca.argmax = dl;
    ca.softmax = rule.member_softmax ? 1 : 0;
    ca.rule = rule.kind == CombinationRule::Kind::majority_vote ? es::kVote
              : rule.kind == CombinationRule::Kind::weighted_averaging ? es::kWeighted
                                                                         : es::kAverage;
    for (int m = 0; m < M; ++m) {
      ca.logits[m] = dev[m];
      ca.weight[m] = rule.kind == CombinationRule::Kind::weighted_averaging
                         ? static_cast<float>(rule.weights[m])
                         : 1.0f / static_cast<float>(M);
    }
    ES_LAUNCH(es::combine_launch(ca, 0));
    ES_CUDA(cudaMemcpy(y, dy, n * sizeof(float), cudaMemcpyDeviceToHost));
    if (winners) ES_CUDA(cudaMemcpy(winners, dl, rows * sizeof(int32_t), cudaMemcpyDeviceToHost));
  } catch (...) {
    for (float* p : dev) cudaFree(p);
    cudaFree(dy);
    cudaFree(dl);
    throw;
  }
  for (float* p : dev) cudaFree(p);
  cudaFree(dy);
  cudaFree(dl);
}

std::string device_identity() {
  const int n = visible_devices();
  cudaDeviceProp p{};
  ES_CUDA(cudaGetDeviceProperties(&p, 0));
  char buf[256];
  std::snprintf(buf, sizeof(buf), "%s/sm_%d%d/%d SMs/%.0f GiB x%d", p.name, p.major, p.minor,
                p.multiProcessorCount, static_cast<double>(p.totalGlobalMem) / (1 << 30), n);
  return buf;
}

void derive_footprint(ModelSpec& model) {
  if (model.arch.kind == MemberArch::Kind::Synthetic) return;
  constexpr double kMiB = 1024.0 * 1024.0;
  if (model.weight_mib <= 0)
    model.weight_mib = static_cast<double>(model.arch.parameter_count()) * 2.0 / kMiB;
  if (model.act_mib_per_sample <= 0) {
    model.act_mib_per_sample = model.arch.activation_elems() * 2.0 / kMiB;
  }
  if (model.cost_per_sample <= 0) model.cost_per_sample = model.arch.flops_per_sample();
}

}  // namespace enserve
