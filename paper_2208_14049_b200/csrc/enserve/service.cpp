// Deploy-mode prediction service (design in service.hpp).
#include "enserve/service.hpp"

#include <cuda_runtime.h>

#include <cstring>

#include "enserve/host_convert.hpp"

namespace enserve {

PredictionService::PredictionService(ClusterSpec cluster, AllocationMatrix matrix,
                                     ServiceConfig config)
    : cluster_(std::move(cluster)), matrix_(std::move(matrix)), config_(std::move(config)) {
  if (!validate_matrix(matrix_, cluster_).ok) throw SpecError("cannot serve an invalid matrix");
  if (config_.input_width == 0) throw SpecError("input width must be positive");
  started_at_ = std::chrono::steady_clock::now();
  config_.pool.copy_outputs = true;
  init_thread_ = std::thread([this] { init_pool(); });
  dispatcher_ = std::thread([this] { dispatcher_loop(); });
}

PredictionService::~PredictionService() {
  stop();
  for (Arena& a : arena_)
    if (a.rows) cudaFreeHost(a.rows);
}

void PredictionService::init_pool() {
  try {
    system_ = std::make_unique<InferenceSystem>(matrix_, cluster_, config_.rule, config_.pool);
    // Pinned slots, streams and the host pool up front (and the input width
    // checked against the members), so the first flush pays none of it.
    system_->run_host_blocks({}, config_.input_width, nullptr, nullptr);
    if (config_.arena_rows > 0)
      for (Arena& a : arena_) {
        void* p = nullptr;
        // Portable: every GPU of a multi-GPU pool DMAs its rows from here.
        if (cudaHostAlloc(&p, config_.arena_rows * config_.input_width * 2, cudaHostAllocPortable) !=
            cudaSuccess) {
          cudaGetLastError();
          throw StartupError("cannot allocate the service's page-locked arenas");
        }
        a.rows = static_cast<std::uint16_t*>(p);
      }
    ready_.store(true);
  } catch (const std::exception& e) {
    std::lock_guard<std::mutex> lock(init_mutex_);
    init_error_ = e.what();
  }
  {
    std::lock_guard<std::mutex> lock(init_mutex_);
    init_done_ = true;
  }
  init_cv_.notify_all();
  buffer_cv_.notify_all();
}

bool PredictionService::wait_ready(std::chrono::milliseconds timeout) {
  std::unique_lock<std::mutex> lock(init_mutex_);
  init_cv_.wait_for(lock, timeout, [&] { return init_done_; });
  return ready_.load();
}

std::string PredictionService::startup_error() const {
  std::lock_guard<std::mutex> lock(init_mutex_);
  return init_error_;
}

std::future<RunOutput> PredictionService::submit(const float* samples, std::size_t rows) {
  auto p = std::make_shared<Pending>();
  std::future<RunOutput> fut = p->promise.get_future();
  if (rows == 0) {  // POST [] -> [] (server.cpp:124-127)
    RunOutput empty;
    empty.output_width = cluster_.models.empty() ? 0 : cluster_.models[0].output_width;
    p->promise.set_value(std::move(empty));
    return fut;
  }
  if (!ready_.load()) throw NotReadyError("service not ready");
  p->rows = rows;
  const std::size_t elems = rows * config_.input_width;
  if (arena_[0].rows) {
    // Reserve rows in the open arena (in buffer order), convert into them
    // outside the lock; the flush waits for the arena's writers.
    std::uint16_t* dst = nullptr;
    {
      std::lock_guard<std::mutex> lock(buffer_mutex_);
      if (stopping_.load()) throw NotReadyError("server shutting down");
      Arena& a = arena_[open_];
      if (a.used + rows <= config_.arena_rows) {
        dst = a.rows + a.used * config_.input_width;
        a.used += rows;
        ++a.writers;
        p->staged = dst;
        p->arena = open_;
        p->arrived = std::chrono::steady_clock::now();
        buffer_.push_back(p);
        buffered_samples_ += rows;
      }
    }
    if (dst) {
      convert_f32_to_bf16_range(samples, dst, elems);
      {
        std::lock_guard<std::mutex> lock(buffer_mutex_);
        --arena_[p->arena].writers;
      }
      buffer_cv_.notify_all();
      return fut;
    }
  }
  // The copy the request needs anyway doubles as the fp32 -> bf16 conversion
  // (on the caller's thread, so it scales with the clients), halving what the
  // flush gathers and sends over PCIe.
  // Arena full or too small for this request.
  p->bf16.resize(elems);
  convert_f32_to_bf16_range(samples, p->bf16.data(), elems);
  {
    std::lock_guard<std::mutex> lock(buffer_mutex_);
    // Checked under the buffer lock: the dispatcher fails whatever it finds
    // buffered after stopping_ flips, so an accepted request never hangs.
    if (stopping_.load()) throw NotReadyError("server shutting down");
    p->arrived = std::chrono::steady_clock::now();
    buffer_.push_back(p);
    buffered_samples_ += rows;
  }
  buffer_cv_.notify_all();
  return fut;
}

void PredictionService::flush_locked(std::unique_lock<std::mutex>& lock) {
  if (arena_[0].rows) {
    // Every reserved row of the open arena converted, then submits move to
    // the other arena (free: the previous flush from it has completed).
    buffer_cv_.wait(lock, [&] { return arena_[open_].writers == 0; });
    open_ ^= 1;
    arena_[open_].used = 0;
  }
  std::vector<std::shared_ptr<Pending>> batch(buffer_.begin(), buffer_.end());
  buffer_.clear();
  buffered_samples_ = 0;
  lock.unlock();
  std::size_t total = 0;
  for (const auto& r : batch) total += r->rows;
  try {
    RunOutput out;
    {
      std::vector<InferenceSystem::HostRowBlock> blocks;
      blocks.reserve(batch.size());
      for (const auto& r : batch) {
        const std::uint16_t* src = r->staged ? r->staged : r->bf16.data();
        InferenceSystem::HostRowBlock& last = blocks.empty() ? blocks.emplace_back() : blocks.back();
        if (r->staged && last.pinned && last.bf16 + last.rows * config_.input_width == src)
          last.rows += r->rows;  // consecutive arena rows: one page-locked block
        else if (blocks.size() == 1 && last.rows == 0)
          last = {src, r->rows, r->staged != nullptr};
        else
          blocks.push_back({src, r->rows, r->staged != nullptr});
      }
      const int C = cluster_.models[0].output_width;
      out.output_width = C;
      out.combined.resize(total * static_cast<std::size_t>(C));
      out.winners.resize(total);
      static_assert(sizeof(int) == sizeof(std::int32_t), "winners are int32 on the wire");
      out.stats.elapsed_s = system_->run_host_blocks(
          blocks, config_.input_width, out.combined.data(),
          reinterpret_cast<std::int32_t*>(out.winners.data()));
      out.stats.nb_samples = total;
      out.stats.segments = num_segments(total, cluster_.segment_size);
    }
    if (out.stats.elapsed_s > 0) last_flush_throughput_.store(total / out.stats.elapsed_s);
    samples_served_.fetch_add(total);
    flushes_.fetch_add(1);
    const std::size_t w = static_cast<std::size_t>(out.output_width);
    std::size_t row = 0;
    for (const auto& r : batch) {
      RunOutput piece;
      piece.output_width = out.output_width;
      piece.combined.assign(out.combined.begin() + row * w, out.combined.begin() + (row + r->rows) * w);
      if (!out.winners.empty())
        piece.winners.assign(out.winners.begin() + row, out.winners.begin() + row + r->rows);
      piece.stats = out.stats;
      r->promise.set_value(std::move(piece));
      requests_served_.fetch_add(1);
      row += r->rows;
    }
  } catch (...) {
    for (const auto& r : batch) r->promise.set_exception(std::current_exception());
  }
  lock.lock();
}

void PredictionService::dispatcher_loop() {
  std::unique_lock<std::mutex> lock(buffer_mutex_);
  while (!stopping_.load()) {
    if (buffer_.empty()) {
      buffer_cv_.wait(lock, [&] { return stopping_.load() || !buffer_.empty(); });
      continue;
    }
    const auto deadline = buffer_.front()->arrived + std::chrono::milliseconds(config_.flush_timeout_ms);
    const bool full = buffered_samples_ >= static_cast<std::size_t>(cluster_.segment_size);
    if (!full && std::chrono::steady_clock::now() < deadline) {
      buffer_cv_.wait_until(lock, deadline, [&] {
        return stopping_.load() ||
               buffered_samples_ >= static_cast<std::size_t>(cluster_.segment_size);
      });
      continue;
    }
    flush_locked(lock);
  }
  for (const auto& r : buffer_)  // so no client hangs
    r->promise.set_exception(std::make_exception_ptr(NotReadyError("server shutting down")));
  buffer_.clear();
  buffered_samples_ = 0;
}

ServiceStats PredictionService::stats() const {
  ServiceStats s;
  s.ready = ready_.load();
  s.requests_served = requests_served_.load();
  s.samples_served = samples_served_.load();
  s.flushes = flushes_.load();
  s.last_flush_throughput = last_flush_throughput_.load();
  {
    std::lock_guard<std::mutex> lock(buffer_mutex_);
    s.pending_requests = buffer_.size();
    s.pending_samples = buffered_samples_;
  }
  s.uptime_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - started_at_).count();
  return s;
}

void PredictionService::stop() {
  bool expected = false;
  if (!stopping_.compare_exchange_strong(expected, true)) return;
  ready_.store(false);
  { std::lock_guard<std::mutex> lock(buffer_mutex_); }  // no lost wake-up
  buffer_cv_.notify_all();
  if (dispatcher_.joinable()) dispatcher_.join();
  if (init_thread_.joinable()) init_thread_.join();
  {  // submits still converting into an arena finish before it can be freed
    std::unique_lock<std::mutex> lock(buffer_mutex_);
    buffer_cv_.wait(lock, [&] { return arena_[0].writers == 0 && arena_[1].writers == 0; });
  }
  if (system_) system_->shutdown();
}

}  // namespace enserve
