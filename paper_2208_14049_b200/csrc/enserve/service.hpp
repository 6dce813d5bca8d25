// Deploy-mode prediction service (the serving core of the
// reference's PredictionServer, src/server/server.cpp:65-288, without the
// HTTP wiring): client requests are buffered and flushed into ONE device
// run per batch -- when a full segment is waiting, or when the oldest request
// has waited flush_timeout_ms (server.cpp:227-273) -- and every request gets
// exactly its own rows of the combined output back.
#pragma once

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <future>
#include <memory>
#include <mutex>
#include <string>
#include <thread>

#include "enserve/runtime.hpp"

namespace enserve {

struct ServiceConfig {  // ServeConfig (server.hpp:19-26), minus bind host / port / backend
  int flush_timeout_ms = 50;
  std::size_t input_width = 16;
  CombinationRule rule = CombinationRule::averaging();
  PoolOptions pool;
  // One-GPU pools: rows per page-locked arena (two: one filling while the
  // other flushes).  Requests are converted to bf16 straight into the open
  // arena by the submitting thread and DMA'd from there; 0 = no arenas.
  // 262144 rows of 784 features = 2 x 411 MB page-locked (profiles/
  // r1j_service_load.md: requests that overflow an arena take the gather path).
  std::size_t arena_rows = 262144;
};

struct ServiceStats {  // GET /v1/stats (server.cpp:88-107)
  bool ready = false;
  std::uint64_t requests_served = 0;
  std::uint64_t samples_served = 0;
  std::uint64_t flushes = 0;
  double last_flush_throughput = 0.0;  // samples/s of the last flush's device window
  std::size_t pending_requests = 0;
  std::size_t pending_samples = 0;
  double uptime_s = 0.0;
};

class PredictionService {
 public:
  // Throws SpecError for an invalid matrix (server.cpp:30-31); the device pool
  // is built on a background thread (init_pool, server.cpp:37-52).
  PredictionService(ClusterSpec cluster, AllocationMatrix matrix, ServiceConfig config);
  ~PredictionService();
  PredictionService(const PredictionService&) = delete;
  PredictionService& operator=(const PredictionService&) = delete;

  bool wait_ready(std::chrono::milliseconds timeout);
  bool ready() const { return ready_.load(); }
  std::string startup_error() const;

  // POST /v1/predict: `rows` samples of input_width features (copied).  The
  // future carries this request's rows only (combined + winners).  Throws
  // NotReadyError (the reference's 503) before the pool is up or after stop();
  // the future throws NotReadyError if the service stops before its flush.
  std::future<RunOutput> submit(const float* samples, std::size_t rows);

  ServiceStats stats() const;
  void stop();  // fails whatever is still buffered ("server shutting down")

 private:
  struct Pending {
    std::vector<std::uint16_t> bf16;     // one-GPU pools: rows converted by the caller
    const std::uint16_t* staged = nullptr;  // ... or their place in a pinned arena
    int arena = -1;
    std::size_t rows = 0;
    std::chrono::steady_clock::time_point arrived;
    std::promise<RunOutput> promise;
  };
  void init_pool();
  void dispatcher_loop();
  void flush_locked(std::unique_lock<std::mutex>& lock);

  ClusterSpec cluster_;
  AllocationMatrix matrix_;
  ServiceConfig config_;
  std::unique_ptr<InferenceSystem> system_;
  std::atomic<bool> ready_{false};
  struct Arena {
    std::uint16_t* rows = nullptr;  // page-locked, arena_rows x input_width bf16
    std::size_t used = 0;           // rows handed out
    int writers = 0;                // submits still converting into it
  };
  Arena arena_[2];
  int open_ = 0;  // the arena submits fill; the other one is flushed
  std::atomic<bool> stopping_{false};
  mutable std::mutex init_mutex_;
  std::condition_variable init_cv_;
  bool init_done_ = false;
  std::string init_error_;
  mutable std::mutex buffer_mutex_;
  std::condition_variable buffer_cv_;
  std::deque<std::shared_ptr<Pending>> buffer_;
  std::size_t buffered_samples_ = 0;
  std::atomic<std::uint64_t> requests_served_{0}, samples_served_{0}, flushes_{0};
  std::atomic<double> last_flush_throughput_{0.0};
  std::chrono::steady_clock::time_point started_at_;
  std::thread init_thread_, dispatcher_;
};

}  // namespace enserve
