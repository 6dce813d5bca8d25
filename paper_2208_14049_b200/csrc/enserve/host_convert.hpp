// Host side of the end-to-end path: a small fixed thread pool and a
// multi-threaded fp32 -> bf16 (round-to-nearest-even) converter, so the
// host->device copy carries 2 bytes per feature instead of 4.  The bits equal
// the device converter's (__float2bfloat16_rn) for every finite input.
#pragma once

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace enserve {

class ThreadPool {
 public:
  explicit ThreadPool(int threads = 0);
  ~ThreadPool();
  ThreadPool(const ThreadPool&) = delete;
  ThreadPool& operator=(const ThreadPool&) = delete;

  int size() const { return static_cast<int>(workers_.size()); }
  // fn(part, parts) on every worker; returns when all parts are done.
  void run(const std::function<void(int, int)>& fn);

 private:
  void loop(int index);
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::mutex run_mu_;  // serialises run() across callers
  std::condition_variable cv_, done_cv_;
  const std::function<void(int, int)>* job_ = nullptr;
  std::uint64_t generation_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

// y[i] = bf16_rn(x[i]) for i in [0, n), split over the pool.
void convert_f32_to_bf16_host(const float* x, std::uint16_t* y, std::size_t n, ThreadPool& pool);

// Single-threaded kernel of the above (exposed for tests).
void convert_f32_to_bf16_range(const float* x, std::uint16_t* y, std::size_t n);

}  // namespace enserve
