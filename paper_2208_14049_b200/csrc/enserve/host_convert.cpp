#include "enserve/host_convert.hpp"

#include <immintrin.h>

#include <algorithm>
#include <cstring>

namespace enserve {

ThreadPool::ThreadPool(int threads) {
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  for (int i = 0; i < threads; ++i) workers_.emplace_back([this, i] { loop(i); });
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> lock(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (std::thread& t : workers_) t.join();
}

void ThreadPool::run(const std::function<void(int, int)>& fn) {
  // One job at a time: a second caller (another thread sharing the pool)
  // waits here instead of overwriting job_/pending_ of the running one.
  std::lock_guard<std::mutex> serial(run_mu_);
  std::unique_lock<std::mutex> lock(mu_);
  job_ = &fn;
  pending_ = size();
  ++generation_;
  cv_.notify_all();
  done_cv_.wait(lock, [&] { return pending_ == 0; });
  job_ = nullptr;
}

void ThreadPool::loop(int index) {
  std::uint64_t seen = 0;
  for (;;) {
    const std::function<void(int, int)>* job;
    {
      std::unique_lock<std::mutex> lock(mu_);
      cv_.wait(lock, [&] { return stop_ || generation_ != seen; });
      if (stop_) return;
      seen = generation_;
      job = job_;
    }
    (*job)(index, size());
    {
      std::lock_guard<std::mutex> lock(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
}

namespace {

inline std::uint16_t bf16_rn(float f) {
  std::uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return static_cast<std::uint16_t>((u | 0x00400000u) >> 16);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<std::uint16_t>(u >> 16);
}

__attribute__((target("avx512f,avx512bf16"))) void convert_avx512bf16(const float* x,
                                                                      std::uint16_t* y,
                                                                      std::size_t n) {
  // Non-temporal stores once y is 64-byte aligned: the destination (a pinned
  // staging slot the DMA engine reads next) is not read for ownership first,
  // which saves a third of the host-memory traffic of a converted chunk.
  std::size_t i = 0;
  for (; i < n && (reinterpret_cast<std::uintptr_t>(y + i) & 63u); ++i) y[i] = bf16_rn(x[i]);
  const __m512i expo = _mm512_set1_epi32(0x7f800000), mant = _mm512_set1_epi32(0x007fffff);
  for (; i + 32 <= n; i += 32) {
    __m512 a = _mm512_loadu_ps(x + i);
    __m512 b = _mm512_loadu_ps(x + i + 16);
    // VCVTNE2PS2BF16 flushes fp32 subnormals to zero; bf16_rn (and the
    // device's __float2bfloat16_rn) keeps them as bf16 subnormals, so a
    // vector holding one takes the scalar rule.
    const __m512i ua = _mm512_castps_si512(a), ub = _mm512_castps_si512(b);
    const __mmask16 sa = _mm512_testn_epi32_mask(ua, expo) & _mm512_test_epi32_mask(ua, mant);
    const __mmask16 sb = _mm512_testn_epi32_mask(ub, expo) & _mm512_test_epi32_mask(ub, mant);
    if (sa | sb) {
      alignas(64) std::uint16_t tmp[32];
      for (int j = 0; j < 32; ++j) tmp[j] = bf16_rn(x[i + j]);
      _mm512_stream_si512(reinterpret_cast<__m512i*>(y + i), _mm512_load_si512(tmp));
      continue;
    }
    __m512bh p = _mm512_cvtne2ps_pbh(b, a);  // low half from a
    _mm512_stream_si512(reinterpret_cast<__m512i*>(y + i), reinterpret_cast<__m512i>(p));
  }
  _mm_sfence();
  for (; i < n; ++i) y[i] = bf16_rn(x[i]);
}

__attribute__((target("avx2"))) void convert_avx2(const float* x, std::uint16_t* y,
                                                  std::size_t n) {
  std::size_t i = 0;
  for (; i < n && (reinterpret_cast<std::uintptr_t>(y + i) & 15u); ++i) y[i] = bf16_rn(x[i]);
  const __m256i one = _mm256_set1_epi32(1), bias = _mm256_set1_epi32(0x7fff);
  for (; i + 8 <= n; i += 8) {
    __m256i u = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(x + i));
    // NaN inputs take the scalar path's quiet-NaN rule below
    const __m256i expo = _mm256_and_si256(u, _mm256_set1_epi32(0x7f800000));
    if (!_mm256_testz_si256(_mm256_cmpeq_epi32(expo, _mm256_set1_epi32(0x7f800000)),
                            _mm256_set1_epi32(-1))) {
      for (std::size_t j = i; j < i + 8; ++j) y[j] = bf16_rn(x[j]);
      continue;
    }
    __m256i lsb = _mm256_and_si256(_mm256_srli_epi32(u, 16), one);
    __m256i r = _mm256_srli_epi32(_mm256_add_epi32(_mm256_add_epi32(u, bias), lsb), 16);
    // pack 8 x u32 (values < 2^16) into 8 x u16
    __m128i lo = _mm256_castsi256_si128(r), hi = _mm256_extracti128_si256(r, 1);
    _mm_stream_si128(reinterpret_cast<__m128i*>(y + i), _mm_packus_epi32(lo, hi));  // see above
  }
  _mm_sfence();
  for (; i < n; ++i) y[i] = bf16_rn(x[i]);
}

bool has_avx512bf16() {
  static const bool yes = __builtin_cpu_supports("avx512bf16");
  return yes;
}

}  // namespace

void convert_f32_to_bf16_range(const float* x, std::uint16_t* y, std::size_t n) {
  if (has_avx512bf16())
    convert_avx512bf16(x, y, n);
  else if (__builtin_cpu_supports("avx2"))
    convert_avx2(x, y, n);
  else
    for (std::size_t i = 0; i < n; ++i) y[i] = bf16_rn(x[i]);
}

void convert_f32_to_bf16_host(const float* x, std::uint16_t* y, std::size_t n, ThreadPool& pool) {
  const std::function<void(int, int)> job = [&](int part, int parts) {
    const std::size_t per = ((n + parts - 1) / parts + 63) / 64 * 64;  // > 0 for any n
    const std::size_t a = std::min(n, static_cast<std::size_t>(part) * per);
    const std::size_t b = std::min(n, a + per);
    if (b > a) convert_f32_to_bf16_range(x + a, y + a, b - a);
  };
  pool.run(job);
}

}  // namespace enserve
