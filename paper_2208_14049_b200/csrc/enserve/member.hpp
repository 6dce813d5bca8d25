// One ensemble member resident on one GPU: the device side of the reference's
// Predictor (/root/reference/proj/include/enserve/runtime/backend.hpp:25-34).
//
//   * Synthetic: synthetic_prediction(model, sample, class), the reference's
//     deterministic stand-in (src/runtime/backend.cpp:21-29).
//   * MLP widths[0] -> ... -> widths[L]: the first L-2 layers run as tcgen05
//     dense layers (bias + ReLU fused, bf16 activations in HBM), the last two
//     as one fused member kernel (hidden layer never leaves the SM): the
//     SM-pair schedule for hidden >= 512, the single-SM TMEM schedule below,
//     the swap-AB schedule when neither fits.
//   * fp32 (load(..., fp32 = true)): the same layers with fp32 X, weights,
//     activations and accumulation on the CUDA cores (cuda/fp32_kernels.cuh),
//     for the 1e-5 fp32 parity mode; forward() then reads an fp32 X.
#pragma once

#include <cuda_runtime.h>

#include "../cuda/batching.cuh"

#include <cstddef>
#include <string>
#include <vector>

#include "enserve/spec.hpp"

namespace enserve {

class DeviceMember {
 public:
  DeviceMember() = default;
  ~DeviceMember();
  DeviceMember(const DeviceMember&) = delete;
  DeviceMember& operator=(const DeviceMember&) = delete;

  // Predictor::load(): false = out of memory (a tile plan does not fit an SM,
  // or a device allocation failed); other failures throw.
  bool load(int device, const ModelSpec& model, int batch, bool fp32 = false);
  bool fp32() const;

  // Logits of every row of segments [s0, s1) of x (bf16 [nb][width], rows
  // indexed globally) into out ([nb][C] fp32).  Returns kernel launches.
  // `marks` (optional, >= max_launches() events): marks[i] is recorded on
  // `stream` right after launch i, so launch i's device time is the interval
  // from the previous mark (or the caller's start event) to marks[i].
  // `claim` (optional, device memory): a data-parallel worker's claimed run
  // (cuda/batching.cuh ClaimedRun, written by es::claim_launch earlier on
  // `stream`); every launch then walks the rows stored there, and [s0, s1)
  // only bounds the grid.
  int forward(const void* x, long long nb, int seg_size, long long s0, long long s1, float* out,
              int grid, cudaStream_t stream, const cudaEvent_t* marks = nullptr,
              const es::ClaimedRun* claim = nullptr);
  // Whether every launch of this member honours a claim (the swap-AB and
  // SIMT schedules do not; their workers keep the static split).
  bool supports_claim() const;

  // Kernel names forward() launches, in order (one per launch).
  std::vector<std::string> kernel_names() const;
  int max_launches() const { return static_cast<int>(kernel_names().size()); }

  int device() const { return device_; }
  std::size_t weight_bytes() const { return bytes_; }
  // Name of the fused head schedule ("pair", "tmem", "swapab", "synthetic").
  std::string schedule() const;

 private:
  struct Impl;
  Impl* impl_ = nullptr;
  int device_ = 0;
  std::size_t bytes_ = 0;
  bool load_fp32(int device);
  int forward_fp32(const float* x, long long nb, long long r0, long long r1, float* out, int grid,
                   cudaStream_t stream, const cudaEvent_t* marks, const es::ClaimedRun* claim);
};

}  // namespace enserve
