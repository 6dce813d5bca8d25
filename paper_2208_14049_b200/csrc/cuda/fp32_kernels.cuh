// FP32-accurate member path (PoolOptions::fp32; north_star: logits and
// averaged probabilities within 1e-5 for fp32).  X, weights, activations and
// accumulation all stay fp32 and run on the CUDA cores: the tensor cores
// have no fp32 operand format, and TF32 (10-bit mantissa) would not hold
// 1e-5.  Same weights (the generator of generate_dense_layer_f32 = the
// oracle's orc_weight / orc_bias unrounded), same layer order and
// layouts as the bf16 kernels, so a member's fp32 logits are comparable
// row for row with the oracle's quantize_bf16 = 0 member.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "batching.cuh"

namespace es {

// y[r][n] = act(sum_k x[r][k] * w[n][k] + b[n]) for rows [row_begin, row_end)
// (or the claim's rows), x [rows][K] and y [rows][N] fp32, rows indexed
// globally.  act = ReLU when relu, else identity (logits).
struct F32DenseArgs {
  const float* x = nullptr;
  const float* w = nullptr;  // [N][K]
  const float* b = nullptr;  // [N]
  float* y = nullptr;
  int K = 0, N = 0;
  bool relu = true;
  long long row_begin = 0, row_end = 0;
  const ClaimedRun* claim = nullptr;
};
int f32_dense_launch(const F32DenseArgs& a, int grid, cudaStream_t s);

// The CNN member's convolution stack in fp32: x [rows][S*S] (one channel),
// conv P x P stride P -> c1 (+b1, ReLU), conv 3 x 3 pad 1 -> c2 (+b2, ReLU),
// out [rows][G*G*c2] in HWC order (the head's K index (h*G + w)*c2 + channel).
// w1 [c1][P*P] (K index a*P + b), w2 [c2][9*c1] (K index tap*c1 + channel,
// tap = 3*(dh+1) + (dw+1)) -- the layouts of conv_kernel.cuh / the oracle.
struct F32ConvArgs {
  const float* x = nullptr;
  const float* w1 = nullptr;
  const float* b1 = nullptr;
  const float* w2 = nullptr;
  const float* b2 = nullptr;
  float* out = nullptr;
  int S = 0, P = 0, c1 = 0, c2 = 0;
  long long row_begin = 0, row_end = 0;
  const ClaimedRun* claim = nullptr;
};
// False when a sample's grids do not fit shared memory.
bool f32_conv_supported(int S, int P, int c1, int c2);
int f32_conv_launch(const F32ConvArgs& a, int grid, cudaStream_t s);

// Synthetic features in fp32: x[i] = U24(splitmix64(seed * 0x2545f4914f6cdd1d + i))
// exactly (the bf16 replica rounds the same values).
int generate_features_f32(uint64_t seed, size_t n, float* y, cudaStream_t s);

}  // namespace es
