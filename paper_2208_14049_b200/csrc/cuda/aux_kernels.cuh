// Device helpers around the member kernel: X fp32 -> bf16 staging, synthetic
// weight generation, and K3 — the fused combination kernel.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "batching.cuh"

namespace es {

// y[i] = bf16_rn(x[i]).
int convert_f32_to_bf16(const float* x, __nv_bfloat16* y, size_t n, cudaStream_t s);

// Synthetic Glorot-uniform weights of dense layer `layer`:
// w[o][i] = bf16_rn((2u-1) * limit), b[o] = (2u'-1) * 0.01, u from splitmix64 of
// (seed, layer, element).  `limit` = (float)sqrt(6/(fan_in+fan_out)).
int generate_dense_layer(uint64_t seed, int layer, int fan_in, int fan_out, float limit,
                         __nv_bfloat16* w, float* b, cudaStream_t s);
// Same values, fp32 (for host-supplied-vs-synthetic checks).
int generate_dense_layer_f32(uint64_t seed, int layer, int fan_in, int fan_out, float limit,
                             float* w, float* b, cudaStream_t s);

enum CombineRule : int { kAverage = 0, kVote = 1, kWeighted = 2 };

constexpr int kMaxMembers = 32;
constexpr int kMaxClasses = 16;

struct CombineArgs {
  const float* logits[kMaxMembers];  // [rows][C] per member, model-id order
  float weight[kMaxMembers];         // per-member fold factor (avg: 1/M; wavg: w_m)
  int M = 0;
  int C = 0;
  int rule = kAverage;
  int softmax = 0;                   // fold softmax(z) instead of z
  long long rows = 0;
  float* y = nullptr;                // [rows][C]
  int32_t* argmax = nullptr;         // [rows] (may be null)
};

// K3: one pass over every member's logits; per row: optional softmax, fold in
// model-id order with separately rounded multiply and add (bit-identical to
// PredictionAccumulator::fold_segment, combine.cpp:99-135), lowest-index argmax.
int combine_launch(const CombineArgs& a, cudaStream_t s);

// Synthetic member: out[r][c] = synthetic_prediction(model_id, r, c) for rows
// of the segments [seg_begin, seg_end) (reference src/runtime/backend.cpp:21-29).
// claim (may be null): rows of a data-parallel worker's claimed run instead.
int synthetic_member_launch(int model_id, int C, int seg_size, long long seg_begin,
                            long long seg_end, long long nb, float* out, cudaStream_t s,
                            const ClaimedRun* claim = nullptr);

// Device FIFO of a data-parallel model (the reference's
// shared per-model segment queue, pipeline.cpp:44-51, :103-104): pop the next
// `chunk` segments of [0, segments) off *counter (atomicAdd; the counter may
// live on a peer GPU), store the run and its rows [.., min(end * seg_size, nb))
// in *out for the worker's member launches, and stamp owner[s] = worker for
// every popped segment (exactly-once evidence; may be null).  An exhausted
// queue stores an empty run.
int claim_launch(unsigned long long* counter, long long segments, long long chunk, int seg_size,
                 long long nb, ClaimedRun* out, int* owner, int worker, cudaStream_t s);

// Synthetic features straight into the bf16 device replica:
// x[i] = bf16_rn(U24(splitmix64(seed * 0x2545f4914f6cdd1d + i))).
int generate_features_bf16(uint64_t seed, size_t n, __nv_bfloat16* y, cudaStream_t s);

// SIMT (CUDA-core) two-layer MLP used only as a device-side cross-check of the
// tensor-core kernel in tests (selected with ES_MEMBER_KERNEL=simt).
int mlp2_simt_launch(const __nv_bfloat16* x, long long nb, int K, const __nv_bfloat16* w1,
                     const float* b1, int H, const __nv_bfloat16* w2, const float* b2, int C,
                     long long row_begin, long long row_end, float* out, cudaStream_t s);

}  // namespace es
