// Dense layer on sm_100a tensor cores: Y = act(X . W^T + b), bf16 in, bf16 out.
//
// Building block for members deeper than the fused two-layer kernel: an MLP
// 784-512-512-10 runs as dense(784->512, ReLU) followed by the fused
// member_mlp2 kernel on the 512-wide activations; the CNN member's convolution
// stack feeds the same fused head.  Activations between launches live in HBM
// as bf16 [rows][N] (row stride N).  Members wider than the fused head's
// 512-column TMEM budget run their hidden layers here and the last layer in
// logits mode (N = 16, fp32 out).
//   UMMA M = 128 rows, N <= 256 per instruction (up to 512 per tile, wider
//   layers in column blocks), K in 64-wide TMA chunks; T tiles share each W
//   chunk; fp32 accumulators in TMEM;
//   epilogue: tcgen05.ld -> +b, ReLU, bf16 -> 128B-swizzled smem staging ->
//   TMA bulk tensor store (one 64-column box per chunk and column half).
#pragma once

#include <cstdint>

#include "batching.cuh"
#include "sm100.cuh"

namespace es {

struct DenseLayout {
  int K = 0, N = 0, kchunks = 0;  // N: columns per block (<= 512)
  int N_total = 0, ncb = 1;       // all output columns, column blocks
  int logits = 0, C = 0;          // final-layer mode: fp32 logits, C <= 16 columns
  int T = 1, nbuf = 1, nh = 1, NH = 0;
  int relu = 1;
  int pair = 0;                   // dense_pair_sm100 layout (SM pairs, cta_group::2)
  int stages = 0, group_cols = 0, tmem_cols = 0;
  uint32_t stage_bytes = 0, off_stage_out = 0, off_bias = 0, off_bar = 0, smem_bytes = 0;
};

struct DenseArgs {
  DenseLayout L;
  long long row_begin = 0, row_end = 0;  // rows of X / Y handled by this launch
  const ClaimedRun* claim = nullptr;      // set: the rows stored there instead
  const float* bias = nullptr;
  float* logits = nullptr;  // logits mode: fp32 [rows][C]
};

// Hidden layer: output width N a multiple of 128 (blocks of up to 512 columns).
bool dense_plan(int K, int N, bool relu, DenseLayout* out);
// Final layer of a member too wide for the fused head: C <= 16 logits.
bool dense_logits_plan(int K, int C, DenseLayout* out);
// x: bf16 [rows >= row_end][K]; w: bf16 [N][K]; y: bf16 [rows][N] (unused in
// logits mode, which writes args.logits).
int dense_launch(const DenseArgs& args, const void* x, long long x_rows, const void* w, void* y,
                 int grid, cudaStream_t stream);

// The same hidden layer on SM pairs (dense_pair_kernel.cu): each SM of a
// 2-CTA cluster streams half of every W chunk.  N a multiple of 128.
bool dense_pair_plan(int K, int N, bool relu, DenseLayout* out);
int dense_pair_launch(const DenseArgs& args, const void* x, long long x_rows, const void* w, void* y,
                      int grid, cudaStream_t stream);

}  // namespace es
