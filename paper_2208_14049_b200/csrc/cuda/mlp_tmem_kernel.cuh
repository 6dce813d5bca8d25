// K1 v2 — fused two-layer MLP member with the hidden layer kept in TMEM.
//
// Same contract as mlp_kernel.cuh (Predictor::predict,
// /root/reference/proj/include/enserve/runtime/backend.hpp:33), different
// schedule, chosen to cut per-SM TMA ingress (the measured limiter: <= 48 B/clk
// per SM from L2, profiles/r1_summary.md):
//
//   layer 1 (samples on M):  D1[s, h] = sum_k X[s, k] W1[h, k]
//                            UMMA M = 128 samples (one tile = b rows of a
//                            segment), N = H split in <= 256-wide halves,
//                            K in 64-wide TMA chunks.  T tiles share every W1
//                            chunk they stream (T*H <= 512 TMEM columns), so W1
//                            ingress per sample drops by T.
//   epilogue 1 (8 warps):    tcgen05.ld fp32 D1 -> +b1, ReLU, bf16x2 ->
//                            tcgen05.st back into the SAME TMEM columns (each
//                            warp overwrites only columns it has already read).
//   layer 2:                 D2[s, c] = sum_h H[s, h] W2[c, h] with the A
//                            operand read straight from TMEM (no smem round
//                            trip), B = W2 resident in smem, N = 16.
//   epilogue 2:              tcgen05.ld D2 -> +b2 -> fp32 logits.
// Warp roles: w0 TMA, w1 TMEM alloc + single-thread UMMA issue, w2..w9
// epilogue (w%4 = TMEM lane quadrant, (w-2)/4 = which half of the hidden
// columns).
#pragma once

#include <cstdint>

#include "batching.cuh"
#include "sm100.cuh"

namespace es {

struct MlpTLayout {
  int H = 0, C = 0, K = 0, kchunks = 0;
  int T = 1;          // 128-row tiles per group (share each W1 chunk)
  int nbuf = 1;       // TMEM group buffers
  int nh = 1;         // layer-1 UMMAs per tile per k-step
  int NH = 0;         // their N (H / nh)
  int stages = 0;
  int group_cols = 0; // T * H
  int d2_sep = 0;     // layer-2 accumulators outside the hidden columns
  int d2_col = 0;     //   (then at d2_col + 16 * d2_parts * k, so the next
                      //    group's layer 1 is not gated by the logits epilogue)
  int d2_parts = 1;   // independent layer-2 partial accumulators (16 columns each)
  int tmem_cols = 0;
  uint32_t stage_bytes = 0;  // T * 16 KB (X tiles) + H * 128 (W1 chunk)
  uint32_t off_w2 = 0, off_bias = 0, off_bar = 0, smem_bytes = 0;
  float est_cycles_per_sample = 0.0f;
};

struct MlpTArgs {
  MlpTLayout L;
  int b = 0;
  int seg_size = 0;
  long long seg_begin = 0, seg_end = 0, nb = 0;
  const float* bias1 = nullptr;
  const float* bias2 = nullptr;
  float* out = nullptr;
  // Dynamic claim (batching.cuh ClaimedRun): when set, the launch walks the
  // segments stored there instead of [seg_begin, seg_end).
  const ClaimedRun* claim = nullptr;
};

bool mlpt_plan(int K, int H, int C, int b, MlpTLayout* out);
int mlpt_launch(const MlpTArgs& args, const void* x, const void* w1, const void* w2, int grid,
                cudaStream_t stream);

}  // namespace es
