// K1 v3 — fused two-layer MLP member on SM PAIRS (tcgen05 cta_group::2).
//
// The TMEM-resident schedule of mlp_tmem_kernel.cuh, issued by the even CTA of
// a 2-CTA cluster for both SMs at once: UMMA M = 256 samples (128 on each SM),
// so each SM streams only HALF of every W1 chunk (B operand split by N across
// the pair).  Per-SM TMA ingress at full tensor rate drops from
// 8192/H + 64/T to 8192/H + 32/T bytes per clock — 48 B/clk for H = 512,
// i.e. the measured TMA ceiling (profiles/r1_summary.md).
//   layer 1:   D1[s, h] += X[s, k] W1[h, k]      cta_group::2, M=256, N<=256
//   epilogue:  each SM turns its own 128 rows to bf16 in its own TMEM
//   layer 2:   D2[s, c] = H[s, h] W2[c, h]       cta_group::2, A from TMEM of
//              both SMs, W2 rows split 8 + 8 across the pair (N = 16)
// Hidden layers wider than 512 (one SM's TMEM) run in passes of HP <= 512
// units: every pass re-streams the tile's X chunks with the next W1 rows, its
// layer-2 partial (W2 columns of the pass) is read out by the epilogue and
// summed in registers; logits are written after the last pass.
// Barriers the leader's UMMA thread waits on (full, a_full, acc_empty, w2_full)
// live in the leader; the peer's TMA completes bytes on them directly and its
// epilogue arrives remotely.  Commits multicast to both SMs.
#pragma once

#include <cstdint>

#include "batching.cuh"
#include "sm100.cuh"

namespace es {

struct MlpPLayout {
  int H = 0, C = 0, K = 0, kchunks = 0;
  int HP = 0;         // hidden units per pass (H / passes <= 512: one SM's TMEM)
  int passes = 1;     // hidden passes; each re-streams X, layer-2 partials summed
  int T = 1;          // 128-row tiles per SM per group
  int nbuf = 1;
  int nh = 1;         // pair UMMAs per tile per k-step
  int NH = 0;         // their N (each SM holds NH/2 rows of the W1 chunk)
  int stages = 0;
  int group_cols = 0;
  int d2_sep = 0;     // layer-2 accumulators outside the hidden columns
  int d2_col = 0;     //   (see mlp_tmem_kernel.cuh)
  int d2_parts = 1;   // independent layer-2 partial accumulators (16 columns each)
  int tmem_cols = 0;
  uint32_t stage_bytes = 0;  // T * 16 KB + H * 64 (half of the W1 chunk)
  uint32_t off_w2 = 0, off_bias = 0, off_bar = 0, smem_bytes = 0;
  float est_cycles_per_sample = 0.0f;
};

struct MlpPArgs {
  MlpPLayout L;
  int b = 0;
  int seg_size = 0;
  long long seg_begin = 0, seg_end = 0, nb = 0;
  const float* bias1 = nullptr;
  const float* bias2 = nullptr;
  float* out = nullptr;
  // Dynamic claim (batching.cuh ClaimedRun): when set, the launch walks the
  // segments stored there instead of [seg_begin, seg_end).
  const ClaimedRun* claim = nullptr;
  // Optional timeline of CTA 0 (globaltimer ns): [group][8] for groups < 32,
  // see the TRACE() points in the kernel.  nullptr = off.
  unsigned long long* trace = nullptr;
};

bool mlpp_plan(int K, int H, int C, int b, MlpPLayout* out);
int mlpp_launch(const MlpPArgs& args, const void* x, const void* w1, const void* w2, int grid,
                cudaStream_t stream);

}  // namespace es
