// K1 — fused two-layer MLP member forward on sm_100a tensor cores.
//
// Replaces the body of Predictor::predict
// (/root/reference/proj/include/enserve/runtime/backend.hpp:33; the reference's
// only implementations sleep or emit hashes, src/runtime/backend.cpp:43-69).
//
//   logits[r, :] = W2 . relu(W1 . x_r + b1) + b2        for every row r of a tile
//
// Work decomposition: one persistent CTA per SM walks the
// worker's tiles — a tile is `b` consecutive samples of one segment, exactly the
// reference batcher's split (src/runtime/pipeline.cpp:155-162).
//   layer 1 (swap-AB):  D1[h, s] = sum_k W1[h, k] * X[s, k]
//                       UMMA M = 128 hidden units per chunk, N = tile width
//                       (b rounded up to 16), K streamed in 64-wide chunks by
//                       TMA (SW128) through a `stages`-deep mbarrier ring.
//   epilogue 1:         TMEM -> regs, +b1, ReLU, bf16, scattered into a K-major
//                       SW128 smem tile Hs[s, h] (never leaves the SM).
//   layer 2:            D2[s, c] = sum_h Hs[s, h] * W2[c, h]
//                       UMMA M = 128 sample rows, N = 16 (C <= 16, zero-padded
//                       by TMA OOB fill), accumulated into the first 16 columns
//                       of the tile's own (already drained) layer-1 TMEM buffer.
//   epilogue 2:         TMEM -> regs, +b2, fp32 logits to HBM at the tile's row.
// Warp roles: w0 TMA producer, w1 TMEM allocator + single-thread UMMA issuer,
// w2..w5 epilogue (each owns the 32 TMEM lanes of its quadrant w%4).
#pragma once

#include <cstdint>

#include "sm100.cuh"

namespace es {

struct Mlp2Layout {
  int H = 0;         // hidden width, multiple of 128, <= 512
  int N = 0;         // tile width (UMMA N for layer 1), multiple of 16, <= 256
  int C = 0;         // classes, <= 16
  int K = 0;         // input width
  int kchunks = 0;   // ceil(K / 64)
  int stages = 0;
  int nbuf = 0;      // TMEM accumulator buffers (1 or 2)
  int buf_cols = 0;  // TMEM columns per buffer: (H/128) * N
  int tmem_cols = 0; // allocated columns (power of two >= 32)
  uint32_t h_chunk_stride = 0;  // bytes between 64-wide K chunks of Hs (= N*128)
  uint32_t off_w2 = 0;
  uint32_t off_stage = 0;
  uint32_t x_bytes = 0;         // N * 128
  uint32_t stage_bytes = 0;     // (N + H) * 128
  uint32_t off_bar = 0;
  uint32_t smem_bytes = 0;      // dynamic smem to request (incl. 1 KB alignment slack)
};

struct Mlp2Args {
  Mlp2Layout L;
  int b = 0;                 // valid samples per tile (the worker's batch)
  int seg_size = 0;          // ClusterSpec::segment_size
  long long seg_begin = 0;   // segments [seg_begin, seg_end) handled by this launch
  long long seg_end = 0;
  long long nb = 0;          // samples in the store
  const float* bias1 = nullptr;  // [H]
  const float* bias2 = nullptr;  // [C]
  float* out = nullptr;          // logits [nb][C]
};

// Host: choose stages / buffers for (H, b); returns false if the tile does not
// fit one SM (227 KB smem, 512 TMEM columns) — the caller maps that to an
// out-of-memory load(), as the reference does for an over-committed worker.
bool mlp2_plan(int K, int H, int C, int b, Mlp2Layout* out);

// Host: launch over segments [seg_begin, seg_end) on `stream`.
// x: bf16 [nb][K] device, w1: bf16 [H][K], w2: bf16 [C][H].
int mlp2_launch(const Mlp2Args& args, const void* x, const void* w1, const void* w2, int grid,
                cudaStream_t stream);

int num_sms(int device);

}  // namespace es
