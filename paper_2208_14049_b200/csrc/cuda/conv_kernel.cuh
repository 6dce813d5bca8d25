// Convolution stack of the CNN member on sm_100a tensor cores.
//
//   x [S*S] (one channel)  --conv P x P, stride P, c1 filters, +b, ReLU-->
//   a1 [G][G][c1]          --conv 3 x 3, pad 1, c2 filters, +b, ReLU-->
//   a2 [G][G][c2] (bf16, HWC order: the fused member_mlp2 head's input row)
//
// Both convolutions are implicit GEMMs on tcgen05 inside ONE persistent kernel;
// the c1-channel intermediate never leaves shared memory:
//   * a tile is T whole samples, so no halo crosses tiles;
//   * conv1: TMA brings the raw images; the TMA warp also writes the im2col
//     rows (one row per output pixel, K = P*P) into a K-major planar operand;
//     one UMMA (M=128, N=c1, K=16) per 128 rows;
//   * conv1's epilogue writes relu(acc+b) as bf16 into a zero-bordered grid,
//     again K-major planar (channels = K).  Grid rows have stride R = G+1 and
//     samples stride R*R: pixel (h, w), 1 <= h <= G, 0 <= w < G, sits at row
//     s*R*R + h*R + w, and row 0 / column G of each sample are zero -- the
//     left neighbour of column 0 is the previous row's column G and the
//     bottom neighbour of row G is the next sample's row 0, so ONE shared
//     border serves both sides (49 of 64 rows useful at G = 7, 2 samples per
//     M block);
//   * conv2: output pixel q at tap (dh, dw) reads grid row q + dh*R + dw, so
//     each of the 9 taps is the SAME operand with the descriptor start moved
//     by whole rows (16 B each) -- nine accumulating UMMAs per K step, no
//     im2col copy, no re-read from memory;
//   * conv2's epilogue keeps the G x G interior and stores bf16 rows to HBM.
// Every operand is K-major without swizzle (sdesc_planar in sm100.cuh).
//
// conv2 schedules.  A tcgen05 M=128, K=16 UMMA costs max(~46, N/2) clk
// whatever its operands (tools/umma_rate.cu, measured on B200), so c2 = 32
// output channels as N runs the tensor core at 16/46 of its rate:
//   * "tap" (any shape): 9 taps x c1/16 K steps of N = c2 per 128-row block;
//   * "split" (3*c2 <= 256, R | 32): the three HORIZONTAL taps dw = -1, 0, +1
//     of one vertical offset dh go into ONE UMMA as N = 3*c2 columns (B rows
//     dw*c2 + o), with A shifted by dh*R - 1 only: 3 x c1/16 UMMAs of N = 96
//     per block instead of 36 of N = 32.  Column group dw of accumulator row
//     p then holds D'[p][dw] = sum_dh X[p - 1 + dh*R] W(dh, dw), and
//         out[q] = D'[q][-1] + D'[q+1][0] + D'[q+2][+1],
//     a lane shift within each 32-lane quadrant (ConvArgs::shifts: by
//     tcgen05.shift in the tensor pipe, by warp shuffles in the epilogue
//     warp that reads the quadrant, or split between the two).  With the
//     grid's border column LAST in a row (w = G), a quadrant's lane 31 is a
//     border pixel and lane 30's missing dw=+1 partial (lane 32's) reads only
//     the border column, i.e. is zero.  The default where the shape allows
//     it (measured faster than tap, conv_plan).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "batching.cuh"

namespace es {

struct ConvLayout {
  int S = 28, P = 4, G = 7, c1 = 64, c2 = 32;
  int R = 8;             // G + 1: grid row stride (shared zero border)
  bool split = false;    // conv2 schedule (see above)
  int n2 = 32;           // conv2 UMMA N: c2 (tap) or 3*c2 (split)
  int T = 4;             // samples per tile
  int mb1 = 2, mb2 = 2;  // 128-row M blocks of conv1 / conv2
  int raw_stages = 4;
  uint32_t raw_stride = 0;                     // bytes per raw image stage
  uint32_t a1_plane = 0, a1_bytes = 0;         // conv1 operand: [2 planes][mb1*128][16 B]
  uint32_t a2_rows = 0, a2_plane = 0, a2_bytes = 0;  // [c1/8 planes][a2_rows][16 B]
  uint32_t off_raw = 0, off_a1 = 0, off_a2 = 0, off_w1 = 0, off_w2 = 0, off_b1 = 0, off_b2 = 0;
  uint32_t off_bar = 0, smem_bytes = 0;
  int tmem_c1 = 0, tmem_c2 = 0, tmem_cols = 0;  // columns per buffer, total allocation
  uint32_t off_rows = 0;  // im2col source offset per tile row, int [T*G*G]
  uint32_t off_xch = 0;  // split: boundary-row exchange, [2][4 quadrants][2][R][kXchStride] fp32
};

struct ConvArgs {
  ConvLayout L;
  long long row_begin = 0, row_end = 0;  // samples handled by this launch
  const ClaimedRun* claim = nullptr;      // set: the rows stored there instead
  const void* w1 = nullptr;              // bf16 [c1][P*P]
  const float* b1 = nullptr;
  const void* w2 = nullptr;  // bf16 [c2][9*c1], K index = tap*c1 + channel, tap = 3*(dh+1)+(dw+1)
  const float* b2 = nullptr;
  // conv2 bias by value (kernel parameter space = constant cache): the conv2
  // epilogue's per-channel bias reads are uniform across lanes, and shared
  // memory reads queue behind the UMMAs' operand reads (tools/umma_contention.cu).
  float b2c[256] = {};
  // split: who moves the dw partials onto the output's lane -- 0: the tensor
  // pipe (tcgen05.shift: dw=0 one lane, dw=+1 two lanes, 12 ops per block);
  // 1: the epilogue (two shuffles per value); 2: both (dw=+1 one lane in the
  // pipe, then one shuffle of D'[p][0] + D'[p+1][+1]).  Measured on B200
  // (tools/trace_conv.cu, 2^20 samples): 2.67 / 2.92 / 2.62 ms.  The conv2
  // epilogue (4 warps, ~0.6 us per 128-row block) gates the issuer through
  // the 3-slot TMEM ring in every mode; the tensor pipe is ~55 % busy.
  int shifts = 2;
  void* out = nullptr;  // bf16 [rows][G*G*c2]
  // Design evidence (tools/trace_conv.cu): globaltimer stamps of CTA 0's
  // first 32 tiles, [tile][16]; nullptr in the product.
  unsigned long long* trace = nullptr;
  // Design evidence only (tools/trace_conv.cu): bits switch epilogue parts
  // off to find the bottleneck (1: conv1 TMEM loads, 2: conv1 smem stores,
  // 4: conv2 TMEM loads, 8: conv2 shuffles/exchange, 16: conv2 global
  // stores).  0 in the product.
  int debug = 0;
};

// False when the shape has no plan (P != 4, S % P != 0, c1 not in
// {32, 64, 128}, c2 not a multiple of 32 up to 256, grids larger than 13 x 13).
// schedule: 0 = split where the shape allows it, else tap; 1 = tap; 2 = split
// (false if the shape does not allow it).
bool conv_plan(int S, int P, int c1, int c2, ConvLayout* out, int schedule = 0);
// x: bf16 [x_rows][S*S].
int conv_launch(const ConvArgs& args, const void* x, long long x_rows, int grid, cudaStream_t stream);

}  // namespace es
