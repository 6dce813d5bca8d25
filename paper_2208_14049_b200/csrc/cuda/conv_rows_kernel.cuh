// Samples-in-M convolution stack of the CNN-s member (28x28 -> conv 4x4/4, 64
// filters -> conv 3x3 pad 1, 32 filters), DESIGN.md §5 "conv_rows".
//
// One UMMA tile is 128 SAMPLES at one spatial position, so a convolution tap
// is a choice of operand, never a lane shift:
//   * conv1 of position (ih, iw): D1[s][c] = sum_k patch(ih, iw)[s][k] W1[c][k].
//     TMA loads the 8-pixel row segments of two neighbouring patches straight
//     into the K-major operand (plane r = image row 4 ih + r), and a
//     block-diagonal W1 (zero for the neighbour's 4 pixels) picks the
//     position: two K = 16 UMMAs of N = 64 per position, no im2col copy.
//   * the conv1 epilogue writes relu(D1 + b1) as bf16 into an A2 slot -- TMEM
//     (the next UMMA reads A from TMEM) or a 128B-swizzled smem tile.
//   * conv2, output row oh, "window" iw: for each vertical tap dh the three
//     horizontal taps are ONE UMMA of N = 96 whose column block j holds
//     output (oh, iw - 1 + j): D = O + 32 (iw - 1) columns.  Successive
//     windows overlap by two blocks and simply ACCUMULATE (UMMAs into
//     overlapping TMEM column ranges sum exactly, tools/conv_probe.cu), so
//     the 9 taps, the border (clipped windows, N = 64 / 32) and the channel
//     sum all happen in the tensor pipe; an output block is final after its
//     right neighbour's window and is drained (bias, ReLU, bf16, HBM) while
//     the next windows run.  Zero-padding taps are never multiplied.
//   * on-chip capacity: a row sweep keeps ~2 input rows live.  The 7 columns
//     are done as two strips (output columns 0-3 from input columns 0-4,
//     4-6 from 3-6; conv1 of columns 3-4 is recomputed), so the live set is
//     3 rows x 5 columns = 15 A2 slots: 6 in TMEM, 9 in shared memory.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "batching.cuh"

namespace es {

struct ConvRowsArgs {
  long long row_begin = 0, row_end = 0;  // samples handled by this launch
  const ClaimedRun* claim = nullptr;     // set: the rows stored there instead
  const void* w1 = nullptr;              // bf16 [64][16], K = 4 r + px
  const void* w2 = nullptr;              // bf16 [32][576], K = (3 dh + dw) 64 + ci
  void* out = nullptr;                   // bf16 [rows][7*7*32], (h, w, c) order
  // biases by value (kernel parameter space = constant cache, uniform reads)
  float b1c[64] = {};
  float b2c[32] = {};
  // Design evidence only (tools/trace_rows.cu): clock64 stamps of CTA 0,
  // [event kind][index < 256]; nullptr in the product.
  unsigned long long* trace = nullptr;
  // Design evidence only: bit 0 = no L2 prefetch of the next tile.  0 in the product.
  int debug = 0;
  // set by conv_rows_launch: x itself, for the L2 prefetch of the next tile
  const void* x = nullptr;
  long long x_rows = 0;
};

// The shape this kernel is written for (BASELINE's CNN-s).
bool conv_rows_supported(int S, int P, int c1, int c2);
// x: bf16 [x_rows][784].
int conv_rows_launch(const ConvRowsArgs& args, const void* x, long long x_rows, int grid,
                     cudaStream_t stream);

}  // namespace es
