// Samples-in-M convolution stack of the CNN-s member (28x28 -> conv 4x4/4, 64
// filters -> conv 3x3 pad 1, 32 filters), DESIGN.md §5 "conv_rows".
//
// One UMMA tile is 128 SAMPLES at one spatial position, so a convolution tap
// is a choice of operand, never a lane shift, and zero-padding taps are never
// multiplied (the positions-in-M kernel, conv_kernel.cuh, pads 49 pixels to 64
// rows and moves partial sums across lanes):
//   * conv1 of position (ih, iw): D1[s][c] = sum_k patch(ih, iw)[s][k] W1[c][k],
//     one K = 16, N = 64 UMMA.  Two builder warps load each patch row's pixels
//     straight from x (L2) and write the K-major im2col operand (TMA boxes
//     must start 16-byte aligned and a patch row segment is 8 bytes,
//     tools/tma_probe.cu); a conv1 issuer warp issues as operands and the two
//     TMEM accumulators free up.
//   * the conv1 epilogue (two groups of four warps, one per accumulator)
//     writes relu(D1 + b1) as bf16 into an A2 slot -- TMEM (the conv2 UMMA
//     then reads A from TMEM) or a 128B-swizzled smem tile.
//   * conv2, output row oh, "window" iw: for each vertical tap dh the three
//     horizontal taps are ONE UMMA of N = 96 whose column block j holds
//     output (oh, iw - 1 + j): D = O + 32 (iw - 1) columns.  Successive
//     windows overlap by two blocks and simply ACCUMULATE (UMMAs into
//     overlapping TMEM column ranges sum exactly, tools/conv_probe.cu), so
//     the 9 taps, the border (clipped windows, N = 64 / 32) and the channel
//     sum all happen in the tensor pipe; an output block is final after its
//     right neighbour's window and is drained (bias, ReLU, bf16, HBM) by four
//     warps while the next windows run.
//   * on-chip capacity: a row sweep keeps 3 input rows live per column.  The
//     7 columns are done as two strips (output columns 0-3 from input
//     columns 0-4, 4-6 from 3-6; conv1 of columns 3-4 is recomputed), so the
//     live set is 3 rows x 5 columns = 15 A2 slots: 8 in TMEM, 7 in smem.
// Measured: every smem-A UMMA of N = 96 moves 7 KB through the
// 128 B/clk shared-memory port, so the smem-A windows saturate it and every
// other smem access (builder and epilogue stores, mbarrier operations) queues
// behind them; the kernel runs about even with the positions-in-M one in the
// cfg2 step.
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
  // Design evidence only (timing probes, results wrong): bit 2 = builders
  // skip their x reads, bit 4 = no A2 smem stores.  0 in the product.
  int debug = 0;
  // set by conv_rows_launch
  const void* x = nullptr;
  long long x_rows = 0;
};

// The shape this kernel is written for (BASELINE's CNN-s).
bool conv_rows_supported(int S, int P, int c1, int c2);
// x: bf16 [x_rows][784].
int conv_rows_launch(const ConvRowsArgs& args, const void* x, long long x_rows, int grid,
                     cudaStream_t stream);
// The input-sweep schedule of the same stack (conv_rows_kernel.cu, namespace
// sweep): each conv1 output feeds all nine of its outputs at once, every conv2
// UMMA reads A from TMEM.
int conv_sweep_launch(const ConvRowsArgs& args, const void* x, long long x_rows, int grid,
                      cudaStream_t stream);

}  // namespace es
