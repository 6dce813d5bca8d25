// The reference's batcher (src/runtime/pipeline.cpp:143-166) as the member
// kernels' tile space: a worker's segment s (rows [s*N, min((s+1)*N, nb)))
// becomes ceil(L/b) tiles of b rows, the last one the remainder
// (tests/test_runtime.cpp:315-332: 300 rows, N = 128, b = 32 -> 9 x 32 + 12).
// Shared by the fused-head kernels and the host (es_batch_rows), so the
// tiles the device runs are the ones the host-side tests check.
#pragma once

namespace es {

struct BatchTiles {
  long long per_seg = 1;    // tiles of a full segment
  long long total = 0;      // tiles of segments [seg_begin, seg_end)
  long long seg_begin = 0;  // first segment of the launch
};

// A data-parallel worker's claimed run (SURVEY.md §8-E device FIFO): the
// claim kernel (aux_kernels.cu) pops [seg_begin, seg_end) off its model's
// shared counter and stores it here, with the matching rows; every launch of
// the worker's member chain reads it at kernel start (stream order makes the
// claim visible), so all of a member's launches -- and every warp role inside
// them -- walk the same segments.
struct ClaimedRun {
  long long seg_begin, seg_end, row_begin, row_end;
};

__host__ __device__ __forceinline__ BatchTiles batch_tiles(long long seg_begin, long long seg_end,
                                                          int seg_size, long long nb, int b) {
  BatchTiles t;
  t.per_seg = (seg_size + b - 1) / b;
  t.seg_begin = seg_begin;
  const long long nseg = seg_end - seg_begin;
  if (nseg <= 0) return t;
  const long long last = seg_end - 1;
  const long long tail = nb - last * seg_size;
  const long long last_len = tail < seg_size ? tail : static_cast<long long>(seg_size);
  t.total = (nseg - 1) * t.per_seg + (last_len + b - 1) / b;
  return t;
}

// First row and row count of tile t (< ts.total).
__host__ __device__ __forceinline__ long long batch_tile(const BatchTiles& ts, long long t,
                                                        long long seg_begin, int seg_size,
                                                        long long nb, int b, int* rows) {
  const long long seg = seg_begin + t / ts.per_seg;
  const long long s1 = seg * seg_size + seg_size < nb ? seg * seg_size + seg_size : nb;
  const long long r0 = seg * seg_size + (t % ts.per_seg) * b;
  *rows = static_cast<int>(s1 - r0 < b ? s1 - r0 : static_cast<long long>(b));
  return r0;
}

}  // namespace es
