// Samples-in-M CNN-s convolution stack (design in conv_rows_kernel.cuh).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "conv_rows_kernel.cuh"
#include "sm100.cuh"
#include "tma_host.hpp"  // ensure_smem_attr

namespace es {

using namespace sm100;

namespace {

constexpr int kS = 28, kG = 7, kC1 = 64, kC2 = 32, kTile = 128;
constexpr int kOutRow = kG * kG * kC2;  // bf16 elements per output sample
constexpr int kBuilders = 2;            // im2col builder warps (kSampPerLane samples per lane)
constexpr int kSampPerLane = 128 / (32 * kBuilders);
constexpr int kThreads = 32 * (kBuilders + 14);  // + conv1 issuer, conv2 issuer, 2 x 4 conv1
                                                 // epilogue, 4 output drain
// Shared memory (offsets from the 1024-aligned base).
constexpr uint32_t kSlotBytes = 16384;  // A2 smem slot: [128 samples][64 ch] bf16, SW128
constexpr int kSmemSlots = 7;
constexpr uint32_t kOffW2 = kSmemSlots * kSlotBytes;  // [dh][ks][plane][96 rows][16 B]
constexpr uint32_t kW2Plane = 96 * 16;
constexpr uint32_t kOffW1 = kOffW2 + 3 * 4 * 2 * kW2Plane;  // [plane][64 c][16 B]
constexpr uint32_t kOffA1 = kOffW1 + 2 * 64 * 16;           // im2col ring: [2 planes][128][16 B]
constexpr uint32_t kA1Bytes = 2 * 128 * 16;
constexpr int kA1Stages = 10;  // two patch rows of im2col operands
constexpr uint32_t kOffBar = kOffA1 + kA1Stages * kA1Bytes;
constexpr int kNumBars = kA1Stages * 2 + 2 + 2 + 15 + 15 + 4 + 4;
constexpr uint32_t kSmemBytes = kOffBar + kNumBars * 8 + 16 + 1024;

// TMEM columns: output-row accumulator O (4 blocks of 32), two conv1
// accumulators of 64, eight A2 slots of 32 (64 bf16 channels packed in pairs).
constexpr uint32_t kTmO = 0, kTmD1 = 128, kTmA2 = 256;

// A2 slot of (strip column j = iw - first column, input-row phase p).  A UMMA
// reading A from smem costs max(N/2, (4096 + 32 N)/128) clk and takes the
// smem bandwidth the builder and epilogue also need; from TMEM N/2
// (tools/conv_probe.cu).  TMEM holds 8 of the 15 slots: columns 0 and 3
// (narrow windows) and column 4 (N = 32, strip A only) at phases 0 and 1;
// shared memory the rest.  Slot id (barriers) = 3 j + p.
__host__ __device__ constexpr bool slot_tmem(int j, int p) { return j == 0 || j == 3 || (j == 4 && p < 2); }
__host__ __device__ constexpr int slot_index(int j, int p) {  // within its memory
  return slot_tmem(j, p) ? (j == 0 ? p : j == 3 ? 3 + p : 6 + p) : (j == 1 ? p : j == 2 ? 3 + p : 6);
}

// bf16x2 {relu(a + ba), relu(b + bb)} (a in the low half), one cvt.relu.
__device__ __forceinline__ uint32_t pack_relu_bf16(uint32_t a, uint32_t b, float ba, float bb) {
  const float lo = __uint_as_float(a) + ba;
  const float hi = __uint_as_float(b) + bb;
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// Stamp event `kind` number i (CTA 0 only, tools/trace_rows.cu).
#define TRACE(kind, i)                                                                      \
  do {                                                                                      \
    if (trace && (i) < 256) trace[(kind) * 256 + (i)] = static_cast<unsigned long long>(clock64()); \
  } while (0)

struct Bars {
  uint64_t* a1_full;   // [kA1Stages] builders -> conv1 issuer
  uint64_t* a1_empty;  // [kA1Stages]
  uint64_t* c1_full;   // [2] conv1 issuer -> epilogue group of that D slot
  uint64_t* c1_empty;  // [2]
  uint64_t* a2_full;   // [15] conv1 epilogue -> conv2 issuer
  uint64_t* a2_empty;  // [15]
  uint64_t* o_full;    // [4] conv2 issuer -> drain
  uint64_t* o_empty;   // [4]
};

// ------------------------------------------------------------ conv2 issuer
struct IssueCtx {
  uint32_t tbase;
  uint64_t a2d;  // SW128 descriptor of A2 smem slot 0
  uint64_t w2d;  // planar descriptor of W2
  Bars b;
  uint32_t a2par;  // per slot id: parity of the next fill to wait for
  uint32_t ouse;   // per O block: parity of its first-touch count
  unsigned long long* trace;
  int w;  // running window index (trace)
};

// D (+)= A2(slot of column J, phase p) x W2(dh, ks, blocks jlo..jlo+n-1).
template <int J, int NB, int P>
__device__ __forceinline__ void mma2(const IssueCtx& c, uint32_t d, int dh, int ks, int jlo,
                                     uint32_t acc) {
  constexpr uint32_t p = P;
  constexpr uint32_t idesc = idesc_bf16_f32(128, 32 * NB);
  const uint64_t bd = c.w2d + static_cast<uint64_t>(((dh * 4 + ks) * 2 * kW2Plane + jlo * 32 * 16) >> 4);
  auto tm = [&](uint32_t t) {
    if (elect_one()) umma_bf16_ta(d, c.tbase + kTmA2 + 32u * t + 8u * ks, bd, idesc, acc);
  };
  auto sm = [&](uint32_t t) {
    if (elect_one())
      umma_bf16(d, c.a2d + static_cast<uint64_t>(t * (kSlotBytes >> 4) + 2u * ks), bd, idesc, acc);
  };
  if constexpr (J == 0 || J == 3) {
    tm((J == 0 ? 0u : 3u) + p);
  } else if constexpr (J == 4) {
    if constexpr (P < 2) tm(6u + p);
    else sm(6u);
  } else {
    sm((J == 1 ? 0u : 3u) + p);
  }
}

__device__ __forceinline__ void wait_slot(IssueCtx& c, uint32_t sid) {
  mbar_wait(&c.b.a2_full[sid], (c.a2par >> sid) & 1u);
  c.a2par ^= 1u << sid;
}

// Window IW of strip ST for output row oh, whose input row has phase P1: the
// phases (slot addresses) are template arguments, so every operand address is
// a constant offset from a uniform base (a run-time phase cost an R2UR per UMMA
// and ~40 clk of issue each).
template <int ST, int IW, int P1>
__device__ __forceinline__ void window(IssueCtx& c, int oh) {
  constexpr uint32_t p1 = P1, p0 = (P1 + 2) % 3, p2 = (P1 + 1) % 3;
  constexpr int c0 = ST ? 3 : 0, ow0 = ST ? 4 : 0, nout = ST ? 3 : 4, iwl = ST ? 6 : 4;
  constexpr int J = IW - c0;
  constexpr int owlo = IW - 1 > ow0 ? IW - 1 : ow0;
  constexpr int owhi = IW + 1 < ow0 + nout - 1 ? IW + 1 : ow0 + nout - 1;
  constexpr int jlo = owlo - IW + 1, NB = owhi - owlo + 1, dblk = owlo - ow0;
  constexpr bool all_new = IW == c0;
  constexpr bool last_new = !all_new && owhi == IW + 1;
  unsigned long long* trace = c.trace;
  TRACE(6, c.w);
  // new input positions: (0, IW) and (1, IW) at the first row, else (oh+1, IW)
  if (oh == 0) wait_slot(c, 3u * J + p1);
  if (oh < kG - 1) wait_slot(c, 3u * J + p2);
  // first touches of O blocks in this output row
#pragma unroll
  for (int b = dblk; b < dblk + NB; ++b)
    if (all_new || (last_new && b == dblk + NB - 1)) {
      mbar_wait(&c.b.o_empty[b], ((c.ouse >> b) & 1u) ^ 1u);
      c.ouse ^= 1u << b;
    }
  tc_fence_after();
  TRACE(7, c.w);
  // Opaque per-window copies of the bases: otherwise the compiler hoists all
  // 36 B descriptors of the strip into uniform registers and spills them.
  IssueCtx cw = c;
  asm volatile("" : "+l"(cw.w2d), "+l"(cw.a2d), "+r"(cw.tbase));
  const uint32_t d = cw.tbase + kTmO + 32u * dblk;
  // dh = 1 (always valid) first: its K step 0 starts the new blocks.
  if constexpr (last_new) {  // old blocks accumulate, the new (last) one starts
    mma2<J, NB - 1, p1>(cw, d, 1, 0, jlo, 1u);
    mma2<J, 1, p1>(cw, d + 32u * (NB - 1), 1, 0, jlo + NB - 1, 0u);
  } else {
    mma2<J, NB, p1>(cw, d, 1, 0, jlo, all_new ? 0u : 1u);
  }
#pragma unroll
  for (int ks = 1; ks < 4; ++ks) mma2<J, NB, p1>(cw, d, 1, ks, jlo, 1u);
  if (oh > 0) {
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) mma2<J, NB, p0>(cw, d, 0, ks, jlo, 1u);
  }
  if (oh < kG - 1) {
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) mma2<J, NB, p2>(cw, d, 2, ks, jlo, 1u);
  }
  // releases: input (oh-1, IW) is dead; at the last row (oh, IW) too
  if (oh > 0 && elect_one()) umma_commit(&c.b.a2_empty[3u * J + p0]);
  if (oh == kG - 1 && elect_one()) umma_commit(&c.b.a2_empty[3u * J + p1]);
  // output blocks completed by this window
  if constexpr (IW - 1 >= ow0 && IW - 1 < ow0 + nout)
    if (elect_one()) umma_commit(&c.b.o_full[IW - 1 - ow0]);
  if constexpr (IW == iwl && IW < ow0 + nout)
    if (elect_one()) umma_commit(&c.b.o_full[IW - ow0]);
  __syncwarp();
  TRACE(8, c.w);
  ++c.w;
}

// Patch row ih of strip ST for this lane's two samples; positions n0 .. n0+J-1.
template <int ST, int SPL = kSampPerLane>
__device__ __forceinline__ void build_row(const ConvRowsArgs& args, uint8_t* smem, const Bars& B,
                                          long long s0, int ih, int warp, int lane, int n0,
                                          uint32_t off_a1 = kOffA1) {
  constexpr int J = ST ? 4 : 5, c0 = ST ? 3 : 0;
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int smp = warp * 32 * SPL + t * 32 + lane;
    const long long s = s0 + smp;
    uint4 ch[4][3];
    const uint8_t* xrow = static_cast<const uint8_t*>(args.x) + s * (kS * kS * 2);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      // first pixel of the aligned 24-pixel window of image row y = 4 ih + r
      const int y = 4 * ih + r;
      const int x0 = ST ? 28 * y + 12 - 4 * ((r + 1) & 1) : 28 * y - 4 * (r & 1);
#pragma unroll
      for (int m = 0; m < 3; ++m)
        ch[r][m] = s < args.x_rows
                       ? __ldg(reinterpret_cast<const uint4*>(xrow + 2 * (x0 + 8 * m)))
                       : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int n = n0 + j;
      const int sl = static_cast<int>(n % kA1Stages);
      if (t == 0) mbar_sleep_wait(&B.a1_empty[sl], (static_cast<uint32_t>(n / kA1Stages) & 1u) ^ 1u);
      uint32_t w[4][2];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        // pixel offset of the position's 4 pixels inside the window
        const int c = c0 + j;
        const int o = ST ? 4 * c - 12 + 4 * ((r + 1) & 1) : 4 * c + 4 * (r & 1);
        const uint4 q = ch[r][o / 8];
        const bool hi = (o % 8) != 0;
        w[r][0] = hi ? q.z : q.x;
        w[r][1] = hi ? q.w : q.y;
      }
      uint8_t* a1 = smem + off_a1 + sl * kA1Bytes + smp * 16;
      *reinterpret_cast<uint4*>(a1) = make_uint4(w[0][0], w[0][1], w[1][0], w[1][1]);
      *reinterpret_cast<uint4*>(a1 + 2048) = make_uint4(w[2][0], w[2][1], w[3][0], w[3][1]);
    }
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < J; ++j) mbar_arrive(&B.a1_full[(n0 + j) % kA1Stages]);
    unsigned long long* trace = blockIdx.x == 0 && warp == 0 ? args.trace : nullptr;
    TRACE(1, static_cast<int>(n0));
  }
}

template <int P>
__device__ __forceinline__ void strip_a(IssueCtx& c, int oh) {
  window<0, 0, P>(c, oh);
  window<0, 1, P>(c, oh);
  window<0, 2, P>(c, oh);
  window<0, 3, P>(c, oh);
  window<0, 4, P>(c, oh);
}
template <int P>
__device__ __forceinline__ void strip_b(IssueCtx& c, int oh) {
  window<1, 3, P>(c, oh);
  window<1, 4, P>(c, oh);
  window<1, 5, P>(c, oh);
  window<1, 6, P>(c, oh);
}

__global__ void __launch_bounds__(kThreads, 1)
    conv_rows_sm100(const ConvRowsArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bar0 = reinterpret_cast<uint64_t*>(smem + kOffBar);
  Bars B;
  B.a1_full = bar0;
  B.a1_empty = B.a1_full + kA1Stages;
  B.c1_full = B.a1_empty + kA1Stages;
  B.c1_empty = B.c1_full + 2;
  B.a2_full = B.c1_empty + 2;
  B.a2_empty = B.a2_full + 15;
  B.o_full = B.a2_empty + 15;
  B.o_empty = B.o_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(B.o_empty + 4);

  const int warp = warp_uniform_id();
  const int lane = threadIdx.x & 31;
  unsigned long long* const trace = blockIdx.x == 0 ? args.trace : nullptr;
  const long long row_begin = args.claim ? args.claim->row_begin : args.row_begin;
  const long long row_end = args.claim ? args.claim->row_end : args.row_end;
  const long long tiles = (row_end - row_begin + kTile - 1) / kTile;
  const int my_tiles =
      blockIdx.x < tiles ? static_cast<int>((tiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kA1Stages; ++i) {
      mbar_init(&B.a1_full[i], kBuilders);
      mbar_init(&B.a1_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) mbar_init(&B.c1_full[i], 1);
    for (int i = 0; i < 2; ++i) mbar_init(&B.c1_empty[i], 4);
    for (int i = 0; i < 15; ++i) {
      mbar_init(&B.a2_full[i], 4);
      mbar_init(&B.a2_empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&B.o_full[i], 1);
      mbar_init(&B.o_empty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);

  // Resident weights.  W2 -> [dh][ks][plane][n = 32 j + co][8 ci] with
  // j = 2 - dw (window column block j is output iw - 1 + j, read through
  // tap dw = 2 - j).  W1 -> [plane][c][8]: K = 4 r + px, plane p = rows
  // 2p, 2p + 1 (the im2col order below).
  {
    const uint4* w2 = static_cast<const uint4*>(args.w2);  // [32][72 chunks of 8]
    for (int i = threadIdx.x; i < kC2 * 72; i += kThreads) {
      const int co = i / 72, ch = i % 72, tap = ch >> 3, rem = ch & 7;
      const int ks = rem >> 1, pl = rem & 1, dh = tap / 3, dw = tap % 3, j = 2 - dw;
      *reinterpret_cast<uint4*>(smem + kOffW2 + ((dh * 4 + ks) * 2 + pl) * kW2Plane +
                                (j * 32 + co) * 16) = w2[i];
    }
    const uint4* w1 = static_cast<const uint4*>(args.w1);  // [64][2 chunks of 8]
    for (int i = threadIdx.x; i < 2 * 64; i += kThreads) {
      const int c = i >> 1, pl = i & 1;
      *reinterpret_cast<uint4*>(smem + kOffW1 + (pl * 64 + c) * 16) = w1[i];
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  if (warp < kBuilders) {
    // ------------------------------------------------------ im2col builders
    // Each lane owns samples 64 w + 32 t + lane (t = 0, 1).  Per patch row it
    // loads, straight from x (L2; no smem staging, whose loads queued behind
    // the UMMA operand reads), the 16-byte-aligned chunks covering the
    // strip's pixels of the 4 image rows, then writes every position's K = 16
    // operand: plane p = rows 2p, 2p + 1 x the position's 4 pixels.
    int n = 0;
    for (int k = 0; k < my_tiles; ++k) {
      const long long s0 = row_begin + (blockIdx.x + static_cast<long long>(k) * gridDim.x) * kTile;
      for (int ih = 0; ih < kG; ++ih) {
        build_row<0>(args, smem, B, s0, ih, warp, lane, n);
        n += 5;
      }
      for (int ih = 0; ih < kG; ++ih) {
        build_row<1>(args, smem, B, s0, ih, warp, lane, n);
        n += 4;
      }
    }
  } else if (warp == kBuilders) {
    // ----------------------------------------------------- conv1 issuer
    // One K = 16 UMMA (N = 64) per position, in production order, as soon as
    // its operand is built and an accumulator is free.  (Feeding conv1 from
    // the conv2 issuer's own stream cost ~800 clk of issue overhead a window.)
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t a1_base = __shfl_sync(0xffffffffu, smem_u32(smem + kOffA1), 0);
    const uint64_t w1d = sdesc_planar(__shfl_sync(0xffffffffu, smem_u32(smem + kOffW1), 0), 1024);
    constexpr uint32_t id1 = idesc_bf16_f32(128, kC1);
    const int npos = my_tiles * 63;
    int sl = 0;
    uint32_t slpar = 0;
    for (int n = 0; n < npos; ++n) {
      mbar_sleep_wait(&B.a1_full[sl], slpar);
      const int dsl = n & 1;
      mbar_sleep_wait(&B.c1_empty[dsl], (static_cast<uint32_t>(n >> 1) & 1u) ^ 1u);
      if (lane == 0) TRACE(2, n);
      tc_fence_after();
      if (elect_one()) {
        umma_bf16(tbase + kTmD1 + 64u * dsl, sdesc_planar(a1_base + sl * kA1Bytes, 2048), w1d, id1, 0);
        umma_commit(&B.c1_full[dsl]);
        umma_commit(&B.a1_empty[sl]);
      }
      __syncwarp();
      if (++sl == kA1Stages) {
        sl = 0;
        slpar ^= 1u;
      }
    }
  } else if (warp == kBuilders + 1) {
    // ----------------------------------------------------- conv2 issuer
    IssueCtx c;
    c.tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    c.a2d = sdesc_k128(__shfl_sync(0xffffffffu, smem_u32(smem), 0));
    c.w2d = sdesc_planar(__shfl_sync(0xffffffffu, smem_u32(smem + kOffW2), 0), kW2Plane);
    c.b = B;
    c.a2par = 0;
    c.ouse = 0;
    c.trace = trace;
    c.w = 0;

    for (int k = 0; k < my_tiles; ++k) {
      const int g0 = (k * 14) % 3;  // row-phase origin of this tile
      for (int oh = 0; oh < kG; ++oh) {
        switch ((g0 + oh) % 3) {
          case 0: strip_a<0>(c, oh); break;
          case 1: strip_a<1>(c, oh); break;
          default: strip_a<2>(c, oh); break;
        }
      }
      for (int oh = 0; oh < kG; ++oh) {
        switch ((g0 + 7 + oh) % 3) {
          case 0: strip_b<0>(c, oh); break;
          case 1: strip_b<1>(c, oh); break;
          default: strip_b<2>(c, oh); break;
        }
      }
    }
  } else if (warp < kBuilders + 10) {
    // ------------------------------------------------- conv1 epilogue
    // Two groups of four warps (one per TMEM lane quadrant), group g owns
    // conv1 accumulator g and takes positions n = g mod 2; each walks every
    // position to keep the slot parities.
    const int g = (warp - kBuilders - 2) >> 2, qd = warp & 3;
    const uint32_t lane_field = static_cast<uint32_t>(qd * 32) << 16;
    const int row = qd * 32 + lane;  // sample within the tile
    uint32_t a2par = 0;              // per slot id: parity of the next empty-wait
    int n = 0;
    for (int k = 0; k < my_tiles; ++k) {
      const int g0 = (k * 14) % 3;
      for (int li = 0; li < 63; ++li, ++n) {  // production order
        {
          const int st = li < 35 ? 0 : 1, ih = st ? (li - 35) / 4 : li / 5, j = st ? (li - 35) % 4 : li % 5;
          {
            const uint32_t ph = static_cast<uint32_t>((g0 + 7 * st + ih) % 3);
            const uint32_t sid = 3u * j + ph;
            const uint32_t par = (a2par >> sid) & 1u;
            a2par ^= 1u << sid;
            const int dsl = static_cast<int>(n & 1);  // this group's D slot
            if (dsl != g) continue;
            mbar_sleep_wait(&B.c1_full[dsl], static_cast<uint32_t>(n >> 1) & 1u);
            if (qd == 0 && lane == 0) TRACE(3, n);
            tc_fence_after();
            uint32_t v0[32], v1[32];
            const uint32_t src = tmem_base + lane_field + kTmD1 + 64u * dsl;
            tmem_ld32_raw(src, v0);
            tmem_ld32_raw(src + 32u, v1);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&B.c1_empty[dsl]);
            uint32_t pk[32];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              pk[i] = pack_relu_bf16(v0[2 * i], v0[2 * i + 1], args.b1c[2 * i], args.b1c[2 * i + 1]);
              pk[16 + i] = pack_relu_bf16(v1[2 * i], v1[2 * i + 1], args.b1c[32 + 2 * i],
                                          args.b1c[33 + 2 * i]);
            }
            mbar_sleep_wait(&B.a2_empty[sid], par ^ 1u);
            if (qd == 0 && lane == 0) TRACE(4, n);
            if (slot_tmem(j, static_cast<int>(ph))) {
              tc_fence_after();
              tmem_st32(tmem_base + lane_field + kTmA2 + 32u * slot_index(j, static_cast<int>(ph)), pk);
              tmem_st_wait();
              tc_fence_before();
            } else {
              uint8_t* dst = smem + slot_index(j, static_cast<int>(ph)) * kSlotBytes + row * 128;
              if (!(args.debug & 4))  // timing probe: no A2 smem stores
#pragma unroll
              for (int cc = 0; cc < 8; ++cc)
                *reinterpret_cast<uint4*>(dst + ((cc ^ (row & 7)) << 4)) =
                    make_uint4(pk[4 * cc], pk[4 * cc + 1], pk[4 * cc + 2], pk[4 * cc + 3]);
              fence_proxy_async_smem();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&B.a2_full[sid]);
            if (qd == 0 && lane == 0) TRACE(5, n);
          }
        }
      }
    }
  } else {
    // ----------------------------------------------------- output drain
    const int qd = warp & 3;
    const uint32_t lane_field = static_cast<uint32_t>(qd * 32) << 16;
    const int row = qd * 32 + lane;
    uint32_t opar = 0;
    int nblk = 0;
    for (int k = 0; k < my_tiles; ++k) {
      const long long s = row_begin + (blockIdx.x + static_cast<long long>(k) * gridDim.x) * kTile + row;
      uint8_t* dst_row = static_cast<uint8_t*>(args.out) + s * (kOutRow * 2);
      const bool valid = s < row_end;
      for (int st = 0; st < 2; ++st)
        for (int oh = 0; oh < kG; ++oh)
          for (int b = 0; b < (st ? 3 : 4); ++b) {
            mbar_sleep_wait(&B.o_full[b], (opar >> b) & 1u);
            opar ^= 1u << b;
            if (qd == 0 && lane == 0) TRACE(9, nblk);
            ++nblk;
            tc_fence_after();
            uint32_t v[32];
            tmem_ld32_raw(tmem_base + lane_field + kTmO + 32u * b, v);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&B.o_empty[b]);
            if (valid) {
              const int ow = (st ? 4 : 0) + b;
              uint4* dst = reinterpret_cast<uint4*>(dst_row + (oh * kG + ow) * kC2 * 2);
#pragma unroll
              for (int c = 0; c < 4; ++c)
                dst[c] = make_uint4(
                    pack_relu_bf16(v[8 * c], v[8 * c + 1], args.b2c[8 * c], args.b2c[8 * c + 1]),
                    pack_relu_bf16(v[8 * c + 2], v[8 * c + 3], args.b2c[8 * c + 2], args.b2c[8 * c + 3]),
                    pack_relu_bf16(v[8 * c + 4], v[8 * c + 5], args.b2c[8 * c + 4], args.b2c[8 * c + 5]),
                    pack_relu_bf16(v[8 * c + 6], v[8 * c + 7], args.b2c[8 * c + 6], args.b2c[8 * c + 7]));
            }
          }
    }
  }

  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// ====================================================================
// conv_sweep_sm100: the input-sweep schedule (conv_rows_kernel.cuh).
//
// Each conv1 output A2(ih, iw) is consumed as soon as it exists: ONE set of
// UMMAs with A read from TMEM adds it to all nine outputs it feeds.  The
// output accumulator O holds three output rows of the strip, laid out
// [j = ow - ow0][r = (oh + 1) mod 3] x 32 channels, so the nine taps of an
// input are 9 CONTIGUOUS 32-column blocks (j = 2 - dw, r from dh); the B
// operand is W2 with its tap blocks in that order, one copy per input-row
// phase q = ih mod 3 (dh = (q + 2 - r) mod 3).  Interior inputs issue
// N = 160 + 128 per K step (all 288 columns), strip-edge inputs N = 192 or
// 96, and the image's top / bottom input rows one N = 64 UMMA per output
// column (the two valid rows).  Every UMMA accumulates: the drain zeroes a
// block after reading it, so the row that next uses the block starts at 0.
namespace sweep {

constexpr int kBuilders = 4;       // one sample per lane: one load round trip per patch row
// Warp roles: kBuilders im2col builders, the conv1 issuer, the conv2 issuer,
// kEpi conv1-epilogue warps (one per TMEM lane quadrant, all 64 channels;
// eight warps of 32 channels measured the same), kDrain drain warps, and a
// watcher that only runs under tools/trace_rows.cu.
constexpr int kEpi = 4;
#ifndef ES_SWEEP_DIRECT
#define ES_SWEEP_DIRECT 0
#endif
constexpr bool kDirectStores = ES_SWEEP_DIRECT;  // A/B build switch (design probe)
constexpr int kDrain = 4;
constexpr int kThreads = 32 * (kBuilders + 2 + kEpi + kDrain + 1);
// Warp -> role.  A warp issues on sub-partition warp % 4, and the epilogue and
// drain warps of TMEM lane quadrant q must sit on sub-partition q; the conv2
// issuer gets sub-partition 1 with no builder beside it (its per-input
// instructions compete for that sub-partition's issue slots, and the tensor
// pipe queues only ~2 UMMAs).
enum Role : int { kRBuild, kRConv1, kRConv2, kREpi, kRDrain, kRWatch };
constexpr int kRoles[kThreads / 32] = {kRBuild, kRConv2, kRBuild, kRBuild, kRBuild, kREpi,   kRConv1, kREpi,
                                       kREpi,   kRDrain, kREpi,   kRDrain, kRDrain, kRWatch, kRDrain};
__host__ __device__ constexpr uint64_t pack_roles() {  // 3 bits per warp: no local-memory table
  uint64_t v = 0;
  for (int w = 0; w < kThreads / 32; ++w) v |= static_cast<uint64_t>(kRoles[w]) << (3 * w);
  return v;
}
__host__ __device__ constexpr uint64_t pack_role_idx() {  // 4 bits per warp: index within its role
  uint64_t v = 0;
  for (int w = 0; w < kThreads / 32; ++w) {
    int k = 0;
    for (int i = 0; i < w; ++i) k += kRoles[i] == kRoles[w];
    v |= static_cast<uint64_t>(k) << (4 * w);
  }
  return v;
}
__host__ __device__ __forceinline__ int role_of(int w) {
  return static_cast<int>((pack_roles() >> (3 * w)) & 7u);
}
__host__ __device__ __forceinline__ int role_idx(int w) {
  return static_cast<int>((pack_role_idx() >> (4 * w)) & 15u);
}  // + conv1 issuer,
                                                                     // conv2 issuer, 8 conv1 epilogue
constexpr uint32_t kQBytes = 4 * 2 * 288 * 16;  // one W2 copy: [ks][plane][288 rows][16 B]
constexpr uint32_t kOffW2 = 0;
constexpr uint32_t kOffW1 = kOffW2 + 3 * kQBytes;
constexpr uint32_t kOffA1 = kOffW1 + 2 * 64 * 16;
// drain staging: per drain warp a ring of kOutStages boxes [32 samples][64 B]
// (one O block of its lane quadrant), 64-byte swizzled, stored by TMA
constexpr int kOutStages = 4;
constexpr uint32_t kOutBox = 32 * 64;
constexpr uint32_t kOffOut = kOffA1 + kA1Stages * kA1Bytes;
constexpr uint32_t kOffBar = kOffOut + 4 * kOutStages * kOutBox;  // 4 drain warps
constexpr int kNumBars = 2 * kA1Stages + 2 + 4 + 24 + 1;
constexpr uint32_t kSmemBytes = kOffBar + kNumBars * 8 + 16 + 1024;
// TMEM: O [0, 384), conv1 accumulator D1 [384, 448), two A2 slots [448, 512).
constexpr uint32_t kTmO = 0, kTmD1 = 384, kTmA2 = 448;

struct Bars {
  uint64_t* a1_full;   // [kA1Stages] builders -> conv1 issuer
  uint64_t* a1_empty;  // [kA1Stages]
  uint64_t* c1_full;   // conv1 issuer -> epilogue
  uint64_t* c1_empty;  // epilogue (8 warps) -> conv1 issuer
  uint64_t* a2_full;   // [2] epilogue -> conv2 issuer
  uint64_t* a2_empty;  // [2]
  uint64_t* o_full;    // [12] block b = 3 j + r: conv2 issuer -> drain
  uint64_t* o_empty;   // [12] drain (4 warps) -> conv2 issuer
};

// Strip geometry: strip 0 = output columns 0-3 from input columns 0-4,
// strip 1 = output columns 4-6 from input columns 3-6.
__host__ __device__ constexpr int c0(int st) { return st ? 3 : 0; }     // first input column
__host__ __device__ constexpr int clast(int st) { return st ? 6 : 4; }  // last input column
__host__ __device__ constexpr int ow0(int st) { return st ? 4 : 0; }    // first output column
__host__ __device__ constexpr int nw(int st) { return st ? 3 : 4; }     // output columns
__host__ __device__ constexpr int slot_r(int oh) { return (oh + 1) % 3; }
__host__ __device__ constexpr int block(int st, int oh, int ow) { return 3 * (ow - ow0(st)) + slot_r(oh); }
__host__ __device__ constexpr bool in_strip(int st, int ow) { return ow >= ow0(st) && ow < ow0(st) + nw(st); }
// (oh, ow) is first touched by input (max(oh - 1, 0), max(ow - 1, c0)) and
// complete after input (min(oh + 1, 6), min(ow + 1, clast)) -- row-major order.
__host__ __device__ constexpr bool first_at(int st, int ih, int iw, int oh, int ow) {
  return in_strip(st, ow) && oh >= 0 && oh < kG && (oh - 1 > 0 ? oh - 1 : 0) == ih &&
         (ow - 1 > c0(st) ? ow - 1 : c0(st)) == iw;
}
__host__ __device__ constexpr bool last_at(int st, int ih, int iw, int oh, int ow) {
  return in_strip(st, ow) && oh >= 0 && oh < kG && (oh + 1 < kG - 1 ? oh + 1 : kG - 1) == ih &&
         (ow + 1 < clast(st) ? ow + 1 : clast(st)) == iw;
}

// The drain's walk: O blocks of one tile in completion order (block id and
// output position oh * 7 + ow), a compile-time table so the drain's control
// flow is one constant-bank load per block (the nested loop with run-time
// last_at() tests cost ~600 clk per block of dependent integer issue).
struct DrainSeq {
  uint8_t blk[kG * kG];
  uint8_t pos[kG * kG];
};
__host__ __device__ constexpr DrainSeq make_drain_seq() {
  DrainSeq d{};
  int k = 0;
  for (int st = 0; st < 2; ++st)
    for (int ih = 0; ih < kG; ++ih)
      for (int iw = c0(st); iw <= clast(st); ++iw)
        for (int oh = ih - 1; oh <= ih; ++oh)
          for (int ow = iw - 1; ow <= iw; ++ow)
            if (last_at(st, ih, iw, oh, ow)) {
              d.blk[k] = static_cast<uint8_t>(block(st, oh, ow));
              d.pos[k] = static_cast<uint8_t>(oh * kG + ow);
              ++k;
            }
  return d;
}
__constant__ DrainSeq kDrainSeq = make_drain_seq();

// Patch row ih of strip ST for this lane's sample (builder warps own 32
// samples each), positions n0 .. n0 + J - 1.  Each position is published as
// soon as it is written (conv1 of the row's first position does not wait for
// the whole row), waits spin (a suspended builder woke late at row starts),
// and the next patch row's image lines are prefetched into L1 before this
// row's operands are written.
__device__ __forceinline__ uint4 ld_hint(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// Strip 0 reads an image band first (evict_last: strip 1 reads it again
// half a tile later), strip 1 last (evict_first).
template <int ST>
__device__ __forceinline__ void build_row_sweep(const ConvRowsArgs& args, uint8_t* smem, const es::Bars& B,
                                                long long s, int ih, int smp, int lane, int n0,
                                                const uint8_t* next_row) {
  const uint64_t pol = ST ? l2_policy_evict_first() : l2_policy_evict_last();
  constexpr int J = ST ? 4 : 5, cs = ST ? 3 : 0;
  uint4 ch[4][3];
  const uint8_t* xrow = static_cast<const uint8_t*>(args.x) + s * (kS * kS * 2);
  const bool in = s < args.x_rows;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int y = 4 * ih + r;
    const int x0 = ST ? 28 * y + 12 - 4 * ((r + 1) & 1) : 28 * y - 4 * (r & 1);
#pragma unroll
    for (int m = 0; m < 3; ++m)
      ch[r][m] = in ? ld_hint(xrow + 2 * (x0 + 8 * m), pol) : make_uint4(0, 0, 0, 0);
  }
  if (next_row) {  // the next patch row's 224 bytes (up to three 128-byte lines)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(next_row));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(next_row + 112));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(next_row + 223));
  }
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int n = n0 + j;
    const int sl = n % kA1Stages;
    mbar_wait(&B.a1_empty[sl], (static_cast<uint32_t>(n / kA1Stages) & 1u) ^ 1u);
    uint32_t w[4][2];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int c = cs + j;
      const int o = ST ? 4 * c - 12 + 4 * ((r + 1) & 1) : 4 * c + 4 * (r & 1);
      const uint4 q = ch[r][o / 8];
      const bool hi = (o % 8) != 0;
      w[r][0] = hi ? q.z : q.x;
      w[r][1] = hi ? q.w : q.y;
    }
    uint8_t* a1 = smem + kOffA1 + sl * kA1Bytes + smp * 16;
    *reinterpret_cast<uint4*>(a1) = make_uint4(w[0][0], w[0][1], w[1][0], w[1][1]);
    *reinterpret_cast<uint4*>(a1 + 2048) = make_uint4(w[2][0], w[2][1], w[3][0], w[3][1]);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&B.a1_full[sl]);
  }
}

struct Ctx {
  uint32_t tbase;
  uint64_t w2d;  // planar descriptor of W2 copy 0, K step 0
  Bars b;
  uint32_t ouse;  // per O block: parity of its next empty-wait
  unsigned long long* trace;
  uint64_t* done;  // trace only: a commit per input, watched by the last warp
};

template <int N>
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b) {
  umma_bf16_ta(d, a, b, idesc_bf16_f32(128, N), 1u);
}

// Input (IH, IW) of strip ST: A2 slot `slot` into every output it feeds.
// 64-bit smem descriptor from a 32-bit low word (start address, LBO) and the
// constant high word: one add per operand instead of a 64-bit add chain.
__device__ __forceinline__ uint64_t desc64(uint32_t lo, uint32_t hi) {
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// kTr: the tools/trace_rows.cu build (clock stamps, completion commits); the
// product instantiation carries no trace code on the issuer's path (the
// tensor pipe queues only ~2 UMMAs, so every instruction between two inputs'
// bursts can idle it).
// O blocks first touched by input (ST, IH, IW): their o_empty waits.
template <int ST, int IH, int IW>
__host__ __device__ constexpr uint32_t new_blocks() {
  uint32_t m = 0;
  for (int oh = 0; oh < kG; ++oh)
    for (int ow = 0; ow < kG; ++ow)
      if (first_at(ST, IH, IW, oh, ow)) m |= 1u << block(ST, oh, ow);
  return m;
}

// Everything input n needs before its UMMAs: its A2 slot filled, and the
// previous occupants of the O blocks it touches first drained.  `ouse` holds
// the blocks' use parities BEFORE this input's first touches.
template <int ST, int IH, int IW>
__device__ __forceinline__ void wait_input(const Ctx& c, uint32_t n, uint32_t ouse) {
  mbar_wait(&c.b.a2_full[n & 1u], (n >> 1) & 1u);
  constexpr uint32_t m = new_blocks<ST, IH, IW>();
#pragma unroll
  for (int b = 0; b < 12; ++b)
    if (m & (1u << b)) mbar_wait(&c.b.o_empty[b], ((ouse >> b) & 1u) ^ 1u);
  tc_fence_after();
}

// Input (IH, IW) of strip ST: A2 slot n & 1 into every output it feeds.
// (Measured and dropped: running the NEXT input's waits inside this input's
// UMMA burst -- blocking there costs 20 %, a non-blocking test gains nothing.)
template <bool kTr, int ST, int IH, int IW>
__device__ __forceinline__ void sweep_input(Ctx& c, uint32_t n) {
  constexpr int q = IH % 3;
  constexpr int jlo = ow0(ST) - (IW - 1) > 0 ? ow0(ST) - (IW - 1) : 0;
  constexpr int jhi = ow0(ST) + nw(ST) - IW < 2 ? ow0(ST) + nw(ST) - IW : 2;
  constexpr int nj = jhi - jlo + 1;
  constexpr int rlo = IH == 0 ? 1 : 0;             // row -1 does not exist
  constexpr int nr = IH == 0 || IH == kG - 1 ? 2 : 3;  // nor row 7
  const uint32_t slot = n & 1u;
  unsigned long long* trace = c.trace;
  if constexpr (kTr) TRACE(6, static_cast<int>(n));
  wait_input<ST, IH, IW>(c, n, c.ouse);
  c.ouse ^= new_blocks<ST, IH, IW>();
  if constexpr (kTr) TRACE(7, static_cast<int>(n));
  Ctx cw = c;
  asm volatile("" : "+l"(cw.w2d), "+r"(cw.tbase));
  const uint32_t a = cw.tbase + kTmA2 + 32u * slot;
  const uint32_t d0 = cw.tbase + kTmO + 96u * (IW - 1 + jlo - ow0(ST));
  const uint32_t blo = static_cast<uint32_t>(cw.w2d) + (q * kQBytes >> 4) + 32u * 3u * jlo;
  const uint32_t bhi = static_cast<uint32_t>(cw.w2d >> 32);
  if (elect_one()) {
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const uint32_t bk = blo + ((ks * 2 * 288 * 16) >> 4);
      const uint32_t ak = a + 8u * ks;
      if constexpr (nr == 3) {
        if constexpr (nj == 3) {
          mma<160>(d0, ak, desc64(bk, bhi));
          mma<128>(d0 + 160u, ak, desc64(bk + 160u, bhi));
        } else {
          mma<96 * nj>(d0, ak, desc64(bk, bhi));
        }
      } else {
#pragma unroll
        for (int j = 0; j < nj; ++j)
          mma<64>(d0 + 96u * j + 32u * rlo, ak, desc64(bk + 96u * j + 32u * rlo, bhi));
      }
    }
    umma_commit(&c.b.a2_empty[slot]);
    if constexpr (kTr)
      if (c.trace) umma_commit(c.done);
#pragma unroll
    for (int oh = 0; oh < kG; ++oh)
#pragma unroll
      for (int ow = 0; ow < kG; ++ow)
        if (last_at(ST, IH, IW, oh, ow)) umma_commit(&c.b.o_full[block(ST, oh, ow)]);
  }
  __syncwarp();
  if constexpr (kTr) TRACE(8, static_cast<int>(n));
}

template <bool kTr, int ST, int IH>
__device__ __forceinline__ void sweep_row(Ctx& c, uint32_t& n) {
  sweep_input<kTr, ST, IH, c0(ST)>(c, n++);
  sweep_input<kTr, ST, IH, c0(ST) + 1>(c, n++);
  sweep_input<kTr, ST, IH, c0(ST) + 2>(c, n++);
  sweep_input<kTr, ST, IH, c0(ST) + 3>(c, n++);
  if constexpr (ST == 0) sweep_input<kTr, ST, IH, 4>(c, n++);
}

template <bool kTr, int ST>
__device__ __forceinline__ void sweep_strip(Ctx& c, uint32_t& n) {
  sweep_row<kTr, ST, 0>(c, n);
  sweep_row<kTr, ST, 1>(c, n);
  sweep_row<kTr, ST, 2>(c, n);
  sweep_row<kTr, ST, 3>(c, n);
  sweep_row<kTr, ST, 4>(c, n);
  sweep_row<kTr, ST, 5>(c, n);
  sweep_row<kTr, ST, 6>(c, n);
}

template <bool kTr>
__global__ void __launch_bounds__(kThreads, 1)
    conv_sweep_sm100(const __grid_constant__ CUtensorMap tm_out, const ConvRowsArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* bar0 = reinterpret_cast<uint64_t*>(smem + kOffBar);
  Bars B;
  B.a1_full = bar0;
  B.a1_empty = B.a1_full + kA1Stages;
  B.c1_full = B.a1_empty + kA1Stages;
  B.c1_empty = B.c1_full + 1;
  B.a2_full = B.c1_empty + 1;
  B.a2_empty = B.a2_full + 2;
  B.o_full = B.a2_empty + 2;
  B.o_empty = B.o_full + 12;
  uint64_t* const done_bar = B.o_empty + 12;  // trace only: conv2 input completions
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done_bar + 1);
  es::Bars rb;  // the builders' view (a1 ring only)
  rb.a1_full = B.a1_full;
  rb.a1_empty = B.a1_empty;

  const int warp = warp_uniform_id();
  const int lane = threadIdx.x & 31;
  unsigned long long* const trace = kTr && blockIdx.x == 0 ? args.trace : nullptr;
  const long long row_begin = args.claim ? args.claim->row_begin : args.row_begin;
  const long long row_end = args.claim ? args.claim->row_end : args.row_end;
  const long long tiles = (row_end - row_begin + kTile - 1) / kTile;
  const int my_tiles =
      blockIdx.x < tiles ? static_cast<int>((tiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kA1Stages; ++i) {
      mbar_init(&B.a1_full[i], kBuilders);
      mbar_init(&B.a1_empty[i], 1);
    }
    mbar_init(B.c1_full, 1);
    mbar_init(B.c1_empty, kEpi);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.a2_full[i], kEpi);
      mbar_init(&B.a2_empty[i], 1);
    }
    for (int i = 0; i < 12; ++i) {
      mbar_init(&B.o_full[i], 1);
      mbar_init(&B.o_empty[i], 4);
    }
    mbar_init(done_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);

  // Resident weights.  W2 copy q -> [ks][plane][row = 32 k + co][8 ci], block
  // k = 3 j + r holding tap (dh = (q + 2 - r) mod 3, dw = 2 - j).  W1 as in
  // conv_rows_sm100.
  {
    const uint4* w2 = static_cast<const uint4*>(args.w2);  // [32][72 chunks of 8]
    for (int i = threadIdx.x; i < 3 * 288 * 8; i += kThreads) {
      const int q = i / 2304, rem = i % 2304, row = rem >> 3, ch = rem & 7;
      const int ks = ch >> 1, pl = ch & 1, k = row >> 5, co = row & 31;
      const int j = k / 3, r = k % 3, dh = (q + 2 - r) % 3, dw = 2 - j;
      *reinterpret_cast<uint4*>(smem + kOffW2 + q * kQBytes + (ks * 2 + pl) * (288 * 16) + row * 16) =
          w2[co * 72 + (3 * dh + dw) * 8 + ch];
    }
    const uint4* w1 = static_cast<const uint4*>(args.w1);  // [64][2 chunks of 8]
    for (int i = threadIdx.x; i < 2 * 64; i += kThreads) {
      const int cc = i >> 1, pl = i & 1;
      *reinterpret_cast<uint4*>(smem + kOffW1 + (pl * 64 + cc) * 16) = w1[i];
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const int role = role_of(warp);
  if (role == kRDrain) {  // O starts at zero (every UMMA accumulates)
    uint32_t z[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) z[i] = 0u;
    const uint32_t lf = static_cast<uint32_t>((warp & 3) * 32) << 16;
#pragma unroll
    for (int cb = 0; cb < 12; ++cb) tmem_st32(tmem_base + lf + kTmO + 32u * cb, z);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (role == kRBuild) {
    // --------------------------------------------- im2col builders (as conv_rows)
    int n = 0;
    for (int k = 0; k < my_tiles; ++k) {
      const long long s0 = row_begin + (blockIdx.x + static_cast<long long>(k) * gridDim.x) * kTile;
      // the next tile's images (contiguous rows of x) into L2 while this one is built
      const long long s1 = s0 + static_cast<long long>(gridDim.x) * kTile;
      if (warp == 0 && lane == 0 && k + 1 < my_tiles) {
        const long long e1 = s1 + kTile < args.x_rows ? s1 + kTile : args.x_rows;
        if (e1 > s1)
          // evict_last: the drain's output stream (2x the image bytes) passes
          // through L2 before this tile is built and evicted the plain prefetch
          prefetch_l2_bulk_hint(static_cast<const uint8_t*>(args.x) + s1 * (kS * kS * 2),
                                static_cast<uint32_t>((e1 - s1) * (kS * kS * 2)), l2_policy_evict_last());
      }
      const int bw = role_idx(warp);
      const int smp = bw * 32 + lane;
      const long long s = s0 + smp;
      const uint8_t* xs = static_cast<const uint8_t*>(args.x) + s * (kS * kS * 2);
      const uint8_t* xn = s + static_cast<long long>(gridDim.x) * kTile < args.x_rows && k + 1 < my_tiles
                              ? xs + static_cast<long long>(gridDim.x) * kTile * (kS * kS * 2)
                              : nullptr;  // the next tile's first patch row
      const bool in = s < args.x_rows;
      for (int ih = 0; ih < kG; ++ih) {
        build_row_sweep<0>(args, smem, rb, s, ih, smp, lane, n,
                           !in ? nullptr : ih + 1 < kG ? xs + 224 * (ih + 1) : xs);
        if (warp == 0 && lane == 0) TRACE(1, n);
        n += 5;
      }
      for (int ih = 0; ih < kG; ++ih) {
        build_row_sweep<1>(args, smem, rb, s, ih, smp, lane, n,
                           !in ? nullptr : ih + 1 < kG ? xs + 224 * (ih + 1) : xn);
        if (warp == 0 && lane == 0) TRACE(1, n);
        n += 4;
      }
    }
  } else if (role == kRConv1) {
    // ------------------------------------------------------- conv1 issuer
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t a1_base = __shfl_sync(0xffffffffu, smem_u32(smem + kOffA1), 0);
    const uint64_t w1d = sdesc_planar(__shfl_sync(0xffffffffu, smem_u32(smem + kOffW1), 0), 1024);
    constexpr uint32_t id1 = idesc_bf16_f32(128, kC1);
    const int npos = my_tiles * 63;
    int sl = 0;
    uint32_t slpar = 0;
    for (int n = 0; n < npos; ++n) {
      mbar_wait(&B.a1_full[sl], slpar);
      if (lane == 0) TRACE(2, n);
      mbar_wait(B.c1_empty, (static_cast<uint32_t>(n) & 1u) ^ 1u);
      if (lane == 0) TRACE(12, n);
      tc_fence_after();
      if (elect_one()) {
        umma_bf16(tbase + kTmD1, sdesc_planar(a1_base + sl * kA1Bytes, 2048), w1d, id1, 0);
        umma_commit(B.c1_full);
        umma_commit(&B.a1_empty[sl]);
      }
      __syncwarp();
      if (++sl == kA1Stages) {
        sl = 0;
        slpar ^= 1u;
      }
    }
  } else if (role == kRConv2) {
    // ------------------------------------------------------- conv2 issuer
    Ctx c;
    c.tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    c.w2d = sdesc_planar(__shfl_sync(0xffffffffu, smem_u32(smem + kOffW2), 0), 288 * 16);
    c.b = B;
    c.ouse = 0;
    c.trace = trace;
    c.done = done_bar;
    uint32_t n = 0;
    for (int k = 0; k < my_tiles; ++k) {
      sweep_strip<kTr, 0>(c, n);
      sweep_strip<kTr, 1>(c, n);
    }
  } else if (role == kRWatch) {
    // trace only: completion time of every conv2 input (CTA 0)
    if (kTr && trace && lane == 0) {
      const int npos = my_tiles * 63;
      for (int n = 0; n < npos && n < 256; ++n) {
        mbar_wait(done_bar, static_cast<uint32_t>(n) & 1u);
        TRACE(13, n);
      }
    }
  } else if (role == kREpi) {
    // ---------------------------------------------------- conv1 epilogue
    // One warp per lane quadrant: relu(D1 + b1) of its 32 samples' 64
    // channels as bf16 pairs into A2 slot n & 1 (the conv2 UMMAs read A from
    // TMEM).
    const int e = role_idx(warp);
    constexpr int kCh = 64, h = 0;
    const uint32_t lf = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int npos = my_tiles * 63;
    for (int n = 0; n < npos; ++n) {
      mbar_wait(B.c1_full, static_cast<uint32_t>(n) & 1u);
      if (e == 0 && lane == 0) TRACE(3, n);
      const uint32_t slot = static_cast<uint32_t>(n) & 1u;
      tc_fence_after();
      uint32_t v[kCh];
#pragma unroll
      for (int c = 0; c < kCh / 32; ++c)
        tmem_ld32_raw(tmem_base + lf + kTmD1 + 32u * (h + c), *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(B.c1_empty);
      uint32_t pk[kCh / 2];
#pragma unroll
      for (int i = 0; i < kCh / 2; ++i)
        pk[i] = pack_relu_bf16(v[2 * i], v[2 * i + 1], args.b1c[32 * h + 2 * i], args.b1c[32 * h + 2 * i + 1]);
      mbar_wait(&B.a2_empty[slot], ((static_cast<uint32_t>(n) >> 1) & 1u) ^ 1u);
      if (e == 0 && lane == 0) TRACE(4, n);
      tc_fence_after();
      tmem_st32(tmem_base + lf + kTmA2 + 32u * slot, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&B.a2_full[slot]);
      if (e == 0 && lane == 0) TRACE(5, n);
    }
  } else {
    // ---------------------------------------------------------- output drain
    // Blocks in completion order: read, zero (the block's next row starts at
    // 0), release, then bias + ReLU + bf16 into a swizzled staging box that
    // one TMA store writes as 32 rows x 64 B (per-lane 16-byte stores to rows
    // 3136 B apart were LSU-bound: the drain, not the tensor pipe, set the
    // kernel's pace).  A partial last tile takes per-lane stores of its valid
    // rows instead (a claimed run must not write past its rows).
    const int dw = role_idx(warp), qd = warp & 3;
    const uint32_t lf = static_cast<uint32_t>(qd * 32) << 16;
    const int row = qd * 32 + lane;
    uint8_t* const ring = smem + kOffOut + dw * (kOutStages * kOutBox);
    int seq = 0;
    uint32_t z[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) z[i] = 0u;
    uint32_t opar = 0, nst = 0;
    const uint64_t out_policy = l2_policy_evict_first();  // read back by the next launch only
    for (int k = 0; k < my_tiles; ++k) {
      const long long s0 = row_begin + (blockIdx.x + static_cast<long long>(k) * gridDim.x) * kTile;
      const long long s = s0 + row;
      uint8_t* dst_row = static_cast<uint8_t*>(args.out) + s * (kOutRow * 2);
      const bool valid = s < row_end;
      const bool full = s0 + kTile <= row_end;
#pragma unroll 1
      for (int i = 0; i < kG * kG; ++i) {
        const int b = kDrainSeq.blk[i], p = kDrainSeq.pos[i];
        const uint32_t par = (opar >> b) & 1u;
        opar ^= 1u << b;
        ++seq;
        mbar_wait(&B.o_full[b], par);
        unsigned long long* const tr = qd == 0 && lane == 0 ? trace : nullptr;
        { unsigned long long* trace = tr; TRACE(9, seq); }
        tc_fence_after();
        uint32_t v[32];
        const uint32_t src = tmem_base + lf + kTmO + 32u * b;
        tmem_ld32_raw(src, v);
        tmem_ld_wait();
        tmem_st32(src, z);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&B.o_empty[b]);
        { unsigned long long* trace = tr; TRACE(10, seq); }
        uint4 q[4];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
          q[cc] = make_uint4(
              pack_relu_bf16(v[8 * cc], v[8 * cc + 1], args.b2c[8 * cc], args.b2c[8 * cc + 1]),
              pack_relu_bf16(v[8 * cc + 2], v[8 * cc + 3], args.b2c[8 * cc + 2], args.b2c[8 * cc + 3]),
              pack_relu_bf16(v[8 * cc + 4], v[8 * cc + 5], args.b2c[8 * cc + 4], args.b2c[8 * cc + 5]),
              pack_relu_bf16(v[8 * cc + 6], v[8 * cc + 7], args.b2c[8 * cc + 6], args.b2c[8 * cc + 7]));
        if (full && !kDirectStores) {
          uint8_t* box = ring + (nst % kOutStages) * kOutBox;
          if (lane == 0) tma_store_wait_read<kOutStages - 1>();  // the box's last store read it
          __syncwarp();
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            *reinterpret_cast<uint4*>(box + lane * 64 + ((cc ^ ((lane >> 1) & 3)) << 4)) = q[cc];
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d_hint(&tm_out, box, p * kC2, static_cast<int32_t>(s0 + qd * 32), out_policy);
            tma_store_commit();
          }
          ++nst;
        } else if (valid) {  // partial tile (or kDirectStores): per-lane 64-byte stores
          uint4* dst = reinterpret_cast<uint4*>(dst_row + p * kC2 * 2);
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) dst[cc] = q[cc];
        }
        { unsigned long long* trace = tr; TRACE(11, seq); }
      }
    }
    if (lane == 0) tma_store_wait_all<0>();
    __syncwarp();
  }

  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace sweep

}  // namespace

bool conv_rows_supported(int S, int P, int c1, int c2) {
  return S == kS && P == 4 && c1 == kC1 && c2 == kC2;
}

int conv_rows_launch(const ConvRowsArgs& args, const void* x, long long x_rows, int grid,
                     cudaStream_t stream) {
  if (x_rows > INT_MAX) return -1;
  // with a claim, [row_begin, row_end) is the worker's whole range (the grid
  // covers any run the claim can hold), as for conv_launch
  const long long tiles = (args.row_end - args.row_begin + kTile - 1) / kTile;
  if (tiles <= 0) return 0;
  grid = static_cast<int>(std::min<long long>(grid, tiles));
  if (ensure_smem_attr(conv_rows_sm100, static_cast<int>(kSmemBytes)) != 0) return -4;
  ConvRowsArgs a = args;
  a.x = x;
  a.x_rows = x_rows;
  conv_rows_sm100<<<grid, kThreads, kSmemBytes, stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int conv_sweep_launch(const ConvRowsArgs& args, const void* x, long long x_rows, int grid,
                      cudaStream_t stream) {
  if (x_rows > INT_MAX) return -1;
  const long long tiles = (args.row_end - args.row_begin + kTile - 1) / kTile;
  if (tiles <= 0) return 0;
  grid = static_cast<int>(std::min<long long>(grid, tiles));
  if (ensure_smem_attr(sweep::conv_sweep_sm100<false>, static_cast<int>(sweep::kSmemBytes)) != 0 ||
      ensure_smem_attr(sweep::conv_sweep_sm100<true>, static_cast<int>(sweep::kSmemBytes)) != 0)
    return -4;
  // output rows [0, row_end): TMA stores only ever cover whole tiles inside it
  CUtensorMap tm_out;
  if (make_bf16_map_box(&tm_out, args.out, kOutRow, static_cast<uint64_t>(args.row_end), 32, 32,
                        CU_TENSOR_MAP_SWIZZLE_64B) != 0)
    return -2;
  ConvRowsArgs a = args;
  a.x = x;
  a.x_rows = x_rows;
  if (a.trace)
    sweep::conv_sweep_sm100<true><<<grid, sweep::kThreads, sweep::kSmemBytes, stream>>>(tm_out, a);
  else
    sweep::conv_sweep_sm100<false><<<grid, sweep::kThreads, sweep::kSmemBytes, stream>>>(tm_out, a);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace es
