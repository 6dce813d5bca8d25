// Convolution stack of the CNN member (design in conv_kernel.cuh).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "conv_kernel.cuh"
#include "sm100.cuh"
#include "tma_host.hpp"

namespace es {

using namespace sm100;

namespace {

// w0 TMA producer + im2col builder, w1 UMMA issuer, w2..w5 conv1 epilogue,
// w6..w9 conv2 epilogue (each group covers the four TMEM lane quadrants).
// Ten warps: extra role warps share the UMMA warp's sub-partition and slow its
// issue loop down (measured with tools/trace_conv.cu).
constexpr int kThreads = 320;
// split schedule: four more conv2-epilogue warps (10-13), see epi2_split.
template <int SPLIT>
constexpr int threads_for() { return SPLIT ? 480 : kThreads; }  // split: + warp 14, the conv2 issuer
constexpr uint32_t kSmemBudget = 232448;
constexpr int kShiftPipe = 0, kShiftShfl = 1, kShiftHybrid = 2;  // ConvArgs::shifts
constexpr int kMargin = 16;  // zero rows before/after the tile's grids; taps reach R+1 rows

// bf16x2 {relu(a + ba), relu(b + bb)} (a in the low half), one cvt.relu.
__device__ __forceinline__ uint32_t pack_relu_bf16(uint32_t a, uint32_t b, float ba, float bb) {
  const float lo = __uint_as_float(a) + ba;
  const float hi = __uint_as_float(b) + bb;
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Stamp slot i of local tile k (CTA 0 only; slots listed in tools/trace_conv.cu).
#define TRACE(k, i)                                                                         \
  do {                                                                                      \
    if (args.trace && blockIdx.x == 0 && (k) < 32) args.trace[(k) * 16 + (i)] = global_ns(); \
  } while (0)

// KP2 = c1 / 16: K steps per tap, unrolled so the issue loop is pure uniform
// adds (tools/umma_rate.cu).  SPLIT: 0 = tap schedule, else the split
// schedule with ConvArgs::shifts = SPLIT - 1 (conv_kernel.cuh), a template
// argument because a runtime switch in the issue and epilogue loops measured
// 50 % slower.
template <int KP2, int SPLIT>
__global__ void __launch_bounds__(threads_for<SPLIT>(), 1)
    conv_stack_sm100(const __grid_constant__ CUtensorMap tm_x, const ConvArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const ConvLayout& L = args.L;
  uint8_t* sRaw = smem + L.off_raw;
  uint8_t* sA1 = smem + L.off_a1;
  uint8_t* sA2 = smem + L.off_a2;
  uint8_t* sW1 = smem + L.off_w1;
  uint8_t* sW2 = smem + L.off_w2;
  float* sB1 = reinterpret_cast<float*>(smem + L.off_b1);
  int* sRowOff = reinterpret_cast<int*>(smem + L.off_rows);  // im2col source offset per row
  int* sGrow = sRowOff + L.T * L.G * L.G;  // conv1 output row -> grid row
  int* sOut = sGrow + L.T * L.G * L.G;     // grid row -> (sample << 24 | byte offset), -1 = border
  uint64_t* raw_full = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* a1_full = raw_full + 2 * L.raw_stages;  // every pair below: one per buffer
  uint64_t* a1_empty = a1_full + 2;
  uint64_t* c1_full = a1_empty + 2;
  uint64_t* c1_empty = c1_full + 2;
  uint64_t* a2_full = c1_empty + 2;
  uint64_t* a2_empty = a2_full + 2;
  uint64_t* c2_full = a2_empty + 2;  // [3]: conv2 accumulator slots (split: 3, tap: 2)
  uint64_t* c2_empty = c2_full + 3;
  uint64_t* mma_done = c2_empty + 3;  // [3] split: a block's UMMAs completed (shifts may go)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_done + 3);

  const int warp = warp_uniform_id();
  const int lane = threadIdx.x & 31;
  // Rows of this launch: its static range, or the data-parallel claim.
  const long long row_begin = args.claim ? args.claim->row_begin : args.row_begin;
  const long long row_end = args.claim ? args.claim->row_end : args.row_end;
  const long long tiles = (row_end - row_begin + L.T - 1) / L.T;
  const int my_tiles =
      blockIdx.x < tiles ? static_cast<int>((tiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int kp = L.c1 / 8;  // 16-byte planes of conv2's K per tap

  if (threadIdx.x == 0) {
    for (int s = 0; s < L.raw_stages; ++s) {
      mbar_init(&raw_full[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&a1_full[b], 1);
      mbar_init(&a1_empty[b], 1);
      mbar_init(&c1_full[b], 1);
      mbar_init(&c1_empty[b], SPLIT ? 8 : 4);
      mbar_init(&a2_full[b], SPLIT ? 256 : 128);
      mbar_init(&a2_empty[b], 1);
    }
    for (int sl = 0; sl < 3; ++sl) {
      mbar_init(&c2_full[sl], 1);
      mbar_init(&c2_empty[sl], 4);
      mbar_init(&mma_done[sl], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch(&tm_x);
  if (warp == 1) tmem_alloc(tmem_slot, static_cast<uint32_t>(L.tmem_cols));

  // Resident operands: weights in the planar K-major layout (plane k of row o
  // = K elements 8k..8k+7), biases, and both grid buffers zeroed once -- the
  // conv1 epilogue only ever rewrites interior rows, so borders stay zero.
  {
    const uint4* w1 = static_cast<const uint4*>(args.w1);  // [c1][16] bf16 = 2 chunks per row
    for (int i = threadIdx.x; i < L.c1 * 2; i += threads_for<SPLIT>()) {
      const int o = i >> 1, k = i & 1;
      *reinterpret_cast<uint4*>(sW1 + (k * L.c1 + o) * 16) = w1[i];
    }
    const uint4* w2 = static_cast<const uint4*>(args.w2);  // [c2][9*c1] bf16 = 9*kp chunks per row
    for (int i = threadIdx.x; i < 9 * kp * L.c2; i += threads_for<SPLIT>()) {
      const int o = i / (9 * kp), rem = i % (9 * kp);  // rem = tap * kp + plane
      if (SPLIT) {
        // [dh][plane][dw*c2 + o]: B of UMMA (dh, K step) holds the three dw taps.
        const int tap = rem / kp, plane = rem % kp, dhi = tap / 3, dwi = tap % 3;
        *reinterpret_cast<uint4*>(sW2 + ((dhi * kp + plane) * L.n2 + dwi * L.c2 + o) * 16) = w2[i];
      } else {
        *reinterpret_cast<uint4*>(sW2 + (rem * L.c2 + o) * 16) = w2[i];
      }
    }
    for (int r = threadIdx.x; r < L.T * L.G * L.G; r += threads_for<SPLIT>()) {
      const int G2r = L.G * L.G, n = r / G2r, p = r % G2r, i = p / L.G, j = p % L.G;
      sRowOff[r] = (n * L.S * L.S + (4 * i) * L.S + 4 * j) * 2;  // patch (i, j) of sample n
      sGrow[r] = kMargin + n * L.R * L.R + (i + 1) * L.R + j;     // column G is the border
    }
    for (int r = threadIdx.x; r < L.mb2 * 128; r += threads_for<SPLIT>()) {
      const int P2r = L.R * L.R, n = r / P2r, rr = r % P2r, h = rr / L.R, w = rr % L.R;
      sOut[r] = (r < L.T * P2r && h >= 1 && w < L.G) ? (n << 24) | (((h - 1) * L.G + w) * L.c2 * 2) : -1;
    }
    for (int i = threadIdx.x; i < L.c1; i += threads_for<SPLIT>()) sB1[i] = args.b1[i];
    uint4* z = reinterpret_cast<uint4*>(sA2);
    for (int i = threadIdx.x; i < static_cast<int>(2 * L.a2_bytes / 16); i += threads_for<SPLIT>())
      z[i] = make_uint4(0, 0, 0, 0);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  const int G2 = L.G * L.G, P2 = L.R * L.R;

  if (warp == 0) {
    // ---------------------------------------------- TMA producer + im2col build
    // One warp: lane 0 keeps raw_stages image loads in flight; the whole warp
    // writes conv1's im2col rows of tile k (one row per output pixel: the
    // 4x4 patch as two 16-byte K planes), then refills the freed stage.
    // Source offsets per row come from a table, so the loop is loads/stores.
    // (A second builder warp measured no faster.)
    const uint64_t pol = l2_policy_evict_first();
    const int rows16 = L.S * L.S / 16;  // the map views x as [rows * S*S/16][16]
    auto load = [&](int k) {
      const int st = k % L.raw_stages;
      const long long s0 = row_begin + (blockIdx.x + static_cast<long long>(k) * gridDim.x) * L.T;
      mbar_arrive_expect_tx(&raw_full[st], static_cast<uint32_t>(L.T * L.S * L.S * 2));
      tma_load_2d(sRaw + st * L.raw_stride, &tm_x, &raw_full[st], 0,
                  static_cast<int32_t>(s0 * rows16), pol);
      TRACE(k, 0);
    };
    if (lane == 0)
      for (int k = 0; k < my_tiles && k < L.raw_stages; ++k) load(k);
    const int rows = L.T * G2;
    for (int k = 0; k < my_tiles; ++k) {
      const int st = k % L.raw_stages;
      const int b = k & 1;
      mbar_sleep_wait(&raw_full[st], static_cast<uint32_t>(k / L.raw_stages) & 1u);
      mbar_sleep_wait(&a1_empty[b], (static_cast<uint32_t>(k >> 1) & 1u) ^ 1u);
      if (lane == 0) TRACE(k, 4);
      const uint8_t* raw = sRaw + st * L.raw_stride;
      uint8_t* a1 = sA1 + b * L.a1_bytes;
      for (int r = lane; r < rows; r += 32) {
        const uint8_t* src = raw + sRowOff[r];
        const uint2 v0 = *reinterpret_cast<const uint2*>(src);
        const uint2 v1 = *reinterpret_cast<const uint2*>(src + L.S * 2);
        const uint2 v2 = *reinterpret_cast<const uint2*>(src + L.S * 4);
        const uint2 v3 = *reinterpret_cast<const uint2*>(src + L.S * 6);
        *reinterpret_cast<uint4*>(a1 + r * 16) = make_uint4(v0.x, v0.y, v1.x, v1.y);
        *reinterpret_cast<uint4*>(a1 + L.a1_plane + r * 16) = make_uint4(v2.x, v2.y, v3.x, v3.y);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&a1_full[b]);
        TRACE(k, 5);
        if (k + L.raw_stages < my_tiles) load(k + L.raw_stages);  // stage st is free again
      }
      __syncwarp();
    }
  } else if (warp == 1 || (SPLIT && warp == 14)) {
    // ------------------------------------------------------------ UMMA issuer
    // The whole warp walks the schedule (uniform descriptor arithmetic); one
    // elected lane issues.  Descriptors advance by adding 16-byte units to
    // the start-address field: taps move the A start by whole grid rows.
    // __shfl_sync(.., 0) marks the bases warp-uniform for the compiler.
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t a1_base = __shfl_sync(0xffffffffu, smem_u32(sA1), 0);
    const uint32_t a2_base = __shfl_sync(0xffffffffu, smem_u32(sA2), 0);
    const uint32_t id1 = idesc_bf16_f32(128, L.c1), id2 = idesc_bf16_f32(128, L.n2);
    const uint64_t w1d = sdesc_planar(__shfl_sync(0xffffffffu, smem_u32(sW1), 0),
                                      static_cast<uint32_t>(L.c1 * 16));
    const uint64_t w2d = sdesc_planar(__shfl_sync(0xffffffffu, smem_u32(sW2), 0),
                                      static_cast<uint32_t>(L.n2 * 16));
    const uint32_t a2_step = L.a2_plane / 8;  // two planes (K += 16), in 16-byte units
    auto conv1 = [&](int k) {
      const int b = k & 1;
      const uint32_t u = static_cast<uint32_t>(k >> 1) & 1u;
      // conv1 accumulators: split keeps ONE buffer (its epilogue releases it
      // as soon as the values are in registers) so TMEM holds 3 conv2 slots.
      const int cb = SPLIT ? 0 : b;
      const uint32_t cu = SPLIT ? static_cast<uint32_t>(k) & 1u : u;
      mbar_sleep_wait(&a1_full[b], u);
      mbar_sleep_wait(&c1_empty[cb], cu ^ 1u);
      TRACE(k, 1);
      tc_fence_after();
      const uint64_t ad = sdesc_planar(a1_base + b * L.a1_bytes, L.a1_plane);
      for (int mb = 0; mb < L.mb1; ++mb)
        if (elect_one())
          umma_bf16(tbase + static_cast<uint32_t>(cb * L.tmem_c1 + mb * L.c1),
                    ad + static_cast<uint64_t>(mb * 128), w1d, id1, 0);
      if (elect_one()) {
        umma_commit(&a1_empty[b]);
        umma_commit(&c1_full[cb]);
      }
      __syncwarp();
    };
    // split: warp 14 issues conv2's UMMAs and the tensor-pipe lane shifts of
    // args.shifts (conv_kernel.cuh).  tcgen05.shift is not ordered behind
    // in-flight UMMAs on the same columns (measured: shifting right after the
    // UMMAs reads partial sums), so a block's shifts go out after the NEXT
    // block's UMMAs are queued, once its own UMMA commit has landed -- the
    // pipe never drains, and UMMAs + shifts come from one issuer (two issuers
    // cost ~25 %, tools/umma_rate.cu).  Warp 1 issues only the conv1 UMMAs.
    constexpr int shifts = SPLIT - 1;
    int pend_blk = -1;
    auto shift_block = [&](int blk) {
      const int sl = blk % 3;
      mbar_sleep_wait(&mma_done[sl], static_cast<uint32_t>(blk / 3) & 1u);
      tc_fence_after();
      const uint32_t d = tbase + static_cast<uint32_t>(L.tmem_c1 + sl * L.n2);
      for (int c = 0; c < L.c2; c += 8) {
        if constexpr (shifts == kShiftPipe)
          if (elect_one()) tmem_shift_down(d + static_cast<uint32_t>(L.c2 + c));
        if (elect_one()) tmem_shift_down(d + static_cast<uint32_t>(2 * L.c2 + c));
        if constexpr (shifts == kShiftPipe)
          if (elect_one()) tmem_shift_down(d + static_cast<uint32_t>(2 * L.c2 + c));
      }
      if (elect_one()) umma_commit(&c2_full[sl]);
      __syncwarp();
    };
    auto conv2_split = [&](int k) {
      // One accumulator slot per 128-row block, alternating over the running
      // block count: the epilogue of block i overlaps the UMMAs of block i+1.
      const int b = k & 1;
      const uint32_t u = static_cast<uint32_t>(k >> 1) & 1u;
      mbar_sleep_wait(&a2_full[b], u);
      TRACE(k, 2);
      const uint64_t ad0 = sdesc_planar(a2_base + b * L.a2_bytes, L.a2_plane);
      for (int mb = 0; mb < L.mb2; ++mb) {
        const int blk = k * L.mb2 + mb, sl = blk % 3;
        mbar_sleep_wait(&c2_empty[sl], (static_cast<uint32_t>(blk / 3) & 1u) ^ 1u);
        TRACE(k, 10 + 3 * mb);
        tc_fence_after();
        const uint32_t d = tbase + static_cast<uint32_t>(L.tmem_c1 + sl * L.n2);
        const uint64_t adm = ad0 + static_cast<uint64_t>(kMargin + mb * 128);
        // D'[p][dw] = sum_dh X[p - 1 + dh*R] W(dh, dw): A shifted by dh*R - 1.
#pragma unroll
        for (int dhi = 0; dhi < 3; ++dhi)
#pragma unroll
          for (int j = 0; j < KP2; ++j) {
            const uint64_t ad =
                adm + static_cast<uint64_t>((dhi - 1) * L.R - 1 + j * static_cast<int>(a2_step));
            const uint64_t bd = w2d + static_cast<uint64_t>((dhi * KP2 + j) * 2 * L.n2);
            if (elect_one()) umma_bf16(d, ad, bd, id2, (dhi | j) != 0);
          }
        if (elect_one()) {
          umma_commit(shifts == kShiftShfl ? &c2_full[sl] : &mma_done[sl]);
          if (mb == L.mb2 - 1) umma_commit(&a2_empty[b]);
        }
        __syncwarp();
        TRACE(k, 11 + 3 * mb);
        if constexpr (shifts != kShiftShfl) {
          if (pend_blk >= 0) shift_block(pend_blk);
          pend_blk = blk;
        }
      }
      TRACE(k, 3);
    };
    auto conv2 = [&](int k) {
      if (SPLIT) {
        conv2_split(k);
        return;
      }
      const int b = k & 1;
      const uint32_t u = static_cast<uint32_t>(k >> 1) & 1u;
      mbar_sleep_wait(&a2_full[b], u);
      mbar_sleep_wait(&c2_empty[b], u ^ 1u);
      TRACE(k, 2);
      tc_fence_after();
      const uint64_t ad0 = sdesc_planar(a2_base + b * L.a2_bytes, L.a2_plane);
      for (int mb = 0; mb < L.mb2; ++mb) {
        const uint32_t d =
            tbase + static_cast<uint32_t>(2 * L.tmem_c1 + b * L.tmem_c2 + mb * L.c2);
        const uint64_t adm = ad0 + static_cast<uint64_t>(kMargin + mb * 128);
#pragma unroll
        for (int t = 0; t < 9; ++t)
#pragma unroll
          for (int j = 0; j < KP2; ++j) {
            // Output row q reads grid row q + (dh * R + dw) at tap (dh, dw).
            const uint64_t ad =
                adm + static_cast<uint64_t>((t / 3 - 1) * L.R + (t % 3 - 1) + j * static_cast<int>(a2_step));
            const uint64_t bd = w2d + static_cast<uint64_t>((t * KP2 + j) * 2 * L.c2);
            if (elect_one()) umma_bf16(d, ad, bd, id2, (t | j) != 0);
          }
      }
      if (elect_one()) {
        umma_commit(&a2_empty[b]);
        umma_commit(&c2_full[b]);
      }
      __syncwarp();
      TRACE(k, 3);
    };
    if (SPLIT) {
      if (warp == 1) {
        for (int k = 0; k < my_tiles; ++k) conv1(k);
      } else {
        for (int k = 0; k < my_tiles; ++k) conv2(k);
        if (pend_blk >= 0) shift_block(pend_blk);
      }
    } else {
      // conv1 runs one tile ahead of conv2 (conv2 of tile k waits for the
      // conv1 epilogue of tile k, which overlaps conv1 of tile k+1).
      for (int k = 0; k < my_tiles; ++k) {
        conv1(k);
        if (k > 0) conv2(k - 1);
      }
      if (my_tiles > 0) conv2(my_tiles - 1);
    }
  } else if (warp < (SPLIT ? 10 : 6)) {
    // ------------------------------------------------------- conv1 epilogue
    // tap: warps 2-5, all c1 channels; split: warps 2-9, two channel halves
    // (its conv2 epilogue is a lane-local sum and needs fewer warps).
    const int ta = threadIdx.x - 64;
    const int q = warp & 3;
    const int cbeg = SPLIT ? ((warp - 2) >> 2) * (L.c1 / 2) : 0;  // split: c1 = 64, 32 per warp
    const uint32_t lane_field = static_cast<uint32_t>(q * 32) << 16;
    const int rows = L.T * G2;
    // relu(acc + bias) as bf16 into grid buffer a2 for the 32 channels from c0.
    auto emit = [&](uint8_t* a2, int mb, int c0, const uint32_t (&v)[32], const float (&bias)[32]) {
      const int r = mb * 128 + q * 32 + lane;
      if (r >= rows || (args.debug & 2)) return;
      const int grow = sGrow[r];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int c = g * 8;
        const uint4 pk = make_uint4(pack_relu_bf16(v[c], v[c + 1], bias[c], bias[c + 1]),
                                    pack_relu_bf16(v[c + 2], v[c + 3], bias[c + 2], bias[c + 3]),
                                    pack_relu_bf16(v[c + 4], v[c + 5], bias[c + 4], bias[c + 5]),
                                    pack_relu_bf16(v[c + 6], v[c + 7], bias[c + 6], bias[c + 7]));
        *reinterpret_cast<uint4*>(a2 + (c0 / 8 + g) * L.a2_plane + grow * 16) = pk;
      }
    };
    auto load_bias = [&](int c0, float (&bias)[32]) {
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        const float4 b4 = *reinterpret_cast<const float4*>(sB1 + c0 + c);
        bias[c] = b4.x;
        bias[c + 1] = b4.y;
        bias[c + 2] = b4.z;
        bias[c + 3] = b4.w;
      }
    };
    float bias_w[32];  // split: this warp's 32 channels, loaded once
    if (SPLIT) load_bias(cbeg, bias_w);
    for (int k = 0; k < my_tiles; ++k) {
      const int b = k & 1;
      const uint32_t u = static_cast<uint32_t>(k >> 1) & 1u;
      uint8_t* a2 = sA2 + b * L.a2_bytes;
      if (SPLIT) {
        // One conv1 buffer: pull this warp's 2 x 32 values into registers,
        // release the TMEM, then convert and store.
        mbar_sleep_wait(&c1_full[0], static_cast<uint32_t>(k) & 1u);
        mbar_sleep_wait(&a2_empty[b], u ^ 1u);
        if (ta == 0) TRACE(k, 6);
        tc_fence_after();
        uint32_t v0[32], v1[32];
        tmem_ld32_raw(tmem_base + lane_field + static_cast<uint32_t>(cbeg), v0);
        if (L.mb1 > 1) tmem_ld32_raw(tmem_base + lane_field + static_cast<uint32_t>(L.c1 + cbeg), v1);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&c1_empty[0]);
        emit(a2, 0, cbeg, v0, bias_w);
        if (L.mb1 > 1) emit(a2, 1, cbeg, v1, bias_w);
      } else {
        mbar_sleep_wait(&c1_full[b], u);
        mbar_sleep_wait(&a2_empty[b], u ^ 1u);
        if (ta == 0) TRACE(k, 6);
        tc_fence_after();
        for (int mb = 0; mb < L.mb1; ++mb)
          for (int c0 = 0; c0 < L.c1; c0 += 32) {
            uint32_t v[32];
            if (args.debug & 1) {
#pragma unroll
              for (int c = 0; c < 32; ++c) v[c] = static_cast<uint32_t>(c);
            } else {
              tmem_ld32_raw(tmem_base + lane_field + static_cast<uint32_t>(b * L.tmem_c1 + mb * L.c1 + c0), v);
              tmem_ld_wait();
            }
            float bias[32];
            load_bias(c0, bias);
            emit(a2, mb, c0, v, bias);
          }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&c1_empty[b]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&a2_full[b]);
      if (ta == 0) TRACE(k, 7);
    }
  } else {
    // ---------------------------------------------------------- conv2 epilogue
    const int q = warp & 3;
    const uint32_t lane_field = static_cast<uint32_t>(q * 32) << 16;
    const int row_bytes = G2 * L.c2 * 2;
    // split: out[q] = D'[q][-1] + D'[q+1][0] + D'[q+2][+1] (conv_kernel.cuh),
    // the lane moves split between the tensor pipe and shuffles by
    // args.shifts.  Lane 30 would need lane 32's dw=+1 partial, which lies in
    // the next quadrant: it is zero (it reads the border column); lane 31 is
    // itself a border pixel and is not stored.  Warps 10-13, every channel,
    // 16 at a time.
    auto epi2_split = [&](int k) {
      const long long s0 = row_begin + (blockIdx.x + static_cast<long long>(k) * gridDim.x) * L.T;
      constexpr int shifts = SPLIT - 1;
      const float keep_p1 = lane == 30 ? 0.0f : 1.0f;
      const float keep_31 = lane == 31 ? 0.0f : 1.0f;  // kShiftHybrid: u[31] takes no dw=+1 term
      for (int mb = 0; mb < L.mb2; ++mb) {
        const int blk = k * L.mb2 + mb, sl = blk % 3;
        const uint32_t ph = static_cast<uint32_t>(blk / 3) & 1u;
        mbar_sleep_wait(&c2_full[sl], ph);
        if (warp == 10 && lane == 0 && mb == 0) TRACE(k, 8);
        tc_fence_after();
        const int r = mb * 128 + q * 32 + lane;  // grid row of the tile
        const int oo = sOut[r];
        const int n = oo >> 24;
        const bool valid = oo >= 0 && s0 + n < row_end;
        uint8_t* dst = static_cast<uint8_t*>(args.out) + (s0 + n) * row_bytes + (oo & 0xFFFFFF);
        const uint32_t col = tmem_base + lane_field + static_cast<uint32_t>(L.tmem_c1 + sl * L.n2);
        for (int c0 = 0; c0 < L.c2; c0 += 16) {
          uint32_t r0[16], r1[16], r2[16];
          if (args.debug & 4) {
#pragma unroll
            for (int c = 0; c < 16; ++c) r0[c] = r1[c] = r2[c] = static_cast<uint32_t>(c + lane);
          } else {
            tmem_ld16_raw(col + static_cast<uint32_t>(c0), r0);
            tmem_ld16_raw(col + static_cast<uint32_t>(L.c2 + c0), r1);
            tmem_ld16_raw(col + static_cast<uint32_t>(2 * L.c2 + c0), r2);
            tmem_ld_wait();
          }
          float v[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            if constexpr (shifts == kShiftPipe) {  // both partials already on this lane
              v[c] = __uint_as_float(r0[c]) + __uint_as_float(r1[c]) + keep_p1 * __uint_as_float(r2[c]);
            } else if constexpr (shifts == kShiftShfl) {
              const uint32_t g0 = __shfl_down_sync(0xffffffffu, r1[c], 1);
              const uint32_t g1 = __shfl_down_sync(0xffffffffu, r2[c], 2);
              v[c] = __uint_as_float(r0[c]) + __uint_as_float(g0) + keep_p1 * __uint_as_float(g1);
            } else {  // dw=+1 moved one lane by the pipe: u[p] = D'[p][0] + D'[p+1][+1]
              const float u = __uint_as_float(r1[c]) + keep_31 * __uint_as_float(r2[c]);
              v[c] = __uint_as_float(r0[c]) + __shfl_down_sync(0xffffffffu, u, 1);
            }
          }
          if (valid && !(args.debug & 16)) {
#pragma unroll
            for (int g = 0; g < 2; ++g) {
              const int c = g * 8;
              const float4 bl = make_float4(args.b2c[c0 + c], args.b2c[c0 + c + 1],
                                            args.b2c[c0 + c + 2], args.b2c[c0 + c + 3]);
              const float4 bh = make_float4(args.b2c[c0 + c + 4], args.b2c[c0 + c + 5],
                                            args.b2c[c0 + c + 6], args.b2c[c0 + c + 7]);
              const uint4 pk = make_uint4(
                  pack_relu_bf16(__float_as_uint(v[c]), __float_as_uint(v[c + 1]), bl.x, bl.y),
                  pack_relu_bf16(__float_as_uint(v[c + 2]), __float_as_uint(v[c + 3]), bl.z, bl.w),
                  pack_relu_bf16(__float_as_uint(v[c + 4]), __float_as_uint(v[c + 5]), bh.x, bh.y),
                  pack_relu_bf16(__float_as_uint(v[c + 6]), __float_as_uint(v[c + 7]), bh.z, bh.w));
              *reinterpret_cast<uint4*>(dst + (c0 + c) * 2) = pk;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&c2_empty[sl]);
      }
      if (warp == 10 && lane == 0) TRACE(k, 9);
    };
    auto epi2 = [&](int k) {
      if (SPLIT) {
        epi2_split(k);
        return;
      }
      const int b = k & 1;
      const uint32_t u = static_cast<uint32_t>(k >> 1) & 1u;
      mbar_sleep_wait(&c2_full[b], u);
      if (warp == 6 && lane == 0) TRACE(k, 8);
      tc_fence_after();
      const long long s0 = row_begin + (blockIdx.x + static_cast<long long>(k) * gridDim.x) * L.T;
      for (int mb = 0; mb < L.mb2; ++mb) {
        const int r = mb * 128 + q * 32 + lane;  // grid row of the tile
        const int oo = sOut[r];
        const int n = oo >> 24;
        const bool valid = oo >= 0 && s0 + n < row_end;
        uint8_t* dst = static_cast<uint8_t*>(args.out) + (s0 + n) * row_bytes + (oo & 0xFFFFFF);
        for (int c0 = 0; c0 < L.c2; c0 += 32) {
          uint32_t v[32];
          tmem_ld32_raw(tmem_base + lane_field +
                            static_cast<uint32_t>(2 * L.tmem_c1 + b * L.tmem_c2 + mb * L.c2 + c0),
                        v);
          tmem_ld_wait();
          if (valid) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const int c = g * 8;
              const float4 bl = make_float4(args.b2c[c0 + c], args.b2c[c0 + c + 1],
                                            args.b2c[c0 + c + 2], args.b2c[c0 + c + 3]);
              const float4 bh = make_float4(args.b2c[c0 + c + 4], args.b2c[c0 + c + 5],
                                            args.b2c[c0 + c + 6], args.b2c[c0 + c + 7]);
              const uint4 pk = make_uint4(pack_relu_bf16(v[c], v[c + 1], bl.x, bl.y),
                                          pack_relu_bf16(v[c + 2], v[c + 3], bl.z, bl.w),
                                          pack_relu_bf16(v[c + 4], v[c + 5], bh.x, bh.y),
                                          pack_relu_bf16(v[c + 6], v[c + 7], bh.z, bh.w));
              *reinterpret_cast<uint4*>(dst + (c0 + c) * 2) = pk;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&c2_empty[b]);
      if (warp == 6 && lane == 0) TRACE(k, 9);
    };
    // conv1 of tile k+1 is issued before conv2 of tile k, so builds run two
    // tiles ahead: the build of tile k+1 never waits behind the epilogue of
    // tile k-1 (which waits for conv2 of tile k-1).
    for (int k = 0; k < my_tiles; ++k) epi2(k);
  }

  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, static_cast<uint32_t>(L.tmem_cols));
  }
}

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

}  // namespace

bool conv_plan(int S, int P, int c1, int c2, ConvLayout* out, int schedule) {
  // Default: split where a plan exists (shape allowed AND it fits TMEM/smem),
  // else tap.
  if (schedule == 0) return conv_plan(S, P, c1, c2, out, 2) || conv_plan(S, P, c1, c2, out, 1);
  if (P != 4 || S < P || S % P != 0 || (S * S) % 16 != 0) return false;
  if ((c1 != 32 && c1 != 64 && c1 != 128) || c2 < 32 || c2 % 32 != 0 || c2 > 256) return false;
  ConvLayout L;
  L.S = S;
  L.P = P;
  L.G = S / P;
  L.c1 = c1;
  L.c2 = c2;
  L.R = L.G + 1;
  if (L.R + 1 > kMargin) return false;
  const int P2 = L.R * L.R, G2 = L.G * L.G;
  // split: N = 3*c2 per UMMA; 128-row blocks and 32-lane quadrants must start
  // on grid-row boundaries (R | 32) so every quadrant's last lane is a border
  // column (the in-quadrant lane shift never needs the next quadrant).
  const bool split_ok = 3 * c2 <= 256 && 32 % L.R == 0 && c1 == 64;
  if (schedule == 2 && !split_ok) return false;
  // Measured on B200 (tools/trace_conv.cu, 2^20 CNN-s samples): split 2.63 ms
  // (one conv1 TMEM buffer + a 3-slot conv2 ring, conv2 UMMAs from one
  // issuer warp, lane shifts as epilogue shuffles, 8 conv1-epilogue warps,
  // row-address tables instead of divisions), tap 3.77 ms.
  L.split = split_ok && schedule != 1;
  L.n2 = L.split ? 3 * c2 : c2;
  for (int T = std::max(1, 256 / P2); T >= 1; --T) {
    L.T = T;
    L.mb1 = (T * G2 + 127) / 128;
    L.mb2 = (T * P2 + 127) / 128;
    if (T * S * S / 16 > 256) continue;  // TMA box rows
    L.tmem_c1 = L.mb1 * c1;
    // split: one N = 3*c2 slot per 128-row block, two slots; tap: a
    // double-buffered [mb2][c2] accumulator per tile.
    L.tmem_c2 = L.split ? L.n2 : L.mb2 * c2;
    // split: one conv1 buffer + a ring of 3 conv2 slots; tap: 2 + 2.
    const int cols = L.split ? L.tmem_c1 + 3 * L.tmem_c2 : 2 * (L.tmem_c1 + L.tmem_c2);
    if (cols > 512) continue;
    int tc = 32;
    while (tc < cols) tc <<= 1;
    L.tmem_cols = tc;
    L.raw_stages = 4;
    L.raw_stride = align_up(static_cast<uint32_t>(T * S * S * 2), 128);
    L.a1_plane = static_cast<uint32_t>(L.mb1 * 128 * 16);
    L.a1_bytes = 2 * L.a1_plane;
    L.a2_rows = static_cast<uint32_t>(kMargin + L.mb2 * 128 + kMargin);
    L.a2_plane = L.a2_rows * 16;
    L.a2_bytes = static_cast<uint32_t>(c1 / 8) * L.a2_plane;
    L.off_raw = 0;
    L.off_a1 = align_up(L.off_raw + L.raw_stages * L.raw_stride, 128);
    L.off_a2 = align_up(L.off_a1 + 2 * L.a1_bytes, 128);
    L.off_w1 = align_up(L.off_a2 + 2 * L.a2_bytes, 128);
    L.off_w2 = align_up(L.off_w1 + static_cast<uint32_t>(c1 * 32), 128);
    L.off_b1 = align_up(L.off_w2 + static_cast<uint32_t>(9 * c1 * c2 * 2), 16);
    L.off_b2 = align_up(L.off_b1 + static_cast<uint32_t>(c1 * 4), 16);
    L.off_rows = align_up(L.off_b2 + static_cast<uint32_t>(c2 * 4), 16);
    L.off_xch = align_up(L.off_rows + static_cast<uint32_t>((2 * T * G2 + L.mb2 * 128) * 4), 16);
    L.off_bar = align_up(L.off_xch, 8);
    const uint32_t bars = static_cast<uint32_t>(2 * L.raw_stages + 21) * 8u + 16u;
    L.smem_bytes = L.off_bar + bars + 1024u;  // + alignment slack of the dynamic base
    if (L.smem_bytes > kSmemBudget) continue;
    *out = L;
    return true;
  }
  return false;
}

int conv_launch(const ConvArgs& args, const void* x, long long x_rows, int grid, cudaStream_t stream) {
  const ConvLayout& L = args.L;
  const long long rows16 = x_rows * (L.S * L.S / 16);
  if (rows16 > INT_MAX) return -1;
  CUtensorMap mx;
  if (make_bf16_map_plain(&mx, x, 16, static_cast<uint64_t>(rows16),
                          static_cast<uint32_t>(L.T * L.S * L.S / 16)) != 0)
    return -1;
  const long long tiles = (args.row_end - args.row_begin + L.T - 1) / L.T;
  if (tiles <= 0) return 0;
  grid = static_cast<int>(std::min<long long>(grid, tiles));
  auto go = [&](auto kernel) {
    if (ensure_smem_attr(kernel, static_cast<int>(kSmemBudget)) != 0) return -4;
    kernel<<<grid, L.split ? threads_for<true>() : threads_for<false>(), L.smem_bytes, stream>>>(mx,
                                                                                                args);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
  };
  if (L.split) {  // split plans have c1 = 64 (conv_plan)
    if (L.c1 != 64) return -1;
    switch (args.shifts) {
      case kShiftPipe: return go(conv_stack_sm100<4, 1 + kShiftPipe>);
      case kShiftShfl: return go(conv_stack_sm100<4, 1 + kShiftShfl>);
      case kShiftHybrid: return go(conv_stack_sm100<4, 1 + kShiftHybrid>);
      default: return -1;
    }
  }
  switch (L.c1) {
    case 32: return go(conv_stack_sm100<2, 0>);
    case 64: return go(conv_stack_sm100<4, 0>);
    case 128: return go(conv_stack_sm100<8, 0>);
    default: return -1;
  }
}

}  // namespace es
