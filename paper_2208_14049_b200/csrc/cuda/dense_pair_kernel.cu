// Dense layer on SM PAIRS (tcgen05 cta_group::2): Y = act(X W^T + b), bf16.
//
// The single-SM dense kernel (dense_kernel.cu) streams the whole W chunk of a
// column block into every SM: a 784->512 layer at one 128-row tile per group
// needs 16 KB of X + 64 KB of W per 64-wide K chunk for 1024 clk of UMMA,
// 80 B/clk against the ~48 B/clk one SM's TMA ingress sustains
// (profiles/r1_summary.md).  Here the even CTA of a 2-CTA cluster issues M=256
// UMMAs for both SMs: each SM loads its own 128-row X tile and HALF of the W
// chunk (B split by N across the pair), 48 B/clk at the same tile shape.
//   TMA (both SMs):  X tile(s) + this SM's N/2 rows of the W chunk, bytes
//                    completing on the leader's stage barrier;
//   UMMA (leader):   D[256 x N] += X . W^T per 16-wide K step, commits
//                    multicast to both SMs;
//   epilogue (both): own 128 TMEM lanes -> +b, ReLU, bf16 -> 128B-swizzled
//                    staging -> TMA bulk store of its own rows; arrivals on
//                    the leader's accumulator barrier.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "dense_kernel.cuh"
#include "tma_host.hpp"

namespace es {

using namespace sm100;

namespace {

constexpr int kThreads = 320;  // w0 TMA, w1 TMEM + UMMA (leader), w2..w9 epilogue
constexpr uint32_t kSmemBudget = 232448;
constexpr uint32_t kMinSmem = 120 * 1024;
constexpr int kMaxT = 2;
constexpr uint16_t kBoth = 0b11;

// Unit i of this pair: T pair-tiles x one column block.  Pair-tile tp covers
// 128-row tiles 2*tp (even CTA) and 2*tp+1 (odd CTA).  Returns the number of
// pair-tiles (both CTAs agree); rows[k] = 0 marks this CTA's tile as absent
// (it still loads valid rows so the leader's byte count holds).
__device__ __forceinline__ int pair_unit(const DenseArgs& a, int i, uint32_t rank, int* cb,
                                         long long (&row0)[kMaxT], bool (&present)[kMaxT]) {
  const long long rb = a.claim ? a.claim->row_begin : a.row_begin;
  const long long tiles = ((a.claim ? a.claim->row_end : a.row_end) - rb + 127) / 128;
  const long long ptiles = (tiles + 1) / 2;
  const long long groups = (ptiles + a.L.T - 1) / a.L.T;
  const long long pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;
  const long long u = pair + static_cast<long long>(i) * pairs;
  if (u >= groups * a.L.ncb) return 0;
  *cb = static_cast<int>(u % a.L.ncb);
  const long long g = u / a.L.ncb;
  int n = 0;
  for (int k = 0; k < a.L.T; ++k) {
    const long long tp = g * a.L.T + k;
    if (tp >= ptiles) break;
    const long long t = 2 * tp + rank;
    present[k] = t < tiles;
    row0[k] = rb + (present[k] ? t : 2 * tp) * 128;
    ++n;
  }
  return n;
}

__device__ __forceinline__ void half_barrier(int half) {
  asm volatile("bar.sync %0, 128;" ::"r"(2 + half) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    dense_pair_sm100(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                     const __grid_constant__ CUtensorMap tm_y, const DenseArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const DenseLayout& L = args.L;
  uint8_t* sOut = smem + L.off_stage_out;  // [2 halves][128 rows][128 B]
  float* sBias = reinterpret_cast<float*>(smem + L.off_bias);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* full = bars;                  // [stages]  (leader's is used)
  uint64_t* empty = full + L.stages;      // [stages]  (each SM's own, multicast commit)
  uint64_t* acc_full = empty + L.stages;  // [2]       (multicast commit)
  uint64_t* acc_empty = acc_full + 2;     // [2]       (leader's; 16 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = warp_uniform_id();
  const int lane = threadIdx.x & 31;
  const int N = L.N;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 16);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_x);
    tma_prefetch(&tm_w);
    tma_prefetch(&tm_y);
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, static_cast<uint32_t>(L.tmem_cols));
  tc_fence_before();
  cluster_sync();  // barrier inits and TMEM of both SMs visible to both
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  long long row0[kMaxT];
  bool present[kMaxT];
  int cb = 0;
  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA (both SMs)
      const uint64_t pol_stream = l2_policy_evict_normal();  // evict_first on X cost the weights their L2 residency
      const uint64_t pol_keep = l2_policy_evict_last();
      const uint32_t half_w = static_cast<uint32_t>(L.NH / 2);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0;; ++i) {
        const int n = pair_unit(args, i, rank, &cb, row0, present);
        if (n == 0) break;
        for (int kc = 0; kc < L.kchunks; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* st = smem + static_cast<size_t>(stage) * L.stage_bytes;
          if (leader)
            mbar_arrive_expect_tx(&full[stage], 2u * (static_cast<uint32_t>(n) * 16384u +
                                                      static_cast<uint32_t>(N) * 64u));
          for (int k = 0; k < n; ++k)
            tma_load_2d_pair(st + k * 16384, &tm_x, &full[stage], kc * 64,
                             static_cast<int32_t>(row0[k]), pol_stream);
          uint8_t* sw = st + L.T * 16384;
          for (int h = 0; h < L.nh; ++h)
            tma_load_2d_pair(sw + h * half_w * 128u, &tm_w, &full[stage], kc * 64,
                             static_cast<int32_t>(cb * N + h * L.NH + rank * half_w), pol_keep);
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // the whole warp walks the schedule; one elected lane issues
      // ------------------------------------------------------------ pair UMMA issuer
      const uint32_t idesc = idesc_bf16_f32(256, L.NH);
      const uint32_t half_w = static_cast<uint32_t>(L.NH / 2);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0;; ++i) {
        const int n = pair_unit(args, i, rank, &cb, row0, present);
        if (n == 0) break;
        const int buf = i % L.nbuf;
        const uint32_t use = static_cast<uint32_t>(i / L.nbuf);
        mbar_wait_cluster(&acc_empty[buf], (use & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d0 = tmem_base + static_cast<uint32_t>(buf * L.group_cols);
        for (int kc = 0; kc < L.kchunks; ++kc) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sx = smem_u32(smem + static_cast<size_t>(stage) * L.stage_bytes);
          const uint32_t sw = sx + static_cast<uint32_t>(L.T) * 16384u;
          const uint64_t xd = sdesc_k128(sx), wd = sdesc_k128(sw);
          for (int k = 0; k < n; ++k)
            for (int h = 0; h < L.nh; ++h)
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint64_t a = xd + static_cast<uint64_t>(k * 1024 + j * 2);
                const uint64_t b = wd + static_cast<uint64_t>(h * half_w * 8u + j * 2);
                if (elect_one())
                  umma_bf16_pair(d0 + static_cast<uint32_t>(k * N + h * L.NH), a, b, idesc,
                                 (kc | j) != 0);
              }
          if (elect_one()) umma_commit_pair(&empty[stage], kBoth);
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (elect_one()) umma_commit_pair(&acc_full[buf], kBoth);
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue (both SMs)
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;  // columns [half*N/2, (half+1)*N/2) of the block
    const uint32_t lane_field = static_cast<uint32_t>(q * 32) << 16;
    const int row = q * 32 + lane;
    const bool issuer = (warp & 3) == 2 && lane == 0;  // one thread per half issues stores
    for (int i = threadIdx.x - 64; i < L.N_total; i += 256) sBias[i] = args.bias[i];
    asm volatile("bar.sync 1, 256;" ::: "memory");
    uint8_t* myout = sOut + half * 16384;
    const uint32_t acc_empty_leader = mapa_shared(smem_u32(&acc_empty[0]), 0);
    for (int i = 0;; ++i) {
      const int n = pair_unit(args, i, rank, &cb, row0, present);
      if (n == 0) break;
      const int buf = i % L.nbuf;
      const uint32_t use = static_cast<uint32_t>(i / L.nbuf);
      mbar_wait(&acc_full[buf], use & 1u);
      tc_fence_after();
      for (int k = 0; k < n; ++k) {
        for (int c = half * (N / 128); c < (half + 1) * (N / 128); ++c) {
          const uint32_t col = static_cast<uint32_t>(buf * L.group_cols + k * N + c * 64);
          uint32_t ra[32], rb[32];
          tmem_ld32_raw(tmem_base + lane_field + col, ra);
          tmem_ld32_raw(tmem_base + lane_field + col + 32, rb);
          tmem_ld_wait();
          if (!present[k]) continue;  // uniform over the CTA
          if (issuer) tma_store_wait_read<0>();
          half_barrier(half);
          uint8_t* stg = myout + row * 128;
          const float* bias = sBias + cb * N + c * 64;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            uint32_t p[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int e = u * 8 + v * 2;
              const uint32_t lo_bits = e < 32 ? ra[e] : rb[e - 32];
              const uint32_t hi_bits = e + 1 < 32 ? ra[e + 1] : rb[e + 1 - 32];
              float lo = __uint_as_float(lo_bits) + bias[e];
              float hi = __uint_as_float(hi_bits) + bias[e + 1];
              if (L.relu) {
                lo = fmaxf(lo, 0.0f);
                hi = fmaxf(hi, 0.0f);
              }
              __nv_bfloat162 pk = __floats2bfloat162_rn(lo, hi);
              p[v] = *reinterpret_cast<uint32_t*>(&pk);
            }
            *reinterpret_cast<uint4*>(stg + ((u ^ (row & 7)) << 4)) = make_uint4(p[0], p[1], p[2], p[3]);
          }
          fence_proxy_async_smem();
          half_barrier(half);
          if (issuer) {
            tma_store_2d(&tm_y, myout, cb * N + c * 64, static_cast<int32_t>(row0[k]));
            tma_store_commit();
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc_empty_leader + static_cast<uint32_t>(buf) * 8u);
    }
    if (issuer) tma_store_wait_all<0>();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer is done with every pair UMMA before TMEM goes away
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, static_cast<uint32_t>(L.tmem_cols));
  }
}

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

}  // namespace

bool dense_pair_plan(int K, int N_total, bool relu, DenseLayout* out) {
  if (K < 1 || K % 8 != 0 || N_total < 128 || N_total % 128 != 0) return false;
  const int kchunks = (K + 63) / 64;
  // Column block N: every divisor of N_total in {512, 384, 256, 128} is costed
  // over the whole row (ncb blocks).  A 512-wide block fills TMEM (one buffer,
  // epilogue not overlapped); 256-wide blocks double-buffer but re-stream X
  // per block.  Measured on 784 -> 512 (tools/time_members.py, MLP-512-512,
  // 4M samples): N = 256, nbuf = 2 5.89 ms vs N = 512, nbuf = 1 6.09 ms, which
  // this model reproduces with an effective TMA ingress of 64 B/clk per SM
  // (tools/tma_mcast.cu: ~80 with enough boxes in flight).
  // Design probes: ES_DPAIR_N / ES_DPAIR_T / ES_DPAIR_NBUF force the plan.
  const char* fn = std::getenv("ES_DPAIR_N");
  const char* ft = std::getenv("ES_DPAIR_T");
  const char* fb = std::getenv("ES_DPAIR_NBUF");
  constexpr double kIngressBpc = 64.0;
  bool found = false;
  DenseLayout best;
  double best_cost = 0.0;
  for (const int N : {512, 384, 256, 128}) {
    if (N > N_total || N_total % N != 0) continue;
    if (fn && N != std::atoi(fn)) continue;
    const int nh = (N + 255) / 256;
    const int NH = N / nh;
    if (NH % 32 != 0) continue;  // N % 16 per UMMA, NH/2 W rows per SM 8-row aligned
    for (int T = 1; T <= kMaxT; ++T)
      for (int nbuf = 1; nbuf <= 2; ++nbuf) {
        if ((ft && T != std::atoi(ft)) || (fb && nbuf != std::atoi(fb))) continue;
        const int cols = nbuf * T * N;
        if (cols > 512) continue;
        DenseLayout L;
        L.K = K;
        L.N = N;
        L.N_total = N_total;
        L.ncb = N_total / N;
        L.kchunks = kchunks;
        L.T = T;
        L.nbuf = nbuf;
        L.nh = nh;
        L.NH = NH;
        L.relu = relu ? 1 : 0;
        L.pair = 1;
        L.group_cols = T * N;
        int tc = 32;
        while (tc < cols) tc <<= 1;
        L.tmem_cols = tc;
        L.stage_bytes = static_cast<uint32_t>(T) * 16384u + static_cast<uint32_t>(N) * 64u;
        const uint32_t out_bytes = 2 * 16384u;
        const uint32_t tail = out_bytes + static_cast<uint32_t>(N_total) * 4u + 256u + 1024u + 64u;
        if (tail >= kSmemBudget) continue;
        const int stages = static_cast<int>(std::min<uint32_t>(8, (kSmemBudget - tail) / L.stage_bytes));
        if (stages < 2) continue;
        L.stages = stages;
        L.off_stage_out = static_cast<uint32_t>(stages) * L.stage_bytes;
        L.off_bias = L.off_stage_out + out_bytes;
        L.off_bar = align_up(L.off_bias + static_cast<uint32_t>(N_total) * 4u, 64);
        L.smem_bytes = std::max(L.off_bar + 256u + 1024u, kMinSmem);
        if (L.smem_bytes > kSmemBudget) continue;
        // Per SM per 128-row tile over the whole row: its half of the M=256
        // UMMAs vs TMA ingress, plus the un-overlapped epilogue of one buffer.
        const double mma = static_cast<double>(kchunks) * T * 2.0 * N;
        const double ingress = static_cast<double>(kchunks) * L.stage_bytes / kIngressBpc;
        const double epi = T * (N / 64.0) * 120.0 + 400.0;
        const double cost = L.ncb * (std::max(mma, ingress) + (nbuf == 1 ? epi : 0.0)) / T;
        if (!found || cost < best_cost) {
          best = L;
          best_cost = cost;
          found = true;
        }
      }
  }
  if (found) *out = best;
  if (found && std::getenv("ES_PAIR_VERBOSE"))
    std::fprintf(stderr, "dense_pair_plan K=%d N_total=%d: N %d T %d nbuf %d ncb %d stages %d\n", K, N_total,
                 best.N, best.T, best.nbuf, best.ncb, best.stages);
  return found;
}

int dense_pair_launch(const DenseArgs& args, const void* x, long long x_rows, const void* w, void* y,
                      int grid, cudaStream_t stream) {
  const DenseLayout& L = args.L;
  CUtensorMap mx, mw, my;
  if (make_bf16_map(&mx, x, static_cast<uint64_t>(L.K), static_cast<uint64_t>(x_rows), 128) != 0)
    return -1;
  if (make_bf16_map(&mw, w, static_cast<uint64_t>(L.K), static_cast<uint64_t>(L.N_total),
                    static_cast<uint32_t>(L.NH / 2)) != 0)
    return -1;
  if (make_bf16_map(&my, y, static_cast<uint64_t>(L.N_total), static_cast<uint64_t>(args.row_end),
                    128) != 0)
    return -1;
  const long long tiles = (args.row_end - args.row_begin + 127) / 128;
  if (tiles <= 0) return 0;
  const long long units = ((tiles + 1) / 2 + L.T - 1) / L.T * L.ncb;
  grid = static_cast<int>(std::min<long long>(grid / 2, units)) * 2;
  if (grid < 2) grid = 2;
  if (ensure_smem_attr(dense_pair_sm100, static_cast<int>(kSmemBudget)) != 0) return -4;
  dense_pair_sm100<<<grid, kThreads, L.smem_bytes, stream>>>(mx, mw, my, args);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace es
