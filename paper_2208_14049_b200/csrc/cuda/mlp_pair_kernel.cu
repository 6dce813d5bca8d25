// K1 v3 — fused two-layer MLP member on SM pairs (design in mlp_pair_kernel.cuh).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "mlp_pair_kernel.cuh"
#include "batching.cuh"
#include "epilogue.cuh"
#include "tma_host.hpp"

namespace es {

using namespace sm100;

namespace {

constexpr int kThreads = 320;             // w0 TMA, w1 TMEM + UMMA (leader), w2..w9 epilogue
constexpr int kEpiThreads = 256;
constexpr uint32_t kSmemBudget = 232448;
constexpr uint32_t kMinSmem = 120 * 1024;
constexpr int kMaxT = 2;
constexpr uint16_t kBoth = 0b11;

using Tiles = BatchTiles;

__device__ __forceinline__ Tiles tile_space(const MlpPArgs& a) {
  if (a.claim) return batch_tiles(a.claim->seg_begin, a.claim->seg_end, a.seg_size, a.nb, a.b);
  return batch_tiles(a.seg_begin, a.seg_end, a.seg_size, a.nb, a.b);
}

// Group g of this pair: pair-tile tp = pair + (g*T + k) * pairs covers tiles
// 2*tp (even CTA) and 2*tp + 1 (odd CTA).  Returns how many pair-tiles exist
// (both CTAs agree); rows = 0 marks this CTA's tile as absent.
__device__ __forceinline__ int group_tiles(const MlpPArgs& a, const Tiles& ts, int g,
                                           uint32_t rank, long long (&row0)[kMaxT],
                                           int (&rows)[kMaxT]) {
  const long long pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;
  int n = 0;
  for (int k = 0; k < a.L.T; ++k) {
    const long long tp = pair + static_cast<long long>(g * a.L.T + k) * pairs;
    if (2 * tp >= ts.total) break;
    const long long t = 2 * tp + rank;
    if (t < ts.total) {
      row0[k] = batch_tile(ts, t, ts.seg_begin, a.seg_size, a.nb, a.b, &rows[k]);
    } else {
      row0[k] = 0;  // load something valid; nothing is written back
      rows[k] = 0;
    }
    ++n;
  }
  return n;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#define TRACE(g, i)                                                       \
  do {                                                                    \
    if (args.trace && blockIdx.x == 0 && (g) < 32) args.trace[(g) * 16 + (i)] = global_ns(); \
  } while (0)

__device__ __forceinline__ void epi_barrier() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

// HPC: the hidden units per pass as a compile-time constant (0 = runtime
// L.HP).  Layer 2's 2 * HP/32 UMMAs then issue from a fully unrolled loop
// with constant TMEM / descriptor offsets: with runtime offsets the issuing
// thread, not the tensor pipe, paced them (tools/umma_contention.cu
// layer2_rate: ~230 vs ~100 clk per N = 16 UMMA).
template <int HPC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    member_mlp2_pair_sm100(const __grid_constant__ CUtensorMap tm_x,
                           const __grid_constant__ CUtensorMap tm_w1,
                           const __grid_constant__ CUtensorMap tm_w2, const MlpPArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const MlpPLayout& L = args.L;
  uint8_t* sW2 = smem + L.off_w2;
  float* sBias = reinterpret_cast<float*>(smem + L.off_bias);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* full = bars;                  // [stages]   (leader's is used)
  uint64_t* empty = full + L.stages;      // [stages]   (each SM's own)
  uint64_t* acc_full = empty + L.stages;  // [2]        (multicast commit)
  uint64_t* acc_empty = acc_full + 2;     // [2]        (leader's; 8 remote arrivals)
  uint64_t* a_full = acc_empty + 2;       // [kMaxT]    (leader's; 16 remote arrivals)
  uint64_t* acc2_full = a_full + kMaxT;   // [kMaxT]    (multicast commit)
  uint64_t* w2_full = acc2_full + kMaxT;  //            (leader's)
  uint64_t* d2_empty = w2_full + 1;       // [kMaxT]    (leader's; 8 remote arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d2_empty + kMaxT);

  const int warp = warp_uniform_id();
  const int lane = threadIdx.x & 31;
  const int H = L.H;    // all hidden units (W2 columns, biases)
  const int HP = HPC ? HPC : L.HP;  // hidden units per pass (TMEM-resident at a time)
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const Tiles ts = tile_space(args);

  if (threadIdx.x == 0) {
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], L.d2_sep ? 16 : 8);
    }
    for (int k = 0; k < kMaxT; ++k) {
      mbar_init(&a_full[k], 16);
      mbar_init(&acc2_full[k], 1);
      mbar_init(&d2_empty[k], 8);
    }
    mbar_init(w2_full, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_x);
    tma_prefetch(&tm_w1);
    tma_prefetch(&tm_w2);
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, static_cast<uint32_t>(L.tmem_cols));
  tc_fence_before();
  cluster_sync();  // barrier inits and TMEM of both SMs visible to both
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA (both SMs)
      const uint64_t pol_stream = l2_policy_evict_normal();  // evict_first on X cost the weights their L2 residency
      const uint64_t pol_keep = l2_policy_evict_last();
      // Hidden passes re-read the same X tiles right away: every pass but the
      // last keeps them in L2 (evict_last), the last lets them go.
      const uint64_t pol_reread = l2_policy_evict_last();
      if (leader) mbar_arrive_expect_tx(w2_full, 2u * static_cast<uint32_t>(H / 64) * 1024u);
      for (int kc = 0; kc < H / 64; ++kc)
        tma_load_2d_pair(sW2 + kc * 1024, &tm_w2, w2_full, kc * 64, static_cast<int32_t>(rank) * 8,
                         pol_keep);
      int stage = 0;
      uint32_t phase = 0;
      long long row0[kMaxT];
      int rows[kMaxT];
      const uint32_t half_w = static_cast<uint32_t>(L.NH / 2);
      for (int g = 0;; ++g) {
        const int n = group_tiles(args, ts, g, rank, row0, rows);
        if (n == 0) break;
        for (int hp = 0; hp < L.passes; ++hp)  // hidden passes re-stream the X tiles
          for (int kc = 0; kc < L.kchunks; ++kc) {
            mbar_wait(&empty[stage], phase ^ 1u);
            if (kc == 0) TRACE(g * L.passes + hp, 7);
            uint8_t* st = smem + static_cast<size_t>(stage) * L.stage_bytes;
            if (leader)
              mbar_arrive_expect_tx(&full[stage], 2u * (static_cast<uint32_t>(n) * 16384u +
                                                        static_cast<uint32_t>(HP) * 64u));
            for (int k = 0; k < n; ++k)
              tma_load_2d_pair(st + k * 16384, &tm_x, &full[stage], kc * 64,
                               static_cast<int32_t>(row0[k]),
                               hp + 1 < L.passes ? pol_reread : pol_stream);
            uint8_t* sw = st + L.T * 16384;
            for (int h = 0; h < L.nh; ++h)
              tma_load_2d_pair(sw + h * half_w * 128u, &tm_w1, &full[stage], kc * 64,
                               static_cast<int32_t>(hp * HP + h * L.NH + rank * half_w), pol_keep);
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
      const uint32_t idesc1 = idesc_bf16_f32(256, L.NH);
      const uint32_t idesc2 = idesc_bf16_f32(256, 16);
      const uint32_t sW2_addr = smem_u32(sW2);
      const uint32_t half_w = static_cast<uint32_t>(L.NH / 2);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t a_par = 0;
      uint32_t d2_par = ~0u;
      bool w2_ready = false;
      int pend_buf = -1, pend_n = 0, pend_next = 0, pend_g = 0, pend_hp = 0;
      auto layer2 = [&](int buf, int k, bool waited) {
        if (!w2_ready) {
          mbar_wait(w2_full, 0);
          w2_ready = true;
        }
        if (!waited) mbar_wait_cluster(&a_full[k], (a_par >> k) & 1u);
        if (k == 0) TRACE(pend_g * L.passes + pend_hp, 8);
        a_par ^= 1u << k;
        tc_fence_after();
        const uint32_t tile = tmem_base + static_cast<uint32_t>(buf * L.group_cols + k * HP);
        uint32_t d2 = tile + static_cast<uint32_t>(HP / 4);
        if (L.d2_sep) {
          mbar_wait_cluster(&d2_empty[k], (d2_par >> k) & 1u);
          d2_par ^= 1u << k;
          d2 = tmem_base + static_cast<uint32_t>(L.d2_col + 16 * L.d2_parts * k);
        }
        // Descriptors advance by (bytes >> 4) in their low field: precomputed
        // bases keep the single issuing thread at a few ALU ops per UMMA.
        const uint64_t w2d = sdesc_k128(sW2_addr);
        const uint32_t pmask = static_cast<uint32_t>(L.d2_parts - 1);  // parts: 1 or 4
        if constexpr (HPC != 0) {
          // pend_hp * HPC is a multiple of 64 hidden units: one runtime add.
          const uint64_t w2p = w2d + static_cast<uint64_t>(pend_hp * HPC / 64) * 64u;
#pragma unroll
          for (int step = 0; step < HPC / 16; ++step) {  // 16 hidden units per step
            const int hh = step / (HPC / 32), kk = step % (HPC / 32);
            const uint32_t h0 = static_cast<uint32_t>(hh * (HPC / 2) + kk * 16);
            const uint32_t a = tile + static_cast<uint32_t>(hh * (HPC / 2) + kk * 8);
            const uint64_t b = w2p + (h0 >> 6) * 64u + (h0 & 63u) / 8u;
            if (elect_one())
              umma_bf16_pair_ta(d2 + 16u * (static_cast<uint32_t>(step) & pmask), a, b, idesc2,
                                static_cast<uint32_t>(step) > pmask);
          }
        } else {
          uint32_t step = 0;
          for (int hh = 0; hh < 2; ++hh)
            for (int kk = 0; kk < HP / 32; ++kk, ++step) {  // 16 hidden units per step
              const uint32_t h0 = static_cast<uint32_t>(pend_hp * HP + hh * (HP / 2) + kk * 16);
              const uint32_t a = tile + static_cast<uint32_t>(hh * (HP / 2) + kk * 8);
              const uint64_t b = w2d + (h0 >> 6) * 64u + (h0 & 63u) / 8u;
              if (elect_one()) umma_bf16_pair_ta(d2 + 16u * (step & pmask), a, b, idesc2, step > pmask);
            }
        }
        if (elect_one()) umma_commit_pair(&acc2_full[k], kBoth);
        if (k == 0) TRACE(pend_g * L.passes + pend_hp, 9);
      };
      auto drain_pending = [&]() {
        for (; pend_next < pend_n; ++pend_next) layer2(pend_buf, pend_next, false);
        pend_buf = -1;
      };
      long long row0[kMaxT];
      int rows[kMaxT];
      for (int v = 0;; ++v) {  // v = group * passes + hidden pass
        const int g = v / L.passes, hp = v % L.passes;
        const int n = group_tiles(args, ts, g, rank, row0, rows);
        if (n == 0) break;
        const int buf = v % L.nbuf;
        const uint32_t use = static_cast<uint32_t>(v / L.nbuf);
        if (pend_buf == buf) drain_pending();
        TRACE(v, 0);
        mbar_wait_cluster(&acc_empty[buf], (use & 1u) ^ 1u);
        TRACE(v, 1);
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
                if (elect_one()) umma_bf16_pair(d0 + static_cast<uint32_t>(k * HP + h * L.NH), a, b, idesc1,
                               (kc | j) != 0);
              }
          if (elect_one()) umma_commit_pair(&empty[stage], kBoth);
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1u;
          }
          while (pend_buf >= 0 && pend_next < pend_n &&
                 __shfl_sync(0xffffffffu, mbar_test_cluster(&a_full[pend_next], (a_par >> pend_next) & 1u), 0)) {
            layer2(pend_buf, pend_next, true);
            ++pend_next;
          }
          if (pend_buf >= 0 && pend_next == pend_n) pend_buf = -1;
        }
        if (elect_one()) umma_commit_pair(&acc_full[buf], kBoth);
        TRACE(v, 2);
        if (pend_buf >= 0) drain_pending();
        pend_buf = buf;
        pend_n = n;
        pend_next = 0;
        pend_g = g;
        pend_hp = hp;
      }
      if (pend_buf >= 0) drain_pending();
    }
  } else {
    // -------------------------------------------------------------- epilogue (both SMs)
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;
    const uint32_t lane_field = static_cast<uint32_t>(q * 32) << 16;
    for (int i = threadIdx.x - 64; i < H; i += kEpiThreads) sBias[i] = args.bias1[i];
    epi_barrier();
    float b2[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) b2[c] = c < L.C ? __ldg(args.bias2 + c) : 0.0f;
    uint32_t acc2_par = 0;
    long long row0[kMaxT];
    int rows[kMaxT];
    const int hw = HP / 2;
    float zs[kMaxT][16];  // logits summed over the hidden passes
    for (int v = 0;; ++v) {
      const int g = v / L.passes, hp = v % L.passes;
      const int n = group_tiles(args, ts, g, rank, row0, rows);
      if (n == 0) break;
      const int buf = v % L.nbuf;
      const uint32_t use = static_cast<uint32_t>(v / L.nbuf);
      mbar_wait(&acc_full[buf], use & 1u);
      if (warp == 2 && lane == 0) TRACE(v, 3);
      tc_fence_after();
      for (int k = 0; k < n; ++k) {
        const uint32_t col0 = static_cast<uint32_t>(buf * L.group_cols + k * HP + half * hw);
        const float* bias = sBias + hp * HP + half * hw;
        hidden_to_bf16(tmem_base + lane_field + col0, bias, hw);
        if (warp == 2 && lane == 0 && k == 0) TRACE(v, 4);
        if (warp == 9 && lane == 0 && k == 0) TRACE(v, 10);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&a_full[k]), 0));
      }
      if (L.d2_sep && lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&acc_empty[buf]), 0));
      if (half == 0) {
        // Pull every tile's D2 into registers first, release the TMEM, then
        // finish the logits off the UMMA thread's critical path.
        float z[kMaxT][16];
#pragma unroll
        for (int k = 0; k < kMaxT; ++k) {
          if (k >= n) continue;
          mbar_wait(&acc2_full[k], (acc2_par >> k) & 1u);
          if (warp == 2 && lane == 0 && k == 0) TRACE(v, 5);
          acc2_par ^= 1u << k;
          tc_fence_after();
          const uint32_t d2col =
              L.d2_sep ? static_cast<uint32_t>(L.d2_col + 16 * L.d2_parts * k)
                       : static_cast<uint32_t>(buf * L.group_cols + k * HP + HP / 4);
          read_d2(tmem_base + lane_field + d2col, L.d2_parts, z[k]);
#pragma unroll
          for (int c = 0; c < 16; ++c) zs[k][c] = hp == 0 ? z[k][c] : zs[k][c] + z[k][c];
          if (L.d2_sep) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&d2_empty[k]), 0));
          }
        }
        if (!L.d2_sep) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&acc_empty[buf]), 0));
        }
        const int r = q * 32 + lane;
#pragma unroll
        for (int k = 0; k < kMaxT; ++k) {
          if (hp + 1 < L.passes || k >= n || r >= rows[k]) continue;
          float* o = args.out + (row0[k] + r) * L.C;
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c < L.C) o[c] = zs[k][c] + b2[c];
        }
        if (warp == 2 && lane == 0) TRACE(v, 6);
      }
    }
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

bool mlpp_plan(int K, int H, int C, int b, MlpPLayout* out) {
  if (K < 1 || K % 8 != 0 || H < 128 || H % 128 != 0 || H > 2048 || C < 1 || C > 16 || b < 1 ||
      b > 128)
    return false;
  // Hidden layers wider than one SM's TMEM run in passes of HP <= 512 units:
  // each pass re-streams the X tiles, and the layer-2 partials of the passes
  // are summed in the epilogue's registers.
  int passes = (H + 511) / 512;
  // ES_PAIR_PASSES / ES_PAIR_T / ES_PAIR_NBUF / ES_PAIR_VERBOSE: design probes
  if (const char* fp = std::getenv("ES_PAIR_PASSES")) passes = std::max(passes, std::atoi(fp));
  if (H % passes != 0 || (H / passes) % 128 != 0) return false;
  const int HP = H / passes;
  const int kchunks = (K + 63) / 64;
  const int nh = (HP + 255) / 256;
  const int NH = HP / nh;
  if (NH % 32 != 0) return false;  // N % 16 per UMMA, NH/2 rows 8-row aligned per SM
  bool found = false;
  MlpPLayout best;
  const char* ft = std::getenv("ES_PAIR_T");
  const char* fb = std::getenv("ES_PAIR_NBUF");
  for (int T = 1; T <= kMaxT; ++T) {
    if (ft && T != std::atoi(ft)) continue;
    for (int nbuf = 1; nbuf <= 2; ++nbuf) {
      if (fb && nbuf != std::atoi(fb)) continue;
      const int cols = nbuf * T * HP;
      if (cols > 512) continue;
      MlpPLayout L;
      L.H = H;
      L.HP = HP;
      L.passes = passes;
      L.C = C;
      L.K = K;
      L.kchunks = kchunks;
      L.T = T;
      L.nbuf = nbuf;
      L.nh = nh;
      L.NH = NH;
      L.group_cols = T * HP;
      // Layer-2 partial accumulators: 4 when there is room (inside the
      // drained half-0 columns [H/4, H/2), or after the hidden columns).
      L.d2_sep = cols + 16 * T <= 512 ? 1 : 0;
      L.d2_parts = L.d2_sep ? (cols + 64 * T <= 512 ? 4 : 1) : (HP >= 256 ? 4 : 1);
      L.d2_col = cols;
      int tc = 32;
      while (tc < cols + (L.d2_sep ? 16 * L.d2_parts * T : 0)) tc <<= 1;
      L.tmem_cols = tc;
      L.stage_bytes = static_cast<uint32_t>(T) * 16384u + static_cast<uint32_t>(HP) * 64u;
      const uint32_t tail = static_cast<uint32_t>(H / 64) * 1024u + static_cast<uint32_t>(H) * 4u +
                            512u + 1024u;
      const int stages =
          static_cast<int>(std::min<uint32_t>(8, (kSmemBudget - tail) / L.stage_bytes));
      if (stages < 2) continue;
      L.stages = stages;
      L.off_w2 = static_cast<uint32_t>(stages) * L.stage_bytes;
      L.off_bias = L.off_w2 + static_cast<uint32_t>(H / 64) * 1024u;
      L.off_bar = align_up(L.off_bias + static_cast<uint32_t>(H) * 4u, 64);
      L.smem_bytes = std::max(L.off_bar + 512u + 1024u, kMinSmem);
      if (L.smem_bytes > kSmemBudget) continue;
      // Per-SM cycles per group: tensor (the pair shares one M=256 UMMA) vs TMA
      // ingress (~44 B/clk) vs HBM share (~25 B/clk) + un-overlapped epilogue.
      const double mma = static_cast<double>(kchunks) * T * 2.0 * HP;
      const double ingress = static_cast<double>(kchunks) * L.stage_bytes / 44.0;
      const double hbm = static_cast<double>(T) * b * K * 2.0 / 25.0 / passes;
      const double epi = T * (HP / 64.0) * 110.0 + 600.0;
      const double per_group = passes * (std::max({mma, ingress, hbm}) +
                                         (nbuf == 1 ? (L.d2_sep ? 0.6 * epi : epi) : 0.0));
      L.est_cycles_per_sample = static_cast<float>(per_group / (static_cast<double>(T) * b));
      if (!found || L.est_cycles_per_sample < best.est_cycles_per_sample) {
        best = L;
        found = true;
      }
    }
  }
  if (found) *out = best;
  if (found && std::getenv("ES_PAIR_VERBOSE"))
    std::fprintf(stderr, "mlpp_plan K=%d H=%d: passes %d HP %d T %d nbuf %d stages %d\n", K, H, best.passes,
                 best.HP, best.T, best.nbuf, best.stages);
  return found;
}

int mlpp_launch(const MlpPArgs& args, const void* x, const void* w1, const void* w2, int grid,
                cudaStream_t stream) {
  const MlpPLayout& L = args.L;
  CUtensorMap mx, mw1, mw2;
  if (make_bf16_map(&mx, x, static_cast<uint64_t>(L.K), static_cast<uint64_t>(args.nb), 128) != 0)
    return -1;
  if (make_bf16_map(&mw1, w1, static_cast<uint64_t>(L.K), static_cast<uint64_t>(L.H),
                    static_cast<uint32_t>(L.NH / 2)) != 0)  // rows of all passes
    return -1;
  if (make_bf16_map(&mw2, w2, static_cast<uint64_t>(L.H), static_cast<uint64_t>(L.C), 8) != 0)
    return -1;
  auto kernel = L.HP == 128   ? member_mlp2_pair_sm100<128>
                : L.HP == 256 ? member_mlp2_pair_sm100<256>
                : L.HP == 384 ? member_mlp2_pair_sm100<384>
                : L.HP == 512 ? member_mlp2_pair_sm100<512>
                              : member_mlp2_pair_sm100<0>;
  if (std::getenv("ES_PAIR_RUNTIME_HP")) kernel = member_mlp2_pair_sm100<0>;  // A/B probe
  if (ensure_smem_attr(kernel, static_cast<int>(kSmemBudget)) != 0) return -4;
  const long long per_seg = (args.seg_size + args.b - 1) / args.b;
  const long long tiles = (args.seg_end - args.seg_begin) * per_seg;
  if (tiles <= 0) return 0;
  const long long pair_groups = (tiles + 2LL * L.T - 1) / (2LL * L.T);
  grid = static_cast<int>(std::min<long long>(grid / 2, pair_groups)) * 2;
  if (grid < 2) grid = 2;
  kernel<<<grid, kThreads, L.smem_bytes, stream>>>(mx, mw1, mw2, args);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace es
