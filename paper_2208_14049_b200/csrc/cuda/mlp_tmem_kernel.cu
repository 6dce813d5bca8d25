// K1 v2 — fused two-layer MLP member, hidden layer resident in TMEM
// (design in mlp_tmem_kernel.cuh).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstdlib>

#include "mlp_tmem_kernel.cuh"
#include "batching.cuh"
#include "epilogue.cuh"
#include "tma_host.hpp"

namespace es {

using namespace sm100;

namespace {

constexpr int kThreads = 320;             // w0 TMA, w1 MMA, w2..w9 epilogue
constexpr int kEpiThreads = 256;
constexpr uint32_t kSmemBudget = 232448;  // 227 KB
constexpr uint32_t kMinSmem = 120 * 1024; // one CTA per SM: TMEM is allocated whole
constexpr int kMaxT = 4;

using Tiles = BatchTiles;

__device__ __forceinline__ Tiles tile_space(const MlpTArgs& a) {
  if (a.claim) return batch_tiles(a.claim->seg_begin, a.claim->seg_end, a.seg_size, a.nb, a.b);
  return batch_tiles(a.seg_begin, a.seg_end, a.seg_size, a.nb, a.b);
}

// Tiles of group g for this CTA: returns how many (<= T) exist.
__device__ __forceinline__ int group_tiles(const MlpTArgs& a, const Tiles& ts, int g,
                                           long long (&row0)[kMaxT], int (&rows)[kMaxT]) {
  int n = 0;
  for (int k = 0; k < a.L.T; ++k) {
    const long long t = blockIdx.x + static_cast<long long>(g * a.L.T + k) * gridDim.x;
    if (t >= ts.total) break;
    row0[k] = batch_tile(ts, t, ts.seg_begin, a.seg_size, a.nb, a.b, &rows[k]);
    ++n;
  }
  return n;
}

__device__ __forceinline__ void epi_barrier() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

// HC: the hidden width as a compile-time constant (0 = runtime L.H), so
// layer 2's H/16 UMMAs issue from a fully unrolled loop with constant
// offsets (mlp_pair_kernel.cu: the issuing thread, not the pipe, paced them).
template <int HC>
__global__ void __launch_bounds__(kThreads, 1)
    member_mlp2_tmem_sm100(const __grid_constant__ CUtensorMap tm_x,
                           const __grid_constant__ CUtensorMap tm_w1,
                           const __grid_constant__ CUtensorMap tm_w2, const MlpTArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const MlpTLayout& L = args.L;
  uint8_t* sW2 = smem + L.off_w2;
  float* sBias = reinterpret_cast<float*>(smem + L.off_bias);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* full = bars;                  // [stages]
  uint64_t* empty = full + L.stages;      // [stages]
  uint64_t* acc_full = empty + L.stages;  // [2] group layer-1 accumulators ready
  uint64_t* acc_empty = acc_full + 2;     // [2] group TMEM buffer free
  uint64_t* a_full = acc_empty + 2;       // [kMaxT] bf16 hidden of tile k in TMEM
  uint64_t* acc2_full = a_full + kMaxT;   // [kMaxT] layer-2 accumulators ready
  uint64_t* w2_full = acc2_full + kMaxT;
  uint64_t* d2_empty = w2_full + 1;       // [kMaxT] separate D2 drained (d2_sep)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d2_empty + kMaxT);

  const int warp = warp_uniform_id();
  const int lane = threadIdx.x & 31;
  const int H = HC ? HC : L.H;
  const Tiles ts = tile_space(args);

  if (threadIdx.x == 0) {
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], L.d2_sep ? 8 : 4);
    }
    for (int k = 0; k < kMaxT; ++k) {
      mbar_init(&a_full[k], 8);
      mbar_init(&acc2_full[k], 1);
      mbar_init(&d2_empty[k], 4);
    }
    mbar_init(w2_full, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_x);
    tma_prefetch(&tm_w1);
    tma_prefetch(&tm_w2);
  }
  if (warp == 1) tmem_alloc(tmem_slot, static_cast<uint32_t>(L.tmem_cols));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      const uint64_t pol_stream = l2_policy_evict_normal();  // evict_first on X cost the weights their L2 residency
      const uint64_t pol_keep = l2_policy_evict_last();
      mbar_arrive_expect_tx(w2_full, static_cast<uint32_t>(H / 64) * 2048u);
      for (int kc = 0; kc < H / 64; ++kc)
        tma_load_2d(sW2 + kc * 2048, &tm_w2, w2_full, kc * 64, 0, pol_keep);
      int stage = 0;
      uint32_t phase = 0;
      long long row0[kMaxT];
      int rows[kMaxT];
      for (int g = 0;; ++g) {
        const int n = group_tiles(args, ts, g, row0, rows);
        if (n == 0) break;
        for (int kc = 0; kc < L.kchunks; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* st = smem + static_cast<size_t>(stage) * L.stage_bytes;
          mbar_arrive_expect_tx(&full[stage], static_cast<uint32_t>(n) * 16384u +
                                                  static_cast<uint32_t>(H) * 128u);
          for (int k = 0; k < n; ++k)
            tma_load_2d(st + k * 16384, &tm_x, &full[stage], kc * 64,
                        static_cast<int32_t>(row0[k]), pol_stream);
          uint8_t* sw = st + L.T * 16384;
          for (int mc = 0; mc < H / 128; ++mc)
            tma_load_2d(sw + mc * 16384, &tm_w1, &full[stage], kc * 64, mc * 128, pol_keep);
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // the whole warp walks the schedule; one elected lane issues
      // ------------------------------------------------------------ UMMA issuer
      const uint32_t idesc1 = idesc_bf16_f32(128, L.NH);
      const uint32_t idesc2 = idesc_bf16_f32(128, 16);
      const uint32_t sW2_addr = smem_u32(sW2);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t a_par = 0;    // bit k: parity of the next a_full[k] completion
      uint32_t d2_par = ~0u; // bit k: parity to wait on d2_empty[k] (first use free)
      bool w2_ready = false;
      // Layer-2 work still owed for the previous group.
      int pend_buf = -1, pend_n = 0, pend_next = 0;
      auto layer2 = [&](int buf, int k, bool waited) {
        if (!w2_ready) {
          mbar_wait(w2_full, 0);
          w2_ready = true;
        }
        if (!waited) mbar_wait(&a_full[k], (a_par >> k) & 1u);
        a_par ^= 1u << k;
        tc_fence_after();
        const uint32_t tile = tmem_base + static_cast<uint32_t>(buf * L.group_cols + k * H);
        uint32_t d2 = tile + static_cast<uint32_t>(H / 4);
        if (L.d2_sep) {
          mbar_wait(&d2_empty[k], (d2_par >> k) & 1u);
          d2_par ^= 1u << k;
          d2 = tmem_base + static_cast<uint32_t>(L.d2_col + 16 * L.d2_parts * k);
        }
        // Descriptors advance by (bytes >> 4) in their low field: precomputed
        // bases keep the single issuing thread at a few ALU ops per UMMA.
        const uint64_t w2d = sdesc_k128(sW2_addr);
        const uint32_t pmask = static_cast<uint32_t>(L.d2_parts - 1);  // parts: 1 or 4
        if constexpr (HC != 0) {
#pragma unroll
          for (int step = 0; step < HC / 16; ++step) {  // 16 hidden units per step
            const int hh = step / (HC / 32), kk = step % (HC / 32);
            const uint32_t h0 = static_cast<uint32_t>(hh * (HC / 2) + kk * 16);
            const uint32_t a = tile + static_cast<uint32_t>(hh * (HC / 2) + kk * 8);
            const uint64_t b = w2d + (h0 >> 6) * 128u + (h0 & 63u) / 8u;
            if (elect_one())
              umma_bf16_ta(d2 + 16u * (static_cast<uint32_t>(step) & pmask), a, b, idesc2,
                           static_cast<uint32_t>(step) > pmask);
          }
        } else {
          uint32_t step = 0;
          for (int hh = 0; hh < 2; ++hh)
            for (int kk = 0; kk < H / 32; ++kk, ++step) {  // 16 hidden units per step
              const uint32_t h0 = static_cast<uint32_t>(hh * (H / 2) + kk * 16);
              const uint32_t a = tile + static_cast<uint32_t>(hh * (H / 2) + kk * 8);
              const uint64_t b = w2d + (h0 >> 6) * 128u + (h0 & 63u) / 8u;
              if (elect_one()) umma_bf16_ta(d2 + 16u * (step & pmask), a, b, idesc2, step > pmask);
            }
        }
        if (elect_one()) umma_commit(&acc2_full[k]);
      };
      auto drain_pending = [&]() {
        for (; pend_next < pend_n; ++pend_next) layer2(pend_buf, pend_next, false);
        pend_buf = -1;
      };
      long long row0[kMaxT];
      int rows[kMaxT];
      for (int g = 0;; ++g) {
        const int n = group_tiles(args, ts, g, row0, rows);
        if (n == 0) break;
        const int buf = g % L.nbuf;
        const uint32_t use = static_cast<uint32_t>(g / L.nbuf);
        if (pend_buf == buf) drain_pending();  // single buffer: finish the last group
        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u);
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
                const uint64_t b = wd + static_cast<uint64_t>(h * L.NH * 8 + j * 2);
                if (elect_one()) umma_bf16(d0 + static_cast<uint32_t>(k * H + h * L.NH), a, b, idesc1,
                          (kc | j) != 0);
              }
          if (elect_one()) umma_commit(&empty[stage]);
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1u;
          }
          // Overlap: issue the previous group's layer 2 as its hidden tiles land.
          while (pend_buf >= 0 && pend_next < pend_n &&
                 __shfl_sync(0xffffffffu, mbar_test(&a_full[pend_next], (a_par >> pend_next) & 1u), 0)) {
            layer2(pend_buf, pend_next, true);
            ++pend_next;
          }
          if (pend_buf >= 0 && pend_next == pend_n) pend_buf = -1;
        }
        if (elect_one()) umma_commit(&acc_full[buf]);
        if (pend_buf >= 0) drain_pending();
        pend_buf = buf;
        pend_n = n;
        pend_next = 0;
      }
      if (pend_buf >= 0) drain_pending();
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const int ew = warp - 2;           // 0..7
    const int q = warp & 3;            // TMEM lane quadrant
    const int half = ew >> 2;          // hidden columns [half*H/2, (half+1)*H/2)
    const uint32_t lane_field = static_cast<uint32_t>(q * 32) << 16;
    for (int i = threadIdx.x - 64; i < H; i += kEpiThreads) sBias[i] = args.bias1[i];
    epi_barrier();
    float b2[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) b2[c] = c < L.C ? __ldg(args.bias2 + c) : 0.0f;
    uint32_t acc2_par = 0;
    long long row0[kMaxT];
    int rows[kMaxT];
    const int hw = H / 2;
    for (int g = 0;; ++g) {
      const int n = group_tiles(args, ts, g, row0, rows);
      if (n == 0) break;
      const int buf = g % L.nbuf;
      const uint32_t use = static_cast<uint32_t>(g / L.nbuf);
      mbar_wait(&acc_full[buf], use & 1u);
      tc_fence_after();
      for (int k = 0; k < n; ++k) {
        const uint32_t col0 =
            static_cast<uint32_t>(buf * L.group_cols + k * H + half * hw);
        const float* bias = sBias + half * hw;
        hidden_to_bf16(tmem_base + lane_field + col0, bias, hw);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[k]);
      }
      // Separate D2: the hidden columns are free for the next group as soon as
      // every warp has converted them (the UMMA thread orders layer 2 first).
      if (L.d2_sep && lane == 0) mbar_arrive(&acc_empty[buf]);
      if (half == 0) {
        // Pull every tile's D2 into registers first, release the TMEM, then
        // finish the logits off the UMMA thread's critical path.
        float z[kMaxT][16];
#pragma unroll
        for (int k = 0; k < kMaxT; ++k) {
          if (k >= n) continue;
          mbar_wait(&acc2_full[k], (acc2_par >> k) & 1u);
          acc2_par ^= 1u << k;
          tc_fence_after();
          const uint32_t d2col =
              L.d2_sep ? static_cast<uint32_t>(L.d2_col + 16 * L.d2_parts * k)
                       : static_cast<uint32_t>(buf * L.group_cols + k * H + H / 4);
          read_d2(tmem_base + lane_field + d2col, L.d2_parts, z[k]);
          if (L.d2_sep) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&d2_empty[k]);
          }
        }
        if (!L.d2_sep) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[buf]);
        }
        const int r = q * 32 + lane;
#pragma unroll
        for (int k = 0; k < kMaxT; ++k) {
          if (k >= n || r >= rows[k]) continue;
          float* o = args.out + (row0[k] + r) * L.C;
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c < L.C) o[c] = z[k][c] + b2[c];
        }
      }
    }
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

bool mlpt_plan(int K, int H, int C, int b, MlpTLayout* out) {
  if (K < 1 || K % 8 != 0 || H < 128 || H % 128 != 0 || H > 512 || C < 1 || C > 16 || b < 1 ||
      b > 128)
    return false;
  const int kchunks = (K + 63) / 64;
  const int nh = (H + 255) / 256;
  const int NH = H / nh;
  if (NH % 16 != 0) return false;
  bool found = false;
  MlpTLayout best;
  const char* ft = std::getenv("ES_TMEM_T");  // design probes: force T, nbuf
  const char* fb = std::getenv("ES_TMEM_NBUF");
  for (int T = 1; T <= kMaxT; ++T) {
    if (ft && T != std::atoi(ft)) continue;
    for (int nbuf = 1; nbuf <= 2; ++nbuf) {
      if (fb && nbuf != std::atoi(fb)) continue;
      const int cols = nbuf * T * H;
      if (cols > 512) continue;
      MlpTLayout L;
      L.H = H;
      L.C = C;
      L.K = K;
      L.kchunks = kchunks;
      L.T = T;
      L.nbuf = nbuf;
      L.nh = nh;
      L.NH = NH;
      L.group_cols = T * H;
      // Layer-2 partial accumulators: 4 when there is room (inside the
      // drained half-0 columns [H/4, H/2), or after the hidden columns).
      L.d2_sep = cols + 16 * T <= 512 ? 1 : 0;
      L.d2_parts = L.d2_sep ? (cols + 64 * T <= 512 ? 4 : 1) : (H >= 256 ? 4 : 1);
      L.d2_col = cols;
      int tc = 32;
      while (tc < cols + (L.d2_sep ? 16 * L.d2_parts * T : 0)) tc <<= 1;
      L.tmem_cols = tc;
      L.stage_bytes = static_cast<uint32_t>(T) * 16384u + static_cast<uint32_t>(H) * 128u;
      const uint32_t tail = static_cast<uint32_t>(H / 64) * 2048u + static_cast<uint32_t>(H) * 4u +
                            512u + 1024u;
      const int stages = static_cast<int>(std::min<uint32_t>(8, (kSmemBudget - tail) / L.stage_bytes));
      if (stages < 2) continue;
      L.stages = stages;
      L.off_w2 = static_cast<uint32_t>(stages) * L.stage_bytes;
      L.off_bias = L.off_w2 + static_cast<uint32_t>(H / 64) * 2048u;
      L.off_bar = align_up(L.off_bias + static_cast<uint32_t>(H) * 4u, 64);
      L.smem_bytes = std::max(L.off_bar + 512u + 1024u, kMinSmem);
      if (L.smem_bytes > kSmemBudget) continue;
      // Cycle model per group (profiles/r1_summary.md): tensor time vs TMA
      // ingress (~44 B/clk/SM sustained) vs an un-overlapped epilogue when the
      // TMEM buffer is single.
      // X also has to come from HBM: ~25 B/clk/SM (7.2 TB/s over 148 SMs).
      const double mma = static_cast<double>(kchunks) * T * 2.0 * H;
      const double ingress = static_cast<double>(kchunks) * L.stage_bytes / 44.0;
      const double hbm = static_cast<double>(T) * b * K * 2.0 / 25.0;
      const double epi = T * (H / 64.0) * 110.0 + 400.0;
      const double per_group =
          std::max({mma, ingress, hbm}) + (nbuf == 1 ? (L.d2_sep ? 0.6 * epi : epi) : 0.0);
      L.est_cycles_per_sample = static_cast<float>(per_group / (static_cast<double>(T) * b));
      if (!found || L.est_cycles_per_sample < best.est_cycles_per_sample) {
        best = L;
        found = true;
      }
    }
  }
  if (found) *out = best;
  if (found && std::getenv("ES_PAIR_VERBOSE"))
    std::fprintf(stderr, "mlpt_plan K=%d H=%d: T %d nbuf %d stages %d d2_sep %d\n", K, H, best.T, best.nbuf,
                 best.stages, best.d2_sep);
  return found;
}

int mlpt_launch(const MlpTArgs& args, const void* x, const void* w1, const void* w2, int grid,
                cudaStream_t stream) {
  const MlpTLayout& L = args.L;
  CUtensorMap mx, mw1, mw2;
  if (make_bf16_map(&mx, x, static_cast<uint64_t>(L.K), static_cast<uint64_t>(args.nb), 128) != 0)
    return -1;
  if (make_bf16_map(&mw1, w1, static_cast<uint64_t>(L.K), static_cast<uint64_t>(L.H), 128) != 0)
    return -1;
  if (make_bf16_map(&mw2, w2, static_cast<uint64_t>(L.H), static_cast<uint64_t>(L.C), 16) != 0)
    return -1;
  auto kernel = L.H == 128   ? member_mlp2_tmem_sm100<128>
                : L.H == 256 ? member_mlp2_tmem_sm100<256>
                : L.H == 384 ? member_mlp2_tmem_sm100<384>
                : L.H == 512 ? member_mlp2_tmem_sm100<512>
                             : member_mlp2_tmem_sm100<0>;
  if (std::getenv("ES_TMEM_RUNTIME_H")) kernel = member_mlp2_tmem_sm100<0>;  // A/B probe
  if (ensure_smem_attr(kernel, static_cast<int>(kSmemBudget)) != 0) return -4;
  const long long per_seg = (args.seg_size + args.b - 1) / args.b;
  const long long tiles = (args.seg_end - args.seg_begin) * per_seg;
  if (tiles <= 0) return 0;
  grid = static_cast<int>(std::min<long long>(grid, (tiles + L.T - 1) / L.T));
  kernel<<<grid, kThreads, L.smem_bytes, stream>>>(mx, mw1, mw2, args);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace es
