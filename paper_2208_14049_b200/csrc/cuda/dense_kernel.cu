// Dense layer Y = act(X W^T + b) on tcgen05 (design in dense_kernel.cuh).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "dense_kernel.cuh"
#include "tma_host.hpp"

namespace es {

using namespace sm100;

namespace {

constexpr int kThreads = 320;  // w0 TMA, w1 TMEM + UMMA, w2..w9 epilogue (2 per lane quadrant)
constexpr uint32_t kSmemBudget = 232448;
constexpr uint32_t kMinSmem = 120 * 1024;
constexpr int kMaxT = 4;

// The CTA's i-th work unit: T consecutive 128-row tiles x one column block.
// Consecutive units of a row group walk its column blocks, so the X tiles are
// re-read from L2 while hot.  Returns the number of tiles (0 = no more work).
__device__ __forceinline__ long long rows_begin(const DenseArgs& a) {
  return a.claim ? a.claim->row_begin : a.row_begin;
}
__device__ __forceinline__ long long rows_end(const DenseArgs& a) {
  return a.claim ? a.claim->row_end : a.row_end;
}

__device__ __forceinline__ int unit_rows(const DenseArgs& a, int i, int* cb, long long (&row0)[kMaxT]) {
  const long long rb = rows_begin(a);
  const long long tiles = (rows_end(a) - rb + 127) / 128;
  const long long groups = (tiles + a.L.T - 1) / a.L.T;
  const long long u = blockIdx.x + static_cast<long long>(i) * gridDim.x;
  if (u >= groups * a.L.ncb) return 0;
  *cb = static_cast<int>(u % a.L.ncb);
  const long long g = u / a.L.ncb;
  int n = 0;
  for (int k = 0; k < a.L.T; ++k) {
    const long long t = g * a.L.T + k;
    if (t >= tiles) break;
    row0[k] = rb + t * 128;
    ++n;
  }
  return n;
}

__device__ __forceinline__ void half_barrier(int half) {
  asm volatile("bar.sync %0, 128;" ::"r"(2 + half) : "memory");
}

// kLogits: the member's last layer -- N = 16 (>= C) columns, no activation,
// fp32 logits [rows][C] stored straight from the epilogue registers.
template <bool kLogits>
__global__ void __launch_bounds__(kThreads, 1)
    dense_sm100(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                const __grid_constant__ CUtensorMap tm_y, const DenseArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const DenseLayout& L = args.L;
  uint8_t* sOut = smem + L.off_stage_out;  // [2 halves][128 rows][128 B]
  float* sBias = reinterpret_cast<float*>(smem + L.off_bias);  // all N_total columns
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* full = bars;
  uint64_t* empty = full + L.stages;
  uint64_t* acc_full = empty + L.stages;  // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = warp_uniform_id();
  const int lane = threadIdx.x & 31;
  const int N = L.N;  // columns per block

  if (threadIdx.x == 0) {
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_x);
    tma_prefetch(&tm_w);
    if (!kLogits) tma_prefetch(&tm_y);
  }
  if (warp == 1) tmem_alloc(tmem_slot, static_cast<uint32_t>(L.tmem_cols));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_stream = l2_policy_evict_normal();  // evict_first on X cost the weights their L2 residency
      const uint64_t pol_keep = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      long long row0[kMaxT];
      int cb = 0;
      for (int i = 0;; ++i) {
        const int n = unit_rows(args, i, &cb, row0);
        if (n == 0) break;
        for (int kc = 0; kc < L.kchunks; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* st = smem + static_cast<size_t>(stage) * L.stage_bytes;
          mbar_arrive_expect_tx(&full[stage], static_cast<uint32_t>(n) * 16384u +
                                                  static_cast<uint32_t>(N) * 128u);
          for (int k = 0; k < n; ++k)
            tma_load_2d(st + k * 16384, &tm_x, &full[stage], kc * 64,
                        static_cast<int32_t>(row0[k]), pol_stream);
          uint8_t* sw = st + L.T * 16384;
          if (kLogits) {
            tma_load_2d(sw, &tm_w, &full[stage], kc * 64, 0, pol_keep);  // one 16-row box
          } else {
            for (int c = 0; c < N / 64; ++c)  // 64-row boxes of the column block of W
              tma_load_2d(sw + c * 8192, &tm_w, &full[stage], kc * 64, cb * N + c * 64, pol_keep);
          }
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // the whole warp walks the schedule; one elected lane issues
      const uint32_t idesc = idesc_bf16_f32(128, L.NH);
      int stage = 0;
      uint32_t phase = 0;
      long long row0[kMaxT];
      int cb = 0;
      for (int i = 0;; ++i) {
        const int n = unit_rows(args, i, &cb, row0);
        if (n == 0) break;
        const int buf = i % L.nbuf;
        const uint32_t use = static_cast<uint32_t>(i / L.nbuf);
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
              for (int j = 0; j < 4; ++j)
                if (elect_one())
                  umma_bf16(d0 + static_cast<uint32_t>(k * N + h * L.NH),
                            xd + static_cast<uint64_t>(k * 1024 + j * 2),
                            wd + static_cast<uint64_t>(h * L.NH * 8 + j * 2), idesc, (kc | j) != 0);
          if (elect_one()) umma_commit(&empty[stage]);
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (elect_one()) umma_commit(&acc_full[buf]);
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;  // bf16 mode: columns [half*N/2, (half+1)*N/2) of the block
    const uint32_t lane_field = static_cast<uint32_t>(q * 32) << 16;
    const int row = q * 32 + lane;  // row within the tile
    const bool issuer = (warp & 3) == 2 && lane == 0;  // one thread per half issues stores
    for (int i = threadIdx.x - 64; i < L.N_total; i += 256) sBias[i] = args.bias[i];
    asm volatile("bar.sync 1, 256;" ::: "memory");
    uint8_t* myout = sOut + half * 16384;
    long long row0[kMaxT];
    int cb = 0;
    for (int i = 0;; ++i) {
      const int n = unit_rows(args, i, &cb, row0);
      if (n == 0) break;
      const int buf = i % L.nbuf;
      const uint32_t use = static_cast<uint32_t>(i / L.nbuf);
      mbar_wait(&acc_full[buf], use & 1u);
      tc_fence_after();
      if (kLogits) {
        if (half == 0) {
          for (int k = 0; k < n; ++k) {
            float v[16];
            tmem_ld16(tmem_base + lane_field + static_cast<uint32_t>(buf * L.group_cols + k * 16), v);
            tmem_ld_wait();
            const long long r = row0[k] + row;
            if (r < rows_end(args)) {
              float* o = static_cast<float*>(args.logits) + r * L.C;
              for (int c = 0; c < L.C; ++c) o[c] = v[c] + sBias[c];
            }
          }
        }
      } else {
        for (int k = 0; k < n; ++k) {
          for (int c = half * (N / 128); c < (half + 1) * (N / 128); ++c) {
            const uint32_t col = static_cast<uint32_t>(buf * L.group_cols + k * N + c * 64);
            uint32_t ra[32], rb[32];
            tmem_ld32_raw(tmem_base + lane_field + col, ra);
            tmem_ld32_raw(tmem_base + lane_field + col + 32, rb);
            tmem_ld_wait();
            // The half's staging tile is free once the previous store read it.
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
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
    if (!kLogits && issuer) tma_store_wait_all<0>();
  }

  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, static_cast<uint32_t>(L.tmem_cols));
  }
}

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

// Shared planner: N = columns per block (16 for logits), N_total = all columns.
bool plan(int K, int N, int N_total, bool relu, bool logits, int C, DenseLayout* out) {
  const int kchunks = (K + 63) / 64;
  const int nh = (N + 255) / 256;
  const int NH = N / nh;
  bool found = false;
  DenseLayout best;
  double best_cost = 0.0;
  for (int T = 1; T <= kMaxT; ++T)
    for (int nbuf = 1; nbuf <= 2; ++nbuf) {
      const int cols = nbuf * T * N;
      if (cols > 512) continue;
      DenseLayout L;
      L.K = K;
      L.N = N;
      L.N_total = N_total;
      L.ncb = N_total / N;
      L.logits = logits ? 1 : 0;
      L.C = C;
      L.kchunks = kchunks;
      L.T = T;
      L.nbuf = nbuf;
      L.nh = nh;
      L.NH = NH;
      L.relu = relu ? 1 : 0;
      L.group_cols = T * N;
      int tc = 32;
      while (tc < cols) tc <<= 1;
      L.tmem_cols = tc;
      L.stage_bytes = static_cast<uint32_t>(T) * 16384u + static_cast<uint32_t>(N) * 128u;
      const uint32_t out_bytes = logits ? 0u : 2 * 16384u;
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
      const double mma = static_cast<double>(kchunks) * T * std::max(2.0 * N, 4 * 46.0);
      const double ingress = static_cast<double>(kchunks) * L.stage_bytes / 44.0;
      const double epi = T * (logits ? 200.0 : (N / 64.0) * 120.0) + 400.0;
      const double cost = (std::max(mma, ingress) + (nbuf == 1 ? epi : 0.0)) / T;
      if (!found || cost < best_cost) {
        best = L;
        best_cost = cost;
        found = true;
      }
    }
  if (found) *out = best;
  return found;
}

}  // namespace

bool dense_plan(int K, int N, bool relu, DenseLayout* out) {
  if (K < 1 || K % 8 != 0 || N < 128 || N % 128 != 0) return false;
  // Column blocks of up to 512 (the TMEM width of one accumulator tile).
  int block = 0;
  for (int b : {512, 384, 256, 128})
    if (N % b == 0) {
      block = b;
      break;
    }
  return plan(K, block, N, relu, false, 0, out);
}

bool dense_logits_plan(int K, int C, DenseLayout* out) {
  if (K < 1 || K % 8 != 0 || C < 1 || C > 16) return false;
  return plan(K, 16, 16, false, true, C, out);
}

int dense_launch(const DenseArgs& args, const void* x, long long x_rows, const void* w, void* y,
                 int grid, cudaStream_t stream) {
  const DenseLayout& L = args.L;
  CUtensorMap mx, mw, my;
  if (make_bf16_map(&mx, x, static_cast<uint64_t>(L.K), static_cast<uint64_t>(x_rows), 128) != 0)
    return -1;
  if (L.logits) {
    // W [C][K]: one 16-row box, rows C..15 zero-filled.
    if (make_bf16_map(&mw, w, static_cast<uint64_t>(L.K), static_cast<uint64_t>(L.C), 16) != 0)
      return -1;
    my = mx;  // unused
  } else {
    if (make_bf16_map(&mw, w, static_cast<uint64_t>(L.K), static_cast<uint64_t>(L.N_total), 64) != 0)
      return -1;
    // Y clipped at row_end: rows of a tile past the worker's range are not written.
    if (make_bf16_map(&my, y, static_cast<uint64_t>(L.N_total), static_cast<uint64_t>(args.row_end),
                      128) != 0)
      return -1;
  }
  const long long tiles = (args.row_end - args.row_begin + 127) / 128;
  if (tiles <= 0) return 0;
  grid = static_cast<int>(std::min<long long>(grid, (tiles + L.T - 1) / L.T * L.ncb));
  auto go = [&](auto kernel) {
    if (ensure_smem_attr(kernel, static_cast<int>(kSmemBudget)) != 0) return -4;
    kernel<<<grid, kThreads, L.smem_bytes, stream>>>(mx, mw, my, args);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
  };
  return L.logits ? go(dense_sm100<true>) : go(dense_sm100<false>);
}

}  // namespace es
