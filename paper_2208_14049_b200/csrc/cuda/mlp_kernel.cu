// K1 — fused two-layer MLP member forward (see mlp_kernel.cuh for the design).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "mlp_kernel.cuh"

namespace es {

using namespace sm100;

namespace {

constexpr int kThreads = 192;            // 6 warps: TMA, MMA, 4 x epilogue
constexpr uint32_t kSmemBudget = 232448; // 227 KB opt-in maximum per CTA
constexpr uint32_t kMinSmem = 120 * 1024;// keep one CTA per SM (TMEM is allocated whole)

__device__ __forceinline__ bool tile_at(const Mlp2Args& a, long long t, long long* row0,
                                        int* rows) {
  const long long per_seg = (a.seg_size + a.b - 1) / a.b;
  const long long seg = a.seg_begin + t / per_seg;
  const long long s0 = seg * a.seg_size;
  const long long s1 = min(s0 + (long long)a.seg_size, a.nb);
  const long long r0 = s0 + (t % per_seg) * a.b;
  if (r0 >= s1) return false;
  *row0 = r0;
  *rows = static_cast<int>(min((long long)a.b, s1 - r0));
  return true;
}

__global__ void __launch_bounds__(kThreads, 1)
    member_mlp2_sm100(const __grid_constant__ CUtensorMap tm_x,
                      const __grid_constant__ CUtensorMap tm_w1,
                      const __grid_constant__ CUtensorMap tm_w2, const Mlp2Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const Mlp2Layout& L = args.L;
  uint8_t* sH = smem;
  uint8_t* sW2 = smem + L.off_w2;
  uint8_t* sStage = smem + L.off_stage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* full = bars;                 // [stages] TMA -> MMA
  uint64_t* empty = bars + L.stages;     // [stages] MMA -> TMA
  uint64_t* acc_full = empty + L.stages; // [2] layer-1 accumulators ready
  uint64_t* acc_empty = acc_full + 2;    // [2] TMEM buffer drained
  uint64_t* acc2_full = acc_empty + 2;   // [2] layer-2 accumulators ready
  uint64_t* h_full = acc2_full + 2;      // Hs written by the epilogue
  uint64_t* h_empty = h_full + 1;        // Hs consumed by layer-2 UMMA
  uint64_t* w2_full = h_empty + 1;       // W2 resident
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w2_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int mchunks = L.H >> 7;
  const int kc2n = L.H >> 6;
  const long long per_seg = (args.seg_size + args.b - 1) / args.b;
  const long long total = (args.seg_end - args.seg_begin) * per_seg;

  if (threadIdx.x == 0) {
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
      mbar_init(&acc2_full[i], 1);
    }
    mbar_init(h_full, 4);
    mbar_init(h_empty, 1);
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
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      const uint64_t pol_stream = l2_policy_evict_normal();  // X: read once; evict_first cost W its L2 residency
      const uint64_t pol_keep = l2_policy_evict_last();     // weights: every CTA re-reads
      mbar_arrive_expect_tx(w2_full, static_cast<uint32_t>(kc2n) * 2048u);
      for (int kc = 0; kc < kc2n; ++kc)
        tma_load_2d(sW2 + kc * 2048, &tm_w2, w2_full, kc * 64, 0, pol_keep);
      int stage = 0;
      uint32_t phase = 0;
      for (long long t = blockIdx.x; t < total; t += gridDim.x) {
        long long row0;
        int rows;
        if (!tile_at(args, t, &row0, &rows)) continue;
        for (int kc = 0; kc < L.kchunks; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* st = sStage + static_cast<size_t>(stage) * L.stage_bytes;
          mbar_arrive_expect_tx(&full[stage], L.stage_bytes);
          tma_load_2d(st, &tm_x, &full[stage], kc * 64, static_cast<int32_t>(row0), pol_stream);
          for (int mc = 0; mc < mchunks; ++mc)
            tma_load_2d(st + L.x_bytes + mc * 16384, &tm_w1, &full[stage], kc * 64, mc * 128,
                        pol_keep);
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ UMMA issuer
      const uint32_t idesc1 = idesc_bf16_f32(128, L.N);
      const uint32_t idesc2 = idesc_bf16_f32(128, 16);
      const uint32_t sH_addr = smem_u32(sH);
      const uint32_t sW2_addr = smem_u32(sW2);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t h_parity = 0;
      bool w2_ready = false;
      int pending = -1;  // TMEM buffer whose layer-2 UMMA is still to be issued
      auto issue_layer2 = [&](int buf, bool already_waited) {
        if (!w2_ready) {
          mbar_wait(w2_full, 0);
          w2_ready = true;
        }
        if (!already_waited) mbar_wait(h_full, h_parity);
        h_parity ^= 1u;
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(buf * L.buf_cols);
        for (int kc = 0; kc < kc2n; ++kc)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t a = sdesc_k128(sH_addr + kc * L.h_chunk_stride + j * 32);
            const uint64_t b = sdesc_k128(sW2_addr + kc * 2048 + j * 32);
            umma_bf16(d, a, b, idesc2, (kc | j) != 0);
          }
        umma_commit(&acc2_full[buf]);
        umma_commit(h_empty);
      };
      int k = 0;
      for (long long t = blockIdx.x; t < total; t += gridDim.x) {
        long long row0;
        int rows;
        if (!tile_at(args, t, &row0, &rows)) continue;
        const int buf = k % L.nbuf;
        const uint32_t use = static_cast<uint32_t>(k / L.nbuf);
        if (pending == buf) {  // single buffer: finish the previous tile first
          issue_layer2(pending, false);
          pending = -1;
        }
        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d0 = tmem_base + static_cast<uint32_t>(buf * L.buf_cols);
        for (int kc = 0; kc < L.kchunks; ++kc) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sx = smem_u32(sStage + static_cast<size_t>(stage) * L.stage_bytes);
          const uint32_t sw = sx + L.x_bytes;
          for (int mc = 0; mc < mchunks; ++mc)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint64_t a = sdesc_k128(sw + mc * 16384 + j * 32);
              const uint64_t b = sdesc_k128(sx + j * 32);
              umma_bf16(d0 + static_cast<uint32_t>(mc * L.N), a, b, idesc1, (kc | j) != 0);
            }
          umma_commit(&empty[stage]);
          if (++stage == L.stages) {
            stage = 0;
            phase ^= 1u;
          }
          if (pending >= 0 && mbar_test(h_full, h_parity)) {
            issue_layer2(pending, true);
            pending = -1;
          }
        }
        umma_commit(&acc_full[buf]);
        if (pending >= 0) issue_layer2(pending, false);
        pending = buf;
        ++k;
      }
      if (pending >= 0) issue_layer2(pending, false);
    }
  } else {
    // -------------------------------------------------- epilogue (4 warps)
    const int q = warp & 3;  // TMEM lane quadrant this warp may touch
    const uint32_t lane_field = static_cast<uint32_t>(q * 32) << 16;
    int k = 0;
    for (long long t = blockIdx.x; t < total; t += gridDim.x) {
      long long row0;
      int rows;
      if (!tile_at(args, t, &row0, &rows)) continue;
      const int buf = k % L.nbuf;
      const uint32_t use = static_cast<uint32_t>(k / L.nbuf);
      const uint32_t tbuf = tmem_base + lane_field + static_cast<uint32_t>(buf * L.buf_cols);
      mbar_wait(&acc_full[buf], use & 1u);
      tc_fence_after();
      mbar_wait(h_empty, (static_cast<uint32_t>(k) & 1u) ^ 1u);
      const int cols = (rows + 15) & ~15;
      for (int mc = 0; mc < mchunks; ++mc) {
        const int h = mc * 128 + q * 32 + lane;
        const float bias = __ldg(args.bias1 + h);
        for (int c0 = 0; c0 < cols; c0 += 16) {
          float v[16];
          tmem_ld16(tbuf + static_cast<uint32_t>(mc * L.N + c0), v);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float y = fmaxf(v[i] + bias, 0.0f);
            *reinterpret_cast<__nv_bfloat16*>(
                sH + sw128_offset(static_cast<uint32_t>(c0 + i), static_cast<uint32_t>(h),
                                  L.h_chunk_stride)) = __float2bfloat16_rn(y);
          }
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(h_full);

      mbar_wait(&acc2_full[buf], use & 1u);
      tc_fence_after();
      float z[16];
      tmem_ld16(tbuf, z);
      const int r = q * 32 + lane;
      if (r < rows) {
        float* o = args.out + (row0 + r) * L.C;
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c < L.C) o[c] = z[c] + __ldg(args.bias2 + c);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
      ++k;
    }
  }

  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, static_cast<uint32_t>(L.tmem_cols));
  }
}

// ---------------------------------------------------------------- host
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// bf16 [rows][inner] row-major, box = 64 x box_rows, 128-byte swizzle.
int make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows,
             uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

}  // namespace

bool mlp2_plan(int K, int H, int C, int b, Mlp2Layout* out) {
  if (K < 1 || K % 8 != 0 || H < 128 || H % 128 != 0 || H > 512 || C < 1 || C > 16 || b < 1 ||
      b > 256)
    return false;
  Mlp2Layout L;
  L.H = H;
  L.C = C;
  L.K = K;
  L.N = std::max(16, (b + 15) / 16 * 16);
  L.kchunks = (K + 63) / 64;
  L.h_chunk_stride = static_cast<uint32_t>(L.N) * 128u;
  const uint32_t h_bytes = static_cast<uint32_t>(H / 64) * L.h_chunk_stride;
  L.off_w2 = align_up(h_bytes, 1024);
  L.off_stage = align_up(L.off_w2 + static_cast<uint32_t>(H / 64) * 2048u, 1024);
  L.x_bytes = static_cast<uint32_t>(L.N) * 128u;
  L.stage_bytes = static_cast<uint32_t>(L.N + H) * 128u;
  const uint32_t bar_bytes = 256;
  const uint32_t room = kSmemBudget - 1024 - bar_bytes;
  if (L.off_stage >= room) return false;
  L.stages = static_cast<int>(std::min<uint32_t>(6, (room - L.off_stage) / L.stage_bytes));
  if (L.stages < 2) return false;
  L.off_bar = L.off_stage + static_cast<uint32_t>(L.stages) * L.stage_bytes;
  // Layer-2 UMMA reads 128 rows of the last Hs chunk; they must stay in smem.
  const uint32_t h_read_end = static_cast<uint32_t>(H / 64 - 1) * L.h_chunk_stride + 128u * 128u;
  L.smem_bytes = std::max({L.off_bar + bar_bytes + 1024, h_read_end + 1024, kMinSmem});
  if (L.smem_bytes > kSmemBudget) return false;
  L.buf_cols = (H / 128) * L.N;
  if (L.buf_cols > 512) return false;
  L.nbuf = 2 * L.buf_cols <= 512 ? 2 : 1;
  int need = L.nbuf * L.buf_cols;
  int cols = 32;
  while (cols < need) cols <<= 1;
  L.tmem_cols = cols;
  *out = L;
  return true;
}

int num_sms(int device) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n;
}

int mlp2_launch(const Mlp2Args& args, const void* x, const void* w1, const void* w2, int grid,
                cudaStream_t stream) {
  const Mlp2Layout& L = args.L;
  CUtensorMap mx, mw1, mw2;
  if (make_map(&mx, x, static_cast<uint64_t>(L.K), static_cast<uint64_t>(args.nb),
               static_cast<uint32_t>(L.N)) != 0)
    return -1;
  if (make_map(&mw1, w1, static_cast<uint64_t>(L.K), static_cast<uint64_t>(L.H), 128) != 0)
    return -1;
  if (make_map(&mw2, w2, static_cast<uint64_t>(L.H), static_cast<uint64_t>(L.C), 16) != 0)
    return -1;
  static std::mutex attr_mu;
  static unsigned long long attr_done = 0;  // one bit per device ordinal
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lock(attr_mu);
    if (!(attr_done & (1ull << dev))) {
      if (cudaFuncSetAttribute(member_mlp2_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(kSmemBudget)) != cudaSuccess)
        return -4;
      attr_done |= 1ull << dev;
    }
  }
  const long long per_seg = (args.seg_size + args.b - 1) / args.b;
  const long long tiles = (args.seg_end - args.seg_begin) * per_seg;
  if (tiles <= 0) return 0;
  grid = static_cast<int>(std::min<long long>(grid, tiles));
  member_mlp2_sm100<<<grid, kThreads, L.smem_bytes, stream>>>(mx, mw1, mw2, args);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace es
