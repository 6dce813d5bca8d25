// X staging, synthetic weights, K3 combine, SIMT cross-check member.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "aux_kernels.cuh"

#include <algorithm>
#include <cstdlib>

namespace es {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__device__ __forceinline__ float unit24(uint64_t key, uint64_t idx) {
  const uint64_t h = splitmix64(key ^ (idx * 0x9e3779b97f4a7c15ULL));
  return __fdiv_rn(static_cast<float>(h >> 40), 16777216.0f);
}

__device__ __forceinline__ uint64_t stream_key(uint64_t seed, int layer, int is_bias) {
  return splitmix64(seed * 0x100000001b3ULL + static_cast<uint64_t>(2 * layer + is_bias + 1));
}

__global__ void convert_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y,
                               size_t n) {
  const size_t n4 = n / 4;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  __nv_bfloat162* y2 = reinterpret_cast<__nv_bfloat162*>(y);
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float4 v = __ldcs(x4 + i);
    y2[2 * i] = __floats2bfloat162_rn(v.x, v.y);
    y2[2 * i + 1] = __floats2bfloat162_rn(v.z, v.w);
  }
  for (size_t i = n4 * 4 + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}

template <bool kBf16>
__global__ void dense_layer_kernel(uint64_t seed, int layer, int fan_in, int fan_out, float limit,
                                   void* w, float* b) {
  const uint64_t wkey = stream_key(seed, layer, 0);
  const uint64_t n = static_cast<uint64_t>(fan_in) * fan_out;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float u = unit24(wkey, i);
    const float v = __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), limit);
    if (kBf16)
      static_cast<__nv_bfloat16*>(w)[i] = __float2bfloat16_rn(v);
    else
      static_cast<float*>(w)[i] = v;
  }
  const uint64_t bkey = stream_key(seed, layer, 1);
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < fan_out; o += gridDim.x * blockDim.x) {
    const float u = unit24(bkey, static_cast<uint64_t>(o));
    b[o] = __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), 0.01f);
  }
}

constexpr int kRowsPerBlock = 128;

// Cooperative, vectorised copy of n floats global -> shared.
__device__ __forceinline__ void stage_in(float* dst, const float* __restrict__ src, int n) {
  if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0 && (n & 3) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int i = threadIdx.x; i < n / 4; i += blockDim.x) d4[i] = __ldcs(s4 + i);
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldcs(src + i);
  }
}

__device__ __forceinline__ void stage_out(float* __restrict__ dst, const float* src, int n) {
  if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && (n & 3) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int i = threadIdx.x; i < n / 4; i += blockDim.x) __stcs(d4 + i, s4[i]);
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) __stcs(dst + i, src[i]);
  }
}

// blockDim.x rows per block; every member's [rows][C] slice is staged into
// shared memory up front (M independent 16-B load streams in flight), then each
// thread folds its own row across members.  The result reuses member 0's slot:
// thread r only ever reads and writes row r there, so no barrier is needed
// between the fold and the write-back.
__global__ void __launch_bounds__(kRowsPerBlock) combine_kernel(const CombineArgs a) {
  extern __shared__ __align__(16) float tiles[];
  const int R = blockDim.x;
  const long long row0 = static_cast<long long>(blockIdx.x) * R;
  const int nrows = static_cast<int>(min(static_cast<long long>(R), a.rows - row0));
  const int C = a.C;
  const int n = nrows * C;
  const int r = threadIdx.x;
  const bool active = r < nrows;

  for (int m = 0; m < a.M; ++m) stage_in(tiles + m * R * C, a.logits[m] + row0 * C, n);
  __syncthreads();

  float acc[kMaxClasses];
#pragma unroll
  for (int c = 0; c < kMaxClasses; ++c) acc[c] = 0.0f;
  if (active) {
    for (int m = 0; m < a.M; ++m) {
      const float* tile = tiles + m * R * C;
      float z[kMaxClasses];
#pragma unroll
      for (int c = 0; c < kMaxClasses; ++c) z[c] = c < C ? tile[r * C + c] : 0.0f;
      if (a.softmax) {
        float mx = z[0];
#pragma unroll
        for (int c = 1; c < kMaxClasses; ++c)
          if (c < C) mx = z[c] > mx ? z[c] : mx;
        float s = 0.0f;
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c)
          if (c < C) {
            z[c] = expf(__fsub_rn(z[c], mx));
            s = __fadd_rn(s, z[c]);
          }
        const float inv = __fdiv_rn(1.0f, s);
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c)
          if (c < C) z[c] = __fmul_rn(z[c], inv);
      }
      if (a.rule == kVote) {
        int best = 0;
        float top = z[0];
#pragma unroll
        for (int c = 1; c < kMaxClasses; ++c)
          if (c < C && z[c] > top) {
            top = z[c];
            best = c;
          }
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c)
          if (c == best) acc[c] = __fadd_rn(acc[c], 1.0f);
      } else {
        const float w = a.weight[m];
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c)
          if (c < C) acc[c] = __fadd_rn(acc[c], __fmul_rn(z[c], w));
      }
    }
    int best = 0;
    float top = acc[0];
#pragma unroll
    for (int c = 0; c < kMaxClasses; ++c) {
      if (c < C) tiles[r * C + c] = acc[c];
      if (c > 0 && c < C && acc[c] > top) {
        top = acc[c];
        best = c;
      }
    }
    if (a.argmax) a.argmax[row0 + r] = best;
  }
  __syncthreads();
  stage_out(a.y + row0 * C, tiles, n);
}

// One block per sample: fp32 accumulation over bf16 operands, hidden rounded
// to bf16 exactly where the tensor-core kernel rounds it.
__global__ void mlp2_simt_kernel(const __nv_bfloat16* __restrict__ x, int K,
                                 const __nv_bfloat16* __restrict__ w1, const float* __restrict__ b1,
                                 int H, const __nv_bfloat16* __restrict__ w2,
                                 const float* __restrict__ b2, int C, long long row_begin,
                                 float* __restrict__ out) {
  extern __shared__ float hid[];
  const long long row = row_begin + blockIdx.x;
  const __nv_bfloat16* xr = x + row * K;
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    const __nv_bfloat16* wr = w1 + static_cast<size_t>(h) * K;
    float acc = 0.0f;
    for (int k = 0; k < K; ++k) acc = fmaf(__bfloat162float(xr[k]), __bfloat162float(wr[k]), acc);
    hid[h] = __bfloat162float(__float2bfloat16_rn(fmaxf(acc + b1[h], 0.0f)));
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const __nv_bfloat16* wr = w2 + static_cast<size_t>(c) * H;
    float acc = 0.0f;
    for (int h = 0; h < H; ++h) acc = fmaf(hid[h], __bfloat162float(wr[h]), acc);
    out[row * C + c] = acc + b2[c];
  }
}

__global__ void synthetic_member_kernel(int model_id, int C, long long row_begin,
                                        long long row_end, float* __restrict__ out,
                                        const ClaimedRun* claim) {
  if (claim) {
    row_begin = claim->row_begin;
    row_end = claim->row_end;
  }
  const uint64_t km = splitmix64(static_cast<uint64_t>(model_id) + 1);
  const long long n = (row_end - row_begin) * C;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long row = row_begin + i / C;
    const int c = static_cast<int>(i % C);
    const uint64_t key = splitmix64(km ^ splitmix64(static_cast<uint64_t>(row) * 0x9e3779b9ULL) ^
                                    splitmix64(static_cast<uint64_t>(c) + 0x51ed270bULL));
    out[row * C + c] = __fdiv_rn(static_cast<float>(key >> 40), 16777216.0f);
  }
}

__global__ void features_kernel(uint64_t seed, size_t n, __nv_bfloat16* __restrict__ y) {
  const uint64_t base = seed * 0x2545f4914f6cdd1dULL;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint64_t h = splitmix64(base + i);
    y[i] = __float2bfloat16_rn(__fdiv_rn(static_cast<float>(h >> 40), 16777216.0f));
  }
}

__global__ void __launch_bounds__(256) claim_kernel(unsigned long long* counter, long long segments,
                                                    long long chunk, int seg_size, long long nb,
                                                    ClaimedRun* out, int* owner, int worker) {
  __shared__ long long run[2];
  if (threadIdx.x == 0) {
    const long long first = static_cast<long long>(atomicAdd(counter, static_cast<unsigned long long>(chunk)));
    const long long b = first < segments ? first : segments;
    const long long e = first + chunk < segments ? first + chunk : segments;
    run[0] = b;
    run[1] = e;
    const long long r1 = e * seg_size < nb ? e * seg_size : nb;
    *out = ClaimedRun{b, e, b * seg_size, b < e ? r1 : b * seg_size};
  }
  __syncthreads();
  if (owner)
    for (long long s = run[0] + threadIdx.x; s < run[1]; s += blockDim.x) owner[s] = worker;
}

int grid_for(size_t n, int threads) {
  size_t blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 32) blocks = 148 * 32;
  return static_cast<int>(blocks < 1 ? 1 : blocks);
}

}  // namespace

int convert_f32_to_bf16(const float* x, __nv_bfloat16* y, size_t n, cudaStream_t s) {
  if (n == 0) return 0;
  convert_kernel<<<grid_for(n / 4 + 1, 256), 256, 0, s>>>(x, y, n);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int generate_dense_layer(uint64_t seed, int layer, int fan_in, int fan_out, float limit,
                         __nv_bfloat16* w, float* b, cudaStream_t s) {
  const size_t n = static_cast<size_t>(fan_in) * fan_out;
  dense_layer_kernel<true><<<grid_for(n, 256), 256, 0, s>>>(seed, layer, fan_in, fan_out, limit,
                                                            w, b);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int generate_dense_layer_f32(uint64_t seed, int layer, int fan_in, int fan_out, float limit,
                             float* w, float* b, cudaStream_t s) {
  const size_t n = static_cast<size_t>(fan_in) * fan_out;
  dense_layer_kernel<false><<<grid_for(n, 256), 256, 0, s>>>(seed, layer, fan_in, fan_out, limit,
                                                             w, b);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int claim_launch(unsigned long long* counter, long long segments, long long chunk, int seg_size,
                 long long nb, ClaimedRun* out, int* owner, int worker, cudaStream_t s) {
  claim_kernel<<<1, 256, 0, s>>>(counter, segments, chunk, seg_size, nb, out, owner, worker);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int synthetic_member_launch(int model_id, int C, int seg_size, long long seg_begin,
                            long long seg_end, long long nb, float* out, cudaStream_t s,
                            const ClaimedRun* claim) {
  const long long r0 = seg_begin * seg_size;
  const long long r1 = seg_end * static_cast<long long>(seg_size) < nb ? seg_end * seg_size : nb;
  if (r1 <= r0) return 0;
  synthetic_member_kernel<<<grid_for(static_cast<size_t>((r1 - r0) * C), 256), 256, 0, s>>>(
      model_id, C, r0, r1, out, claim);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int generate_features_bf16(uint64_t seed, size_t n, __nv_bfloat16* y, cudaStream_t s) {
  if (n == 0) return 0;
  features_kernel<<<grid_for(n, 256), 256, 0, s>>>(seed, n, y);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// One thread per row, the row's C logits of each member read straight into
// registers (8-byte loads when C is even; a warp's 32 rows are one contiguous
// 32*4C-byte run, so the loads of one member hit the same L1 lines), no shared
// memory and no block barrier: occupancy hides the HBM latency.  Same fold
// arithmetic, in the same order, as combine_kernel.
template <int C>
__global__ void __launch_bounds__(256) combine_rows_kernel(const CombineArgs a) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r < a.rows;
       r += stride) {
    float acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = 0.0f;
    for (int m = 0; m < a.M; ++m) {
      float z[C];
      const float* src = a.logits[m] + r * C;
      if constexpr (C % 2 == 0) {
#pragma unroll
        for (int c = 0; c < C; c += 2) {
          const float2 v = __ldcs(reinterpret_cast<const float2*>(src + c));
          z[c] = v.x;
          z[c + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int c = 0; c < C; ++c) z[c] = __ldcs(src + c);
      }
      if (a.softmax) {
        float mx = z[0];
#pragma unroll
        for (int c = 1; c < C; ++c) mx = z[c] > mx ? z[c] : mx;
        float sum = 0.0f;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          z[c] = expf(__fsub_rn(z[c], mx));
          sum = __fadd_rn(sum, z[c]);
        }
        const float inv = __fdiv_rn(1.0f, sum);
#pragma unroll
        for (int c = 0; c < C; ++c) z[c] = __fmul_rn(z[c], inv);
      }
      if (a.rule == kVote) {
        int best = 0;
        float top = z[0];
#pragma unroll
        for (int c = 1; c < C; ++c)
          if (z[c] > top) {
            top = z[c];
            best = c;
          }
#pragma unroll
        for (int c = 0; c < C; ++c)
          if (c == best) acc[c] = __fadd_rn(acc[c], 1.0f);
      } else {
        const float w = a.weight[m];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(z[c], w));
      }
    }
    int best = 0;
    float top = acc[0];
#pragma unroll
    for (int c = 1; c < C; ++c)
      if (acc[c] > top) {
        top = acc[c];
        best = c;
      }
    float* dst = a.y + r * C;
    if constexpr (C % 2 == 0) {
#pragma unroll
      for (int c = 0; c < C; c += 2) __stcs(reinterpret_cast<float2*>(dst + c), make_float2(acc[c], acc[c + 1]));
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c) __stcs(dst + c, acc[c]);
    }
    if (a.argmax) a.argmax[r] = best;
  }
}

template <int C>
int launch_rows(const CombineArgs& a, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long want = (a.rows + 255) / 256;
  const long long blocks = std::min<long long>(want, static_cast<long long>(sms) * 8);
  combine_rows_kernel<C><<<static_cast<unsigned>(blocks), 256, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int combine_launch(const CombineArgs& a, cudaStream_t s) {
  if (a.rows <= 0) return 0;
  if (a.M < 1 || a.M > kMaxMembers || a.C < 1 || a.C > kMaxClasses) return -2;
  if (!std::getenv("ES_COMBINE_STAGED")) {
    switch (a.C) {
      case 2: return launch_rows<2>(a, s);
      case 3: return launch_rows<3>(a, s);
      case 4: return launch_rows<4>(a, s);
      case 5: return launch_rows<5>(a, s);
      case 8: return launch_rows<8>(a, s);
      case 10: return launch_rows<10>(a, s);
      case 16: return launch_rows<16>(a, s);
      default: break;  // other widths: the staged kernel
    }
  }
  // Rows per block: 128, fewer when M*C slices would not fit 48 KB of smem.
  int R = kRowsPerBlock;
  while (R > 8 && static_cast<size_t>(a.M) * R * a.C * sizeof(float) > 48 * 1024) R /= 2;
  const size_t smem = static_cast<size_t>(a.M) * R * a.C * sizeof(float);
  const long long blocks = (a.rows + R - 1) / R;
  combine_kernel<<<static_cast<unsigned>(blocks), R, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int mlp2_simt_launch(const __nv_bfloat16* x, long long nb, int K, const __nv_bfloat16* w1,
                     const float* b1, int H, const __nv_bfloat16* w2, const float* b2, int C,
                     long long row_begin, long long row_end, float* out, cudaStream_t s) {
  (void)nb;
  if (row_end <= row_begin) return 0;
  mlp2_simt_kernel<<<static_cast<unsigned>(row_end - row_begin), 256, H * sizeof(float), s>>>(
      x, K, w1, b1, H, w2, b2, C, row_begin, out);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace es
