// FP32-accurate member kernels (design in fp32_kernels.cuh).
#include "fp32_kernels.cuh"

#include <algorithm>

namespace es {

namespace {

constexpr int kBM = 64, kBN = 64, kBK = 16, kThreads = 256;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Persistent SGEMM tiles of 64 rows x 64 outputs, K in steps of 16; each of
// the 256 threads owns a 4 x 4 block of outputs.  Operands are staged
// transposed (k-major) so the inner loop reads two float4s per k.
__global__ void __launch_bounds__(kThreads) f32_dense_kernel(const F32DenseArgs a) {
  __shared__ __align__(16) float As[kBK][kBM];
  __shared__ __align__(16) float Bs[kBK][kBN];
  const long long rb = a.claim ? a.claim->row_begin : a.row_begin;
  const long long re = a.claim ? a.claim->row_end : a.row_end;
  const long long mtiles = (re - rb + kBM - 1) / kBM;
  const int ntiles = (a.N + kBN - 1) / kBN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  for (long long t = blockIdx.x; t < mtiles * ntiles; t += gridDim.x) {
    const long long r0 = rb + (t / ntiles) * kBM;
    const int n0 = static_cast<int>(t % ntiles) * kBN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < a.K; k0 += kBK) {
      // 64 x 16 of x and of w: four elements per thread each.
      for (int i = threadIdx.x; i < kBM * kBK; i += kThreads) {
        const int m = i / kBK, k = i % kBK;
        const long long r = r0 + m;
        As[k][m] = (r < re && k0 + k < a.K) ? a.x[r * a.K + k0 + k] : 0.0f;
        const int n = n0 + m;
        Bs[k][m] = (n < a.N && k0 + k < a.K) ? __ldg(a.w + static_cast<long long>(n) * a.K + k0 + k)
                                              : 0.0f;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kBK; ++k) {
        const float4 av = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
        const float4 bv = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
        const float ar[4] = {av.x, av.y, av.z, av.w};
        const float br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long long r = r0 + ty * 4 + i;
      if (r >= re) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + tx * 4 + j;
        if (n >= a.N) continue;
        const float v = acc[i][j] + __ldg(a.b + n);
        a.y[r * a.N + n] = a.relu ? fmaxf(v, 0.0f) : v;
      }
    }
  }
}

// One sample at a time per CTA, conv2's weights resident in shared memory
// (row stride 9*c1 + 1 floats: threads of a warp read different output
// channels of one K index without bank conflicts).  The image and conv1's
// output (with a zero border) are staged per sample.  conv2: thread t owns
// channel t % c2 of positions t / c2, t / c2 + groups, ...; the positions'
// activations are warp-uniform (broadcast reads).  Every output is one fmaf
// chain in K order (tap-major, then input channel), like the oracle.
__global__ void __launch_bounds__(kThreads) f32_conv_kernel(const F32ConvArgs a) {
  extern __shared__ float smem[];
  const int S = a.S, P = a.P, G = S / P, GP = G + 2, c1 = a.c1, c2 = a.c2;
  const int K2 = 9 * c1, ws = K2 + 1;
  float* w2 = smem;                 // [c2][9*c1 + 1]
  float* img = w2 + c2 * ws;        // [S*S]
  float* a1 = img + S * S;          // [(G+2)*(G+2)][c1], border zero
  const long long rb = a.claim ? a.claim->row_begin : a.row_begin;
  const long long re = a.claim ? a.claim->row_end : a.row_end;
  for (int i = threadIdx.x; i < c2 * K2; i += kThreads) w2[(i / K2) * ws + i % K2] = a.w2[i];
  for (int i = threadIdx.x; i < GP * GP * c1; i += kThreads) a1[i] = 0.0f;
  const int groups = kThreads / c2;  // c2 divides 256 or groups = 0 (handled below)
  for (long long s = rb + blockIdx.x; s < re; s += gridDim.x) {
    __syncthreads();  // the previous sample's a1 / img reads are done
    for (int i = threadIdx.x; i < S * S; i += kThreads) img[i] = a.x[s * S * S + i];
    __syncthreads();
    for (int o = threadIdx.x; o < G * G * c1; o += kThreads) {
      const int c = o % c1, p = o / c1, pi = p / G, pj = p % G;
      float acc = 0.0f;
      for (int u = 0; u < P; ++u)
        for (int v = 0; v < P; ++v)
          acc = fmaf(img[(P * pi + u) * S + P * pj + v], __ldg(a.w1 + c * P * P + u * P + v), acc);
      a1[((pi + 1) * GP + pj + 1) * c1 + c] = fmaxf(acc + __ldg(a.b1 + c), 0.0f);
    }
    __syncthreads();
    float* dst = a.out + s * static_cast<long long>(G * G * c2);
    if (groups > 0 && threadIdx.x < groups * c2) {
      constexpr int kPos = 8;  // positions per pass of a thread
      const int co = threadIdx.x % c2, pg = threadIdx.x / c2;
      const float* w = w2 + co * ws;
      const float bias = __ldg(a.b2 + co);
      for (int p0 = pg; p0 < G * G; p0 += groups * kPos) {
        float acc[kPos];
        int base[kPos];
#pragma unroll
        for (int q = 0; q < kPos; ++q) {
          acc[q] = 0.0f;
          const int p = min(p0 + q * groups, G * G - 1);
          base[q] = ((p / G) * GP + p % G) * c1;  // a1 row of tap (dh, dw) = (-1, -1)
        }
        for (int tap = 0; tap < 9; ++tap) {
          const int toff = ((tap / 3) * GP + tap % 3) * c1;
          const float* wt = w + tap * c1;
          for (int ci = 0; ci < c1; ++ci) {
            const float wv = wt[ci];
#pragma unroll
            for (int q = 0; q < kPos; ++q) acc[q] = fmaf(a1[base[q] + toff + ci], wv, acc[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < kPos; ++q) {
          const int p = p0 + q * groups;
          if (p < G * G) dst[p * c2 + co] = fmaxf(acc[q] + bias, 0.0f);
        }
      }
    } else if (groups == 0) {  // c2 > 256: one output at a time
      for (int o = threadIdx.x; o < G * G * c2; o += kThreads) {
        const int co = o % c2, p = o / c2;
        const float* w = w2 + co * ws;
        const int b0 = ((p / G) * GP + p % G) * c1;
        float acc = 0.0f;
        for (int tap = 0; tap < 9; ++tap)
          for (int ci = 0; ci < c1; ++ci)
            acc = fmaf(a1[b0 + ((tap / 3) * GP + tap % 3) * c1 + ci], w[tap * c1 + ci], acc);
        dst[p * c2 + co] = fmaxf(acc + __ldg(a.b2 + co), 0.0f);
      }
    }
  }
}

__global__ void features_f32_kernel(uint64_t seed, size_t n, float* __restrict__ y) {
  const uint64_t base = seed * 0x2545f4914f6cdd1dULL;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    y[i] = __fdiv_rn(static_cast<float>(mix64(base + i) >> 40), 16777216.0f);
}

size_t conv_smem(int S, int P, int c1, int c2) {
  const int G = S / P;
  return static_cast<size_t>(c2 * (9 * c1 + 1) + S * S + (G + 2) * (G + 2) * c1) * sizeof(float);
}

}  // namespace

int f32_dense_launch(const F32DenseArgs& a, int grid, cudaStream_t s) {
  if (a.K < 1 || a.N < 1) return -1;
  const long long tiles = (a.row_end - a.row_begin + kBM - 1) / kBM * ((a.N + kBN - 1) / kBN);
  if (tiles <= 0) return 0;
  grid = static_cast<int>(std::min<long long>(static_cast<long long>(grid) * 4, tiles));
  f32_dense_kernel<<<grid, kThreads, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

bool f32_conv_supported(int S, int P, int c1, int c2) {
  return P >= 1 && S >= P && S % P == 0 && c1 >= 1 && c2 >= 1 && conv_smem(S, P, c1, c2) <= 200 * 1024;
}

int f32_conv_launch(const F32ConvArgs& a, int grid, cudaStream_t s) {
  if (!f32_conv_supported(a.S, a.P, a.c1, a.c2)) return -1;
  const long long rows = a.row_end - a.row_begin;
  if (rows <= 0) return 0;
  const size_t smem = conv_smem(a.S, a.P, a.c1, a.c2);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(f32_conv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return -4;
  grid = static_cast<int>(std::min<long long>(static_cast<long long>(grid) * 4, rows));
  f32_conv_kernel<<<grid, kThreads, smem, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int generate_features_f32(uint64_t seed, size_t n, float* y, cudaStream_t s) {
  if (n == 0) return 0;
  const int grid = static_cast<int>(std::min<size_t>((n + 255) / 256, 65535));
  features_f32_kernel<<<grid, 256, 0, s>>>(seed, n, y);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace es
