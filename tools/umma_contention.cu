// Design evidence, not product: (1) rate of a back-to-back tcgen05.mma chain
// (M=128, N, K=16, planar no-swizzle operands -- the conv2 UMMA shape) while
// other warps of the CTA stream shared memory (STS.128 / LDS.128), i.e. is the
// conv stack's UMMA chain slowed by shared-memory bandwidth; (2) the same chain
// issued over an SM pair (cta_group::2, M = 256, each SM holding half of B).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I../paper_2208_14049_b200/csrc umma_contention.cu -o umma_contention
#include <cuda_runtime.h>

#include <cstdio>

#include "cuda/sm100.cuh"

using namespace es::sm100;

constexpr long long kWindow = 40000;  // load warps run this many clocks (inside the chain)
constexpr int kRegion = 100 * 1024;  // load warps use smem from here (8 KB each)

__global__ void __launch_bounds__(384, 1) contention(int N, int reps, int kind, int load_warps,
                                                     unsigned long long* out, uint4* gout) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  for (int i = threadIdx.x; i < (kRegion + 8 * 8192) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    done = 0;
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long bytes = 0;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
    const uint32_t idesc = idesc_bf16_f32(128, N > 0 ? N : 96);
    const uint64_t ad = sdesc_planar(a, 160 * 16), bd = sdesc_planar(b, N * 16);
    t0 = clock64();
    if (N > 0) {
      for (int r = 0; r < reps; ++r) umma_bf16(tmem, ad, bd, idesc, r != 0);
      umma_commit(&bar);
      mbar_wait(&bar, 0);
    } else {  // no UMMAs: the load warps' uncontended rate
      while (clock64() - t0 < kWindow + 2000) {
      }
    }
    t1 = clock64();
    done = 1;
  } else if (warp >= 4 && warp < 4 + load_warps) {
    uint4* p = reinterpret_cast<uint4*>(smem + kRegion + (warp - 4) * 8192) + lane;
    uint4 acc = make_uint4(0, 0, 0, 0);
    const long long ts = clock64();
    long long now = ts;
    while (now - ts < kWindow) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const uint32_t addr = smem_u32(p + u * 32);
        if (kind == 0) {
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(u), "r"(lane),
                       "r"(acc.x), "r"(acc.y)
                       : "memory");
        } else if (kind == 2) {  // shuffles (bytes counted as 16 per lane, like the others)
          acc.x = __shfl_down_sync(0xffffffffu, acc.x + u, 1);
          acc.y = __shfl_down_sync(0xffffffffu, acc.y + u, 2);
          acc.z = __shfl_down_sync(0xffffffffu, acc.z + u, 1);
          acc.w = __shfl_down_sync(0xffffffffu, acc.w + u, 2);
        } else if (kind == 3) {  // global stores, 16 B per lane, coalesced
          gout[((blockIdx.x * 8 + (warp - 4)) * 16 + u) * 32 + lane] = make_uint4(u, lane, acc.x, 0);
        } else if (kind == 4) {  // tcgen05.ld 32 columns x 32 lanes (= 16 B per lane x 8)
          uint32_t r[32];
          tmem_ld32_raw(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 256u, r);
          tmem_ld_wait();
          acc.x ^= r[u] + r[31 - u];
        } else {
          uint32_t x, y, z, w;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                       : "r"(addr)
                       : "memory");
          acc.x ^= x + z;
          acc.y ^= y + w;
        }
      }
      bytes += 16 * 512;
      now = clock64();
    }
    if (acc.x == 12345) p[0] = acc;
  }
  __shared__ unsigned long long total;
  if (threadIdx.x == 0) total = 0;
  __syncthreads();
  if (lane == 0 && bytes) atomicAdd(&total, bytes);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = static_cast<unsigned long long>(t1 - t0);
    out[1] = total;
  }
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_rate(int N, int reps, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc_pair(&slot, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (cluster_ctarank() == 0 && threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
    const uint32_t idesc = idesc_bf16_f32(256, N);
    const uint64_t ad = sdesc_planar(a, 128 * 16), bd = sdesc_planar(b, (N / 2) * 16);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) umma_bf16_pair(tmem, ad, bd, idesc, r != 0);
    umma_commit_pair(&bar, 3);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = static_cast<unsigned long long>(t1 - t0);
  } else if (threadIdx.x == 0) {
    mbar_wait_cluster(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc_pair(tmem, 256);
}

// Layer 2 of the pair head: M = 256 over the pair, A (bf16 hidden) from
// TMEM, N = 16, one dependent chain (or `parts` independent chains) -- vs the
// same UMMAs issued per CTA with cta_group::1 (M = 128 each, both SMs in
// parallel).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    layer2_rate(int pair_mode, int parts, int reps, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    if (pair_mode) tmem_alloc_pair(&slot, 512);
    else tmem_alloc(&slot, 512);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  const bool issuer = pair_mode ? (cluster_ctarank() == 0 && threadIdx.x < 32) : threadIdx.x < 32;
  if (issuer) {
    const uint32_t b = smem_u32(smem + 64 * 1024);
    const uint32_t idesc = idesc_bf16_f32(pair_mode ? 256 : 128, 16);
    const uint64_t bd = sdesc_k128(b);
    const long long t0 = clock64();
    if (parts == 0) {
      // unrolled: 32 UMMAs per round with compile-time offsets (4 chains)
      for (int r = 0; r < reps; r += 32) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const uint32_t a = tmem + static_cast<uint32_t>(i * 8);
          const uint32_t d = tmem + 256u + 16u * static_cast<uint32_t>(i & 3);
          if (elect_one()) {
            if (pair_mode) umma_bf16_pair_ta(d, a, bd + (i % 8) * 2, idesc, (r | (i >> 2)) != 0);
            else umma_bf16_ta(d, a, bd + (i % 8) * 2, idesc, (r | (i >> 2)) != 0);
          }
        }
      }
    } else {
      for (int r = 0; r < reps; ++r) {
        const uint32_t a = tmem + static_cast<uint32_t>((r % 32) * 8);
        const uint32_t d = tmem + 256u + 16u * static_cast<uint32_t>(r % parts);
        if (elect_one()) {
          if (pair_mode) umma_bf16_pair_ta(d, a, bd + (r % 8) * 2, idesc, r >= parts);
          else umma_bf16_ta(d, a, bd + (r % 8) * 2, idesc, r >= parts);
        }
      }
    }
    if (elect_one()) {
      if (pair_mode) umma_commit_pair(&bar, 3);
      else umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = static_cast<unsigned long long>(t1 - t0);
  } else if (pair_mode && threadIdx.x == 0) {
    mbar_wait_cluster(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (threadIdx.x < 32) {
    if (pair_mode) tmem_dealloc_pair(tmem, 512);
    else tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int smem = kRegion + 8 * 8192 + 1024;
  cudaFuncSetAttribute(contention, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 1024;
  const char* kinds[] = {"STS ", "LDS ", "SHFL", "STG ", "TMLD"};
  uint4* gbuf;
  cudaMalloc(&gbuf, 148 * 8 * 16 * 32 * 16);
  for (int N : {0, 96})
    for (int kind = 0; kind < 5; ++kind)
      for (int w : {0, 1, 2, 4, 8}) {
        if (kind > 0 && w == 0) continue;
        contention<<<148, 384, smem>>>(N, reps, kind, w, d, gbuf);
        unsigned long long h[2] = {0, 0};
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        std::printf("N=%3d %s warps=%d: %6.1f clk/MMA  UMMA smem %5.1f B/clk  other %5.1f B/clk %s\n",
                    N, kinds[kind], w, double(h[0]) / reps,
                    (128.0 * 32 + N * 32.0) * reps / double(h[0]), double(h[1]) / double(kWindow),
                    cudaGetErrorString(cudaGetLastError()));
      }
  cudaFuncSetAttribute(layer2_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int pm = 0; pm < 2; ++pm)
    for (int parts : {0, 1, 4}) {
      layer2_rate<<<148, 128, 100 * 1024>>>(pm, parts, 512, d);
      unsigned long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      std::printf("layer2 %s N=16 A=tmem parts=%d (0 = unrolled, constant offsets): %6.1f clk/MMA %s\n",
                  pm ? "pair M=256 (cta_group::2)" : "per CTA M=128 (cta_group::1)", parts,
                  double(c) / 512, cudaGetErrorString(cudaGetLastError()));
    }
  cudaFuncSetAttribute(pair_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {64, 96, 128, 192, 256}) {
    pair_rate<<<148, 128, 100 * 1024>>>(N, reps, d);
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    std::printf("pair M=256 N=%3d: %6.1f clk/MMA  (%5.0f MAC/clk per SM) %s\n", N,
                double(c) / reps, 128.0 * N * 16 * reps / double(c),
                cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
