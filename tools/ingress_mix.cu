// Design evidence, not product: does an SM ingest more than its TMA cap
// (~48 B/clk, tools/tma_bw.cu) when cp.async (LSU path) loads run beside TMA?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2208_14049_b200/csrc \
//        ingress_mix.cu -o ingress_mix
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "cuda/sm100.cuh"
#include "cuda/tma_host.hpp"

using namespace es::sm100;

// warp 0: TMA stream of 16 KB boxes (stages deep) from a per-SM L2-resident
// region; warps 1..W: cp.async 16 B per lane into their own smem area from
// another per-SM region, `depth` groups in flight.  mode bit 0: TMA on, bit 1:
// cp.async on.
__global__ void __launch_bounds__(288, 1)
    mix(const __grid_constant__ CUtensorMap map, const uint4* src, int mode, int iters,
        unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = align_smem_1024(raw);
  constexpr int stages = 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    stop = 0;
  }
  __syncthreads();
  unsigned long long cp_bytes = 0;
  const long long t0 = clock64();
  if (warp == 0) {
    if ((mode & 1) && lane == 0) {
      for (int i = 0; i < iters; ++i) {
        const int s = i % stages;
        if (i >= stages) mbar_wait(&full[s], ((i / stages) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], 16384);
        tma_load_2d(smem + s * 16384, &map, &full[s], 0, (blockIdx.x * 32 + i % 32) * 128, 0);
      }
      for (int s = 0; s < stages; ++s) mbar_wait(&full[(iters - stages + s) % stages], ((iters - stages + s) / stages) & 1);
    }
    __syncwarp();
    if (lane == 0) stop = 1;
    if (!(mode & 1)) {
      for (volatile int d = 0; d < 1; ++d) {
      }
    }
  } else if (mode & 2) {
    const uint4* base = src + (size_t(blockIdx.x) * 8 + (warp - 1)) * 32 * 64;  // 32 KB per warp
    uint8_t* dst = smem + 128 * 1024 + (warp - 1) * 8192;
    long long it = 0;
    while (!stop || !(mode & 1)) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint4* g = base + ((it * 8 + u) % 64) * 32 + lane;
        const uint32_t d = smem_u32(dst + ((u * 32 + lane) % 512) * 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(g) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 4;" ::: "memory");
      cp_bytes += 8 * 16 * 32;
      ++it;
      if (!(mode & 1) && it >= iters * 4) break;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  const long long t1 = clock64();
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  if (blockIdx.x == 0 && warp == 1 && lane == 0) out[1] = cp_bytes;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = size_t(256) << 20;
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  CUtensorMap map;
  es::make_bf16_map(&map, buf, 64, bytes / 128, 128);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(mix, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  const char* nm[4] = {"", "TMA only", "cp.async only (8 warps)", "TMA + cp.async"};
  for (int mode = 1; mode < 4; ++mode) {
    const int iters = 4096;
    cudaMemset(d, 0, 16);
    mix<<<sms, 288, 210 * 1024>>>(map, static_cast<const uint4*>(buf) + (64 << 20) / 16, mode, iters, d);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double tma = (mode & 1) ? double(iters) * 16384 : 0;
    const double cp = double(h[1]) * 8;  // 8 cp.async warps, warp 1 counted
    std::printf("%-26s %8llu clk: TMA %.1f B/clk, cp.async %.1f B/clk, total %.1f B/clk/SM %s\n", nm[mode],
                h[0], tma / h[0], cp / h[0], (tma + cp) / h[0], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
