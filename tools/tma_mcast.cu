// Design evidence, not product: is the ~48 B/clk per-SM TMA ingress
// (tools/tma_bw.cu) a limit on the bytes an SM RECEIVES or on the loads it
// ISSUES?  Clusters of 2 CTAs; mode 0: each CTA loads every box itself;
// mode 1: each CTA issues half the boxes with .multicast::cluster to both.
// Both modes deliver the same bytes to every SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2208_14049_b200/csrc \
//        tma_mcast.cu -o tma_mcast
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "cuda/sm100.cuh"
#include "cuda/tma_host.hpp"

using namespace es::sm100;

constexpr int kStages = 8;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1)
    run(const __grid_constant__ CUtensorMap map, int mode, int iters, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = align_smem_1024(raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * 16384);
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  cluster_sync();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % kStages;
      if (i >= kStages) mbar_wait(&full[s], ((i / kStages) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], 16384);
      const int tile = (blockIdx.x / 2) * 32 + i % 32;
      if (mode == 0) {
        tma_load_2d(smem + s * 16384, &map, &full[s], 0, tile * 128, 0);
      } else if ((i & 1) == static_cast<int>(rank)) {  // this CTA issues every other box, to both
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
            " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem + s * 16384)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&full[s])), "r"(0), "r"(tile * 128),
            "h"(static_cast<uint16_t>(0b11))
            : "memory");
      }
    }
    for (int s = 0; s < kStages; ++s) {
      const int i = iters - kStages + s;
      mbar_wait(&full[i % kStages], (i / kStages) & 1);
    }
  }
  const long long t1 = clock64();
  cluster_sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
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
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  for (int mode = 0; mode < 2; ++mode) {
    const int iters = 4096;
    run<<<(sms / 2) * 2, 64, 140 * 1024>>>(map, mode, iters, d);
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    std::printf("%-34s %.1f B/clk received per SM %s\n",
                mode ? "half the boxes each, multicast" : "every box by each CTA",
                double(iters) * 16384 / c, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
