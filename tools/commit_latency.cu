// Design evidence, not product: time from issuing k UMMAs (N = 160, A from
// TMEM) + tcgen05.commit to the issuing thread observing the mbarrier phase.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I../paper_2208_14049_b200/csrc \
//        commit_latency.cu -o commit_latency
#include <cuda_runtime.h>

#include <cstdio>

#include "cuda/sm100.cuh"

using namespace es::sm100;

__global__ void __launch_bounds__(128, 1) run(int k, int N, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 100 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    unsigned long long tot = 0;
    uint32_t par = 0;
    for (int rep = 0; rep < 64; ++rep) {
      const long long t0 = clock64();
      if (elect_one()) {
        const uint64_t bd = sdesc_planar(smem_u32(smem + 32 * 1024), N * 16);
        for (int r = 0; r < k; ++r) umma_bf16_ta(tmem, tmem + 448u, bd, idesc_bf16_f32(128, N), 1u);
        umma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, par);
      par ^= 1u;
      const long long t1 = clock64();
      if (rep >= 8) tot += t1 - t0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = tot / 56;
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  for (int N : {64, 160})
    for (int k : {1, 2, 4, 8, 16}) {
      run<<<148, 128, 110 * 1024>>>(k, N, d);
      unsigned long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      std::printf("N=%3d k=%2d UMMAs + commit -> phase observed: %5llu clk (%5.1f per UMMA) %s\n", N, k, c,
                  double(c) / k, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
