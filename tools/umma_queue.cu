// Design evidence, not product: how many tcgen05.mma (N = 160, A from TMEM)
// one thread can issue before the issue blocks (tensor-pipe queue depth), and
// what a gap of G clk between two bursts costs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I../paper_2208_14049_b200/csrc \
//        umma_queue.cu -o umma_queue
#include <cuda_runtime.h>

#include <cstdio>

#include "cuda/sm100.cuh"

using namespace es::sm100;

__global__ void __launch_bounds__(128, 1) run(int k, int gap, unsigned long long* out) {
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
  if (threadIdx.x == 0) {
    const uint64_t bd = sdesc_planar(smem_u32(smem + 32 * 1024), 160 * 16);
    const uint32_t id = idesc_bf16_f32(128, 160);
    const long long t0 = clock64();
    for (int r = 0; r < k; ++r) umma_bf16_ta(tmem, tmem + 448u, bd, id, 1u);
    const long long t1 = clock64();  // issue of the first burst done
    const long long tg = t1 + gap;
    while (clock64() < tg) {
    }
    for (int r = 0; r < k; ++r) umma_bf16_ta(tmem, tmem + 448u, bd, id, 1u);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  for (int k : {1, 2, 4, 8, 16, 32})
    for (int gap : {0, 200, 400, 800}) {
      run<<<148, 128, 110 * 1024>>>(k, gap, d);
      unsigned long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      std::printf("burst %2d x N=160, gap %4d: first burst issued in %5llu clk; both bursts done at %6llu "
                  "(pipe-only %5d + gap) %s\n",
                  k, gap, h[0], h[1], 2 * k * 80, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
