// Design evidence, not product: latency of tcgen05.ld / tcgen05.st (+ wait)
// issued by other warps while one thread streams UMMAs (A from TMEM or smem,
// N configurable) -- the conv sweep's epilogue and drain are such warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I../paper_2208_14049_b200/csrc \
//        tmem_latency.cu -o tmem_latency
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "cuda/sm100.cuh"

using namespace es::sm100;

// mode: 0 = no UMMA stream, 1 = A from TMEM, 2 = A from smem
__global__ void __launch_bounds__(256, 1) lat(int mode, int N, int reps, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    stop = 0;
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (mode && elect_one()) {
      const uint32_t idesc = idesc_bf16_f32(128, N);
      const uint64_t bd = sdesc_planar(smem_u32(smem + 64 * 1024), N * 16);
      const uint64_t ad = sdesc_k128(smem_u32(smem));
      for (int r = 0; r < reps; ++r) {
        if (mode == 1)
          umma_bf16_ta(tmem, tmem + 448u + 8u * (r & 3), bd, idesc, 1u);
        else
          umma_bf16(tmem, ad, bd, idesc, 1u);
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
    }
    __syncwarp();
    if (lane == 0) stop = 1;
  } else if (warp >= 4) {  // lanes quadrant warp & 3: ld / st latency samples
    const uint32_t lf = static_cast<uint32_t>((warp & 3) * 32) << 16;
    unsigned long long sld = 0, sst = 0, n = 0, mld = 0, mst = 0;
    uint32_t v[32];
    while (!stop && n < 4000) {
      const long long t0 = clock64();
      tmem_ld32_raw(tmem + lf + 384u, v);
      tmem_ld_wait();
      const long long t1 = clock64();
      tmem_st32(tmem + lf + 416u, v);
      tmem_st_wait();
      const long long t2 = clock64();
      sld += t1 - t0;
      sst += t2 - t1;
      mld = max(mld, (unsigned long long)(t1 - t0));
      mst = max(mst, (unsigned long long)(t2 - t1));
      ++n;
      for (int d = 0; d < 20; ++d) __nanosleep(32);
    }
    if (blockIdx.x == 0 && lane == 0 && warp == 4) {
      out[0] = n ? sld / n : 0;
      out[1] = n ? sst / n : 0;
      out[2] = mld;
      out[3] = mst;
      out[4] = n;
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 5 * 8);
  cudaFuncSetAttribute(lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int mode = 0; mode < 3; ++mode)
    for (int N : {64, 160, 256}) {
      if (mode == 0 && N != 64) continue;
      cudaMemset(d, 0, 40);
      lat<<<148, 256, 100 * 1024>>>(mode, N, 20000, d);
      unsigned long long h[5];
      cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
      std::printf("mode %d (%s) N=%3d: ld+wait avg %4llu clk (max %6llu), st+wait avg %4llu (max %6llu), %llu samples %s\n",
                  mode, mode == 0 ? "idle" : mode == 1 ? "UMMA A=tmem" : "UMMA A=smem", N, h[0], h[2],
                  h[1], h[3], h[4], cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
