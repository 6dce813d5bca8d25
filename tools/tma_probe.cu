// Design evidence, not product: TMA tile loads of [128 rows][8 bf16] boxes at
// arbitrary (unaligned) column offsets -- the conv_rows conv1 operand planes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_2208_14049_b200/csrc tma_probe.cu -o tma_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "cuda/sm100.cuh"
#include "cuda/tma_host.hpp"
using namespace es::sm100;

__global__ void probe(const __grid_constant__ CUtensorMap tm, int x, int y, int mode, uint16_t* out) {
  __shared__ alignas(1024) uint8_t buf[2048];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t pol = mode ? l2_policy_evict_first() : l2_policy_evict_normal();
    mbar_arrive_expect_tx(&bar, 2048);
    tma_load_2d(buf, &tm, &bar, x, y, pol);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(buf)[i];
}

int main() {
  const int rows = 300, W = 784;
  std::vector<uint16_t> h(rows * W);
  for (int r = 0; r < rows; ++r) for (int c = 0; c < W; ++c) h[r * W + c] = static_cast<uint16_t>(r * 7 + c);
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&o, 2048);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(W * 2)};
  cuuint32_t box[2] = {8, 128};
  cuuint32_t estr[2] = {1, 1};
  for (int prom = 0; prom < 2; ++prom) {
    CUresult r = es::encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, estr,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode promotion=%d: %d\n", prom, static_cast<int>(r));
    for (int mode = 0; mode < 2; ++mode)
      for (int x : {0, 4, 12, 28, 776}) {
        probe<<<1, 128>>>(m, x, 5, mode, o);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("prom %d mode %d x %d: %s\n", prom, mode, x, cudaGetErrorString(e)); return 1; }
        std::vector<uint16_t> g(1024);
        cudaMemcpy(g.data(), o, 2048, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int rr = 0; rr < 128; ++rr) for (int c = 0; c < 8; ++c) {
          const int R = 5 + rr, C = x + c;
          const uint16_t want = (R < rows && C < W) ? static_cast<uint16_t>(R * 7 + C) : 0;
          if (g[rr * 8 + c] != want) ++bad;
        }
        printf("prom %d mode %d x %3d: %d bad\n", prom, mode, x, bad);
      }
  }
  return 0;
}
