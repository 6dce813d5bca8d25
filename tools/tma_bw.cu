// Microbenchmark (design evidence, not product): how many bytes per cycle can
// one SM ingest through TMA from L2 / HBM, as a function of pipeline depth and
// of whether all SMs read the same tiles (weights) or distinct tiles (samples)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2208_14049_b200/csrc \
//        tma_bw.cu -o tma_bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cuda/sm100.cuh"

using namespace es::sm100;

constexpr int kTileRows = 128;  // 128 rows x 128 B = 16 KB per TMA box

__global__ void __launch_bounds__(64, 1)
    tma_stream(const __grid_constant__ CUtensorMap map, int stages, int iters, int mode,
               int region_tiles, unsigned long long* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~1023ull);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * 16384);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const uint64_t pol = l2_policy_evict_last();
  if (threadIdx.x == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&empty[stage], phase ^ 1u);
      mbar_arrive_expect_tx(&full[stage], 16384);
      int tile;
      if (mode == 0) tile = i % region_tiles;                                  // shared by all SMs
      else if (mode == 1) tile = blockIdx.x * region_tiles + i % region_tiles; // per-SM, L2 resident
      else tile = (blockIdx.x + i * gridDim.x) % region_tiles;                 // streaming
      tma_load_2d(smem + stage * 16384, &map, &full[stage], 0, tile * kTileRows, pol);
      if (++stage == stages) {
        stage = 0;
        phase ^= 1u;
      }
    }
  } else if (threadIdx.x == 32) {
    int stage = 0;
    uint32_t phase = 0;
    unsigned long long acc = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[stage], phase);
      acc += smem[stage * 16384 + (i & 127)];
      mbar_arrive(&empty[stage]);
      if (++stage == stages) {
        stage = 0;
        phase ^= 1u;
      }
    }
    if (acc == 0x12345) *sink = acc;
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (argc > 1) sms = std::atoi(argv[1]);  // fewer CTAs: per-SM vs aggregate limit
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const size_t bytes = size_t(8) << 30;  // 8 GiB
  void* buf = nullptr;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {64, bytes / 128};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, kTileRows};
  cuuint32_t es_[2] = {1, 1};
  reinterpret_cast<EncodeFn>(fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box,
                                 es_, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[3] = {"shared (all SMs same 1 MiB)", "per-SM 512 KiB (L2 resident)",
                          "streaming 8 GiB (HBM)"};
  printf("SMs %d, clock %.0f MHz\n", sms, clk_khz / 1e3);
  for (int mode = 0; mode < 3; ++mode) {
    int region = mode == 0 ? 64 : mode == 1 ? 32 : int(bytes / 16384);
    for (int stages : {2, 4, 6, 8, 12}) {
      int iters = 4096;
      size_t smem = stages * 16384 + 2 * stages * 8 + 1024;
      tma_stream<<<sms, 64, smem>>>(map, stages, 256, mode, region, sink);  // warm
      cudaEventRecord(a);
      tma_stream<<<sms, 64, smem>>>(map, stages, iters, mode, region, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      double tot = double(sms) * iters * 16384;
      double gbs = tot / (ms * 1e-3) / 1e9;
      printf("%-32s stages %2d  %8.1f GB/s  %6.1f B/clk/SM (at max clock)\n", names[mode], stages,
             gbs, gbs * 1e9 / sms / (clk_khz * 1e3));
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
