// Design evidence, not product: timeline of CTA 0 of the CNN convolution-stack
// kernel (globaltimer, microseconds from the first stamp).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I../paper_2208_14049_b200/csrc \
//        trace_conv.cu -o trace_conv -L../paper_2208_14049_b200 -lenserve_b200 \
//        -Xlinker -rpath,'$ORIGIN/../paper_2208_14049_b200'
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cuda/aux_kernels.cuh"
#include "cuda/conv_kernel.cuh"

// SM clock while the GPU is busy: clock64 vs globaltimer over ~2 ms of spinning.
__global__ void clock_probe(double* mhz) {
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const long long c0 = clock64();
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  } while (g1 - g0 < 2000000ull);
  const long long c1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *mhz = double(c1 - c0) / double(g1 - g0) * 1e3;
}

int main(int argc, char** argv) {
  const int c1 = argc > 1 ? std::atoi(argv[1]) : 64;
  const int c2 = argc > 2 ? std::atoi(argv[2]) : 32;
  const int sched = argc > 3 ? std::atoi(argv[3]) : 0;  // conv_plan schedule
  const int debug = argc > 4 ? std::atoi(argv[4]) : 0;  // ConvArgs::debug bits
  const int shifts = argc > 5 ? std::atoi(argv[5]) : -1;  // ConvArgs::shifts (-1 = default)
  const int grid_div = argc > 6 ? std::atoi(argv[6]) : 1;  // run on sms / grid_div CTAs
  const long long nb = 1 << 20;
  const int S = 28, P = 4, G = 7;
  __nv_bfloat16 *x, *w1, *w2, *y;
  float *b1, *b2;
  unsigned long long* trace;
  cudaMalloc(&x, nb * S * S * 2);
  cudaMalloc(&w1, size_t(c1) * 16 * 2);
  cudaMalloc(&w2, size_t(c2) * 9 * c1 * 2);
  cudaMalloc(&b1, c1 * 4);
  cudaMalloc(&b2, c2 * 4);
  cudaMalloc(&y, nb * G * G * c2 * 2);
  cudaMalloc(&trace, 32 * 16 * 8);
  es::generate_features_bf16(1, nb * S * S, x, 0);
  es::generate_dense_layer(7, 0, 16, c1, std::sqrt(6.0f / (16 + c1)), w1, b1, 0);
  es::generate_dense_layer(7, 1, 9 * c1, c2, std::sqrt(6.0f / (9 * c1 + c2)), w2, b2, 0);
  es::ConvArgs a;
  if (!es::conv_plan(S, P, c1, c2, &a.L, sched)) {
    std::printf("no plan\n");
    return 1;
  }
  std::printf("c1=%d c2=%d %s T=%d mb1=%d mb2=%d smem=%u tmem=%d\n", c1, c2,
              a.L.split ? "split" : "tap", a.L.T, a.L.mb1, a.L.mb2, a.L.smem_bytes, a.L.tmem_cols);
  a.debug = debug;
  a.row_begin = 0;
  a.row_end = nb;
  a.w1 = w1;
  a.b1 = b1;
  a.w2 = w2;
  a.b2 = b2;
  if (shifts >= 0) a.shifts = shifts;
  cudaDeviceSynchronize();
  cudaMemcpy(a.b2c, b2, c2 * sizeof(float), cudaMemcpyDeviceToHost);
  a.out = y;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(trace, 0, 32 * 16 * 8);
    a.trace = rep == 2 ? trace : nullptr;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    es::conv_launch(a, x, nb, sms / grid_div, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("rep %d: %.3f ms = %.3e samples/s (%s)\n", rep, ms, nb / (ms * 1e-3),
                cudaGetErrorString(cudaGetLastError()));
  }
  {
    double* mhz;
    cudaMalloc(&mhz, 8);
    clock_probe<<<148, 128>>>(mhz);
    double h = 0;
    cudaMemcpy(&h, mhz, 8, cudaMemcpyDeviceToHost);
    std::printf("SM clock right after: %.0f MHz\n", h);
  }
  std::vector<unsigned long long> t(32 * 16);
  cudaMemcpy(t.data(), trace, t.size() * 8, cudaMemcpyDeviceToHost);
  const unsigned long long t0 = t[0];
  std::printf("tile  tma  build_go build_end  c1_go  epi1_go epi1_end  c2_go  c2_iss  epi2_go epi2_end\n");
  for (int k = 0; k < 32; ++k) {
    auto r = [&](int i) { return t[k * 16 + i] ? double(t[k * 16 + i] - t0) / 1e3 : -1.0; };
    std::printf("%4d %6.2f %8.2f %9.2f %6.2f %8.2f %8.2f %6.2f %7.2f %8.2f %8.2f", k, r(0), r(4),
                r(5), r(1), r(6), r(7), r(2), r(3), r(8), r(9));
    for (int i = 10; i < 16; ++i) std::printf(" %7.2f", r(i));
    std::printf("\n");
  }
  return 0;
}
