// Design evidence, not product: timeline of CTA 0 of conv_rows_sm100 (clock64
// stamps, in SM clocks from the first stamp) plus whole-launch timing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I../paper_2208_14049_b200/csrc \
//        trace_rows.cu -o trace_rows -L../paper_2208_14049_b200 -lenserve_b200 \
//        -Xlinker -rpath,'$ORIGIN/../paper_2208_14049_b200'
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cuda/aux_kernels.cuh"
#include "cuda/conv_rows_kernel.cuh"

int main(int argc, char** argv) {
  const long long nb = argc > 1 ? std::atoll(argv[1]) : (1 << 20);
  const int grid_div = argc > 2 ? std::atoi(argv[2]) : 1;
  const int debug = argc > 3 ? std::atoi(argv[3]) : 0;
  const bool sweep = argc > 4 && std::atoi(argv[4]) != 0;  // conv_sweep_sm100
  const int S = 28, G = 7, c1 = 64, c2 = 32;
  __nv_bfloat16 *x, *w1, *w2, *y;
  float *b1, *b2;
  unsigned long long* trace;
  cudaMalloc(&x, nb * S * S * 2);
  cudaMalloc(&w1, size_t(c1) * 16 * 2);
  cudaMalloc(&w2, size_t(c2) * 9 * c1 * 2);
  cudaMalloc(&b1, c1 * 4);
  cudaMalloc(&b2, c2 * 4);
  cudaMalloc(&y, nb * G * G * c2 * 2);
  cudaMalloc(&trace, 16 * 256 * 8);
  es::generate_features_bf16(1, nb * S * S, x, 0);
  es::generate_dense_layer(7, 0, 16, c1, std::sqrt(6.0f / (16 + c1)), w1, b1, 0);
  es::generate_dense_layer(7, 1, 9 * c1, c2, std::sqrt(6.0f / (9 * c1 + c2)), w2, b2, 0);
  es::ConvRowsArgs a;
  a.row_begin = 0;
  a.row_end = nb;
  a.w1 = w1;
  a.w2 = w2;
  a.out = y;
  a.debug = debug;
  cudaDeviceSynchronize();
  cudaMemcpy(a.b1c, b1, c1 * sizeof(float), cudaMemcpyDeviceToHost);
  cudaMemcpy(a.b2c, b2, c2 * sizeof(float), cudaMemcpyDeviceToHost);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemset(trace, 0, 16 * 256 * 8);
    a.trace = rep == 3 ? trace : nullptr;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int rc = sweep ? es::conv_sweep_launch(a, x, nb, sms / grid_div, 0)
                         : es::conv_rows_launch(a, x, nb, sms / grid_div, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tiles = double(nb) / 128 / (sms / grid_div);
    std::printf("rep %d rc %d: %.3f ms = %.3e samples/s, %.0f ns per tile per CTA (%s)\n", rep, rc, ms,
                nb / (ms * 1e-3), ms * 1e6 / tiles, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<unsigned long long> t(16 * 256);
  cudaMemcpy(t.data(), trace, t.size() * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull;
  for (auto v : t)
    if (v && v < t0) t0 = v;
  auto r = [&](int k, int i) { return t[k * 256 + i] ? (long long)(t[k * 256 + i] - t0) : -1ll; };
  std::printf("pos   tma  c1_a1  c1_iss  epi_c1  epi_a2e  epi_done c1_issued\n");
  for (int n = 0; n < 130; ++n)
    std::printf("%3d %7lld %7lld %7lld %7lld %7lld %7lld %7lld %7lld\n", n, r(0, n), r(1, n), r(2, n), r(3, n),
                r(4, n), r(5, n), r(12, n), r(15, n));
  std::printf("win  start  done  waited  issued\n");
  for (int w = 0; w < 130; ++w) std::printf("%3d %7lld %7lld %7lld %7lld\n", w, r(6, w), r(13, w), r(7, w), r(8, w));
  std::printf("feed-block  pos  start  a1_ok  c1e_ok\n");
  for (int n = 0; n < 130; ++n)
    if (r(11, n) >= 0) std::printf("%3d %7lld %7lld %7lld\n", n, r(11, n), r(12, n), r(13, n));
  std::printf("blk  o_full  released  stored\n");
  for (int b = 0; b < 256; ++b) std::printf("%3d %7lld %7lld %7lld\n", b, r(9, b), r(10, b), r(11, b));
  return 0;
}
