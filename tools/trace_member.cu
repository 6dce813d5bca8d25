// Design evidence, not product: timeline of CTA 0 of the SM-pair member kernel
// (globaltimer ns) to see where a tile's time goes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I../paper_2208_14049_b200/csrc \
//        trace_member.cu -o trace_member -L../paper_2208_14049_b200 -lenserve_b200 \
//        -Xlinker -rpath,'$ORIGIN/../paper_2208_14049_b200'
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cuda/aux_kernels.cuh"
#include "cuda/mlp_pair_kernel.cuh"

int main(int argc, char** argv) {
  const int H = argc > 1 ? std::atoi(argv[1]) : 512;
  const int grid_div = argc > 2 ? std::atoi(argv[2]) : 1;  // fewer SMs: per-SM vs aggregate limits
  const long long nb = 1 << 22;
  const int K = 784, C = 10, b = 128;
  __nv_bfloat16 *x, *w1, *w2;
  float *b1, *b2, *out;
  unsigned long long* trace;
  cudaMalloc(&x, nb * K * 2);
  cudaMalloc(&w1, size_t(H) * K * 2);
  cudaMalloc(&w2, size_t(C) * H * 2);
  cudaMalloc(&b1, H * 4);
  cudaMalloc(&b2, C * 4);
  cudaMalloc(&out, nb * C * 4);
  cudaMalloc(&trace, 32 * 16 * 8);
  es::generate_features_bf16(1, nb * K, x, 0);
  es::generate_dense_layer(7, 0, K, H, std::sqrt(6.0f / (K + H)), w1, b1, 0);
  es::generate_dense_layer(7, 1, H, C, std::sqrt(6.0f / (H + C)), w2, b2, 0);
  es::MlpPArgs a;
  if (!es::mlpp_plan(K, H, C, b, &a.L)) {
    std::printf("no plan\n");
    return 1;
  }
  std::printf("H=%d T=%d nbuf=%d stages=%d d2_sep=%d NH=%d\n", H, a.L.T, a.L.nbuf, a.L.stages,
              a.L.d2_sep, a.L.NH);
  a.b = b;
  a.seg_size = 128;
  a.seg_begin = 0;
  a.seg_end = nb / 128;
  a.nb = nb;
  a.bias1 = b1;
  a.bias2 = b2;
  a.out = out;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(trace, 0, 32 * 16 * 8);
    a.trace = rep == 2 ? trace : nullptr;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    es::mlpp_launch(a, x, w1, w2, sms / grid_div, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("rep %d: %.3f ms = %.1f TFLOP/s per SM-share (grid %d) (%s)\n", rep, ms,
                2.0 * nb * (double(K) * H + double(H) * C) / (ms * 1e-3) / 1e12 * grid_div, sms / grid_div,
                cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<unsigned long long> t(32 * 16);
  cudaMemcpy(t.data(), trace, t.size() * 8, cudaMemcpyDeviceToHost);
  const unsigned long long t0 = t[0];
  std::printf("grp  prod_kc0 mma_wait mma_go mma_issued epi_acc bf16_w2 bf16_w9 mma_afull mma2_iss epi_acc2 logits\n");
  for (int g = 0; g < 32; ++g) {
    auto r = [&](int i) { return t[g * 16 + i] ? double(t[g * 16 + i] - t0) / 1e3 : -1.0; };
    std::printf("%3d %9.2f %8.2f %6.2f %10.2f %7.2f %7.2f %7.2f %9.2f %8.2f %8.2f %6.2f\n", g, r(7),
                r(0), r(1), r(2), r(3), r(4), r(10), r(8), r(9), r(5), r(6));
  }
  return 0;
}
