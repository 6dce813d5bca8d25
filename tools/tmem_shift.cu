// Design evidence, not product: semantics and issue rate of tcgen05.shift
// (TMEM rows shifted down by one lane), measured on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_2208_14049_b200/csrc \
//        tmem_shift.cu -o tmem_shift
#include <cuda_runtime.h>

#include <cstdio>

#include "cuda/sm100.cuh"

using namespace es::sm100;

__device__ __forceinline__ void tmem_shift_down(uint32_t taddr) {
  asm volatile("tcgen05.shift.cta_group::1.down [%0];" ::"r"(taddr) : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// mode 0: one shift at column col0, dump [128][32]; mode 1: time `reps` shifts.
__global__ void __launch_bounds__(128, 1) shift_test(int mode, int col0, int reps, float* dump,
                                                     unsigned long long* clk) {
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lf = static_cast<uint32_t>(warp * 32) << 16;
  uint32_t v[32];
  for (int c = 0; c < 32; ++c) v[c] = __float_as_uint(static_cast<float>((warp * 32 + lane) * 100 + c));
  tmem_st32(tmem + lf, v);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    const long long t0 = clock64();
    const int n = mode == 0 ? 1 : reps;
    for (int i = 0; i < n; ++i)
      if (elect_one()) tmem_shift_down(tmem + static_cast<uint32_t>(col0 + (mode == 2 ? (i & 3) * 8 : 0)));
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0 && lane == 0) clk[0] = static_cast<unsigned long long>(clock64() - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  tmem_ld32_raw(tmem + lf, v);
  tmem_ld_wait();
  if (blockIdx.x == 0)
    for (int c = 0; c < 32; ++c) dump[(warp * 32 + lane) * 32 + c] = __uint_as_float(v[c]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 64);
}

int main() {
  float* d;
  unsigned long long* c;
  cudaMalloc(&d, 128 * 32 * 4);
  cudaMalloc(&c, 8);
  float h[128 * 32];
  shift_test<<<1, 128>>>(0, 0, 1, d, c);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  std::printf("one shift.down at column 0 (%s): value = 100*source_lane + column\n",
              cudaGetErrorString(cudaGetLastError()));
  for (int r : {0, 1, 2, 31, 32, 33, 64, 126, 127}) {
    std::printf("lane %3d:", r);
    for (int col = 0; col < 12; ++col) std::printf(" %6.0f", h[r * 32 + col]);
    std::printf("\n");
  }
  for (int mode = 1; mode <= 2; ++mode)
    for (int reps : {64, 512}) {
      shift_test<<<148, 128>>>(mode, 0, reps, d, c);
      unsigned long long k = 0;
      cudaMemcpy(&k, c, 8, cudaMemcpyDeviceToHost);
      std::printf("%s %d shifts: %.1f clk/shift (%s)\n", mode == 1 ? "same-col" : "4 col-blocks",
                  reps, double(k) / reps, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
