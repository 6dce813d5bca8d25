// Design evidence, not product: UMMA stream rate (N = 160 + 128, A from TMEM,
// the conv sweep's interior pattern) while 4 other warps run one kind of
// background traffic, to find what slows the tensor pipe inside the sweep.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I../paper_2208_14049_b200/csrc \
//        umma_load.cu -o umma_load
#include <cuda_runtime.h>

#include <cstdio>

#include "cuda/sm100.cuh"

using namespace es::sm100;

// load: 0 none, 1 tcgen05.st (other columns), 2 tcgen05.ld, 3 STS, 4 LDS, 5 LDG (L2),
// 6 mbarrier try_wait spin on a never-completing barrier, 7 STG, 8 TMA-free smem+fence.proxy
__global__ void __launch_bounds__(256, 1) run(int load, int reps, const uint4* gsrc, uint4* gdst,
                                               unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar, never;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&never, 1);
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
    if (elect_one()) {
      const uint64_t bd = sdesc_planar(smem_u32(smem + 96 * 1024), 288 * 16);
      const long long t0 = clock64();
      for (int r = 0; r < reps; ++r) {
        const uint32_t a = tmem + 448u + 8u * (r & 3);
        // load 19/20: each group of 4 pairs is one "input" whose D window slides
        // by 96 columns (partial overlap with the previous input, as in the conv
        // sweep) / or the previous window is disjoint (20: slide by 288)
        const uint32_t d0 = load == 19 ? 96u * ((r >> 2) % 2) : load == 20 ? 0u : 0u;
        umma_bf16_ta(tmem + d0, a, bd, idesc_bf16_f32(128, 160), 1u);
        umma_bf16_ta(tmem + d0 + 160u, a, bd + 160u, idesc_bf16_f32(128, 128), 1u);
        if (load == 9 && (r & 3) == 3) umma_commit(&never);        // a commit per 4 pairs
        if (load == 16 && (r & 3) == 3) tc_fence_after();          // tcgen05.fence::after_thread_sync per 4 pairs
        if (load == 17 && (r & 3) == 3) tc_fence_before();         // tcgen05.fence::before_thread_sync per 4 pairs
        if (load == 18 && (r & 3) == 3) {                          // a satisfied try_wait + fence, as per input
          mbar_try_wait(&bar, 1u);
          tc_fence_after();
        }
        if (load == 10 && (r & 3) == 3) {                          // + conv1-like UMMA
          umma_bf16(tmem + 384u, sdesc_planar(smem_u32(smem), 2048), sdesc_planar(smem_u32(smem + 8192), 1024),
                    idesc_bf16_f32(128, 64), 0u);
          umma_commit(&never);
        }
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      if (blockIdx.x == 0) out[0] = static_cast<unsigned long long>(clock64() - t0);
    }
    __syncwarp();
    if (lane == 0) stop = 1;
  } else if (warp == 1 && load == 11) {  // a second warp issuing conv1-like UMMAs + commits
    while (!stop) {
      if (elect_one()) {
        umma_bf16(tmem + 384u, sdesc_planar(smem_u32(smem), 2048), sdesc_planar(smem_u32(smem + 8192), 1024),
                  idesc_bf16_f32(128, 64), 0u);
        umma_commit(&never);
      }
      __syncwarp();
      for (int d = 0; d < 10; ++d) __nanosleep(50);
    }
  } else if (warp >= 4) {
    const uint32_t lf = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = i;
    uint8_t* my = smem + (warp - 4) * 8192;
    uint4 acc = make_uint4(0, 0, 0, 0);
    long long it = 0;
    while (!stop) {
      ++it;
      if (load == 1) {
        tmem_st32(tmem + lf + 384u, v);
        tmem_st_wait();
      } else if (load == 2) {
        tmem_ld32_raw(tmem + lf + 384u, v);
        tmem_ld_wait();
      } else if (load == 3) {
#pragma unroll
        for (int c = 0; c < 4; ++c) reinterpret_cast<uint4*>(my + lane * 64)[c] = make_uint4(it, c, 0, 0);
      } else if (load == 4) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc.x += reinterpret_cast<volatile uint32_t*>(my + lane * 64)[4 * c];
        }
      } else if (load == 5) {
        const uint4* p = gsrc + ((blockIdx.x * 4 + (warp - 4)) * 32 + lane) * 196 + (it % 98) * 2;
        uint4 q = __ldg(p);
        acc.x += q.x;
      } else if (load == 6) {
        mbar_try_wait(&never, 0);
      } else if (load == 7) {
        gdst[((blockIdx.x * 4 + (warp - 4)) * 32 + lane) * 196 + (it % 196)] = make_uint4(it, 0, 0, 0);
      } else if (load >= 12 && load <= 15) {
        // 12/13: ld / st inside the UMMAs' D columns; 14/15: just outside them
        const uint32_t col = load < 14 ? 64u : 320u;
        if (load & 1) {
          tmem_st32(tmem + lf + col, v);
          tmem_st_wait();
        } else {
          tmem_ld32_raw(tmem + lf + col, v);
          tmem_ld_wait();
        }
        for (int d = 0; d < 4; ++d) __nanosleep(100);
      } else if (load == 8) {
#pragma unroll
        for (int c = 0; c < 4; ++c) reinterpret_cast<uint4*>(my + lane * 64)[c] = make_uint4(it, c, 0, 0);
        fence_proxy_async_smem();
        __syncwarp();
      }
    }
    if (acc.x == 12345) out[1] = acc.x + v[3];
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  uint4 *gs, *gd;
  const size_t n = size_t(148) * 128 * 196;
  cudaMalloc(&gs, n * 16);
  cudaMalloc(&gd, n * 16);
  cudaMemset(gs, 0, n * 16);
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  const char* names[] = {"none", "tcgen05.st", "tcgen05.ld", "STS", "LDS", "LDG", "try_wait spin", "STG",
                         "STS+fence.proxy.async", "commit per 4 pairs", "conv1 UMMA+commit per 4",
                         "2nd warp conv1 UMMAs", "ld in D cols (paced)", "st in D cols (paced)",
                         "ld outside D (paced)", "st outside D (paced)", "fence::after per 4 pairs",
                         "fence::before per 4 pairs", "try_wait + fence per 4 pairs",
                         "D slides by 96 per 4 pairs"};
  for (int load = 0; load < 20; ++load) {
    run<<<148, 256, 170 * 1024>>>(load, 4000, gs, gd, d);
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    std::printf("%-24s %6.1f clk per N=160+128 pair (pipe-only ideal 144) %s\n", names[load], double(c) / 4000,
                cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
