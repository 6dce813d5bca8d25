// Design evidence, not product: three hardware questions behind the
// samples-in-M conv stack (conv_rows_kernel.cu), measured on B200.
//   1. overlap: UMMAs accumulating into OVERLAPPING TMEM column windows
//      (D = O + (iw-1)*32, N = 96) give the exact sum (small-integer operands,
//      so fp32 sums are exact) -- and at what rate, against the same UMMAs
//      into one D;
//   2. ld: tcgen05.ld 32x32b.x32 throughput per SM with 4 / 8 / 16 warps;
//   3. ta: N = 96 UMMA rate with A from TMEM vs A from shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_2208_14049_b200/csrc \
//        conv_probe.cu -o conv_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cuda/sm100.cuh"

using namespace es::sm100;


// Operands: 7 windows, A_iw [128][16] and B_iw [96][16] bf16 in the planar
// K-major layout (2 planes of [rows][16 B]).
constexpr int kW = 7;
constexpr uint32_t kAPlane = 128 * 16, kABytes = 2 * kAPlane;
constexpr uint32_t kBPlane = 96 * 16, kBBytes = 2 * kBPlane;
constexpr uint32_t kSmem = kW * (kABytes + kBBytes) + 1024;

// mode 0: sliding windows (N = 64/96.../64 at (iw-1)*32, clipped); mode 1: the
// same UMMAs all into columns [0, N); mode 2: mode 0 with A from TMEM (A_iw
// copied to TMEM columns 256 + 8*iw).  reps > 1: timing; reps == 1: dump D.
template <int mode>
__global__ void __launch_bounds__(128, 1)
    overlap_test(const uint16_t* gA, const uint16_t* gB, int reps, int inner, float* dump,
                 unsigned long long* clk) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = align_smem_1024(raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kW * 128 * 2; i += 128) {  // A: [iw][plane][row][16 B]
    const int iw = i / 256, rem = i % 256, row = rem / 2, pl = rem % 2;
    *reinterpret_cast<uint4*>(sm + iw * kABytes + pl * kAPlane + row * 16) =
        *reinterpret_cast<const uint4*>(gA + (iw * 128 + row) * 16 + pl * 8);
  }
  uint8_t* sB = sm + kW * kABytes;
  for (int i = threadIdx.x; i < kW * 96 * 2; i += 128) {
    const int iw = i / 192, rem = i % 192, row = rem / 2, pl = rem % 2;
    *reinterpret_cast<uint4*>(sB + iw * kBBytes + pl * kBPlane + row * 16) =
        *reinterpret_cast<const uint4*>(gB + (iw * 96 + row) * 16 + pl * 8);
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lf = static_cast<uint32_t>(warp * 32) << 16;
  {
    uint32_t z[32];
    for (int c = 0; c < 32; ++c) z[c] = 0;
    for (int c = 0; c < 256; c += 32) tmem_st32(tmem + lf + c, z);
    if (mode == 2) {  // A_iw -> TMEM: lane = row, 8 columns of bf16 pairs
      for (int iw = 0; iw < kW; ++iw) {
        uint32_t v[32];
        const int row = warp * 32 + lane;
        for (int c = 0; c < 8; ++c) v[c] = reinterpret_cast<const uint32_t*>(gA + (iw * 128 + row) * 16)[c];
        for (int c = 8; c < 32; ++c) v[c] = 0;
        tmem_st32(tmem + lf + 256 + 32 * iw, v);
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    const uint32_t a0 = __shfl_sync(0xffffffffu, smem_u32(sm), 0);
    const uint32_t b0 = __shfl_sync(0xffffffffu, smem_u32(sB), 0);
    const uint32_t id96 = idesc_bf16_f32(128, 96), id64 = idesc_bf16_f32(128, 64);
    const uint64_t ad0 = sdesc_planar(a0, kAPlane), bd0 = sdesc_planar(b0, kBPlane);
    const uint32_t ta0 = __shfl_sync(0xffffffffu, tmem + 256u, 0), td0 = __shfl_sync(0xffffffffu, tmem, 0);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int iw = 0; iw < kW; ++iw) {
        // window iw covers output blocks iw-1..iw+1; B rows j*32.. map to block iw-1+j
        constexpr int dummy = 0;
        const int jlo = iw == 0 ? 1 : 0, jhi = iw == kW - 1 ? 2 : 3;
        const uint32_t id = (jhi - jlo) == 3 ? id96 : id64;
        const uint64_t bd = bd0 + static_cast<uint64_t>((iw * kBBytes + jlo * 32 * 16) >> 4);
        const uint64_t ad = ad0 + static_cast<uint64_t>((iw * kABytes) >> 4);
        const uint32_t dcol = mode == 1 ? 0u : static_cast<uint32_t>((iw - 1 + jlo) * 32);
#pragma unroll
        for (int i = 0; i < 12; ++i) {
          if constexpr (mode == 2) {
            if (elect_one()) umma_bf16_ta(td0 + dcol, ta0 + 32 * iw, bd, id, 1);
          } else {
            if (elect_one()) umma_bf16(td0 + dcol, ad, bd, id, 1);
          }
        }
        (void)dummy;
      }
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (lane == 0) clk[0] = static_cast<unsigned long long>(clock64() - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (reps == 1) {
    for (int c = 0; c < 224; c += 32) {
      uint32_t v[32];
      tmem_ld32_raw(tmem + lf + c, v);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) dump[(warp * 32 + lane) * 224 + c + j] = __uint_as_float(v[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

// tcgen05.ld throughput: every warp loads 32 columns x 32 lanes of its
// quadrant `reps` times (wait after each `batch` loads).
__global__ void ld_rate(int reps, int batch, int st, unsigned long long* clk, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  float acc = 0.f;
  const long long t0 = clock64();
  uint32_t v[32];
  for (int c = 0; c < 32; ++c) v[c] = c;
  for (int r = 0; r < reps; r += batch) {
    for (int b = 0; b < batch; ++b) {
      const uint32_t col = static_cast<uint32_t>(((r + b) * 32 + (warp >> 2) * 128) & 511);
      if (st) {
        tmem_st32(tmem + col, v);
      } else {
        tmem_ld32_raw(tmem + col, v);
      }
    }
    if (st) {
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else {
      tmem_ld_wait();
      for (int c = 0; c < 32; ++c) acc += __uint_as_float(v[c]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) clk[blockIdx.x] = static_cast<unsigned long long>(clock64() - t0);
  if (acc == 12345.f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 512);
}


// Fixed-N rate: 12 x 7 UMMAs per rep into one D, A from TMEM (TA = 1) or smem.
template <int N, int TA>
__global__ void __launch_bounds__(128, 1) fixed_rate(int reps, unsigned long long* clk) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = align_smem_1024(raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 49152 / 16; i += 128) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    const uint32_t td0 = __shfl_sync(0xffffffffu, slot, 0);
    const uint64_t ad = sdesc_planar(__shfl_sync(0xffffffffu, smem_u32(sm), 0), 2048);
    const uint64_t bd = sdesc_planar(__shfl_sync(0xffffffffu, smem_u32(sm + 4096), 0), 4096);
    const uint64_t ad128 = sdesc_k128(__shfl_sync(0xffffffffu, smem_u32(sm), 0));
    const uint64_t bd128 = sdesc_k128(__shfl_sync(0xffffffffu, smem_u32(sm + 16384), 0));
    constexpr uint32_t id = idesc_bf16_f32(128, N);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int i = 0; i < 84; ++i) {
        if constexpr (TA == 1) {
          if (elect_one()) umma_bf16_ta(td0, td0 + 256u + 8u * (i & 3), bd, id, 1);
        } else if constexpr (TA == 2) {  // A: K-major SW128 [128][64], K step = +32 B
          if (elect_one()) umma_bf16(td0, ad128 + 2u * (i & 3), bd, id, 1);
        } else if constexpr (TA == 3) {  // A SW128, B SW128 [N][64]
          if (elect_one()) umma_bf16(td0, ad128 + 2u * (i & 3), bd128 + 2u * (i & 3), id, 1);
        } else {
          if (elect_one()) umma_bf16(td0, ad + 2u * (i & 3), bd, id, 1);
        }
      }
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (lane == 0 && blockIdx.x == 0) clk[0] = static_cast<unsigned long long>(clock64() - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 512);
}

template <int N, int TA>
static void run_fixed(unsigned long long* clk) {
  cudaFuncSetAttribute(fixed_rate<N, TA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
  fixed_rate<N, TA><<<148, 128, 60000>>>(100, clk);
  cudaDeviceSynchronize();
  unsigned long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  printf("fixed N=%3d A from %s: %.1f clk/UMMA\n", N, TA == 1 ? "TMEM" : TA == 2 ? "smem SW128 (B planar)" : TA == 3 ? "smem SW128 (B SW128)" : "smem planar", double(c) / (100.0 * 84));
}

// Commit cost: 96 UMMAs (N = 96, A from TMEM) per rep, a tcgen05.commit to a
// dummy mbarrier after every `every` UMMAs (0 = none).
template <int EVERY>
__global__ void __launch_bounds__(128, 1) commit_rate(int reps, unsigned long long* clk) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = align_smem_1024(raw);
  __shared__ uint64_t bar, dummy;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 16384 / 16; i += 128) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&dummy, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    const uint32_t td0 = __shfl_sync(0xffffffffu, slot, 0);
    const uint64_t bd = sdesc_planar(__shfl_sync(0xffffffffu, smem_u32(sm + 4096), 0), 4096);
    constexpr uint32_t id = idesc_bf16_f32(128, 96);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int i = 0; i < 96; ++i) {
        if (elect_one()) umma_bf16_ta(td0, td0 + 256u + 8u * (i & 3), bd, id, 1);
        if constexpr (EVERY > 0)
          if ((i + 1) % EVERY == 0 && elect_one()) umma_commit(&dummy);
        if constexpr (EVERY < 0)
          if ((i + 1) % (-EVERY) == 0) tc_fence_after();
      }
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (lane == 0 && blockIdx.x == 0) clk[0] = static_cast<unsigned long long>(clock64() - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 512);
}

template <int EVERY>
static void run_commit(unsigned long long* clk) {
  cudaFuncSetAttribute(commit_rate<EVERY>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  commit_rate<EVERY><<<148, 128, 40000>>>(50, clk);
  cudaDeviceSynchronize();
  unsigned long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  printf("%s every %2d UMMAs (N=96, TMEM A): %.1f clk/UMMA\n", EVERY < 0 ? "fence::after_thread_sync" : "commit", EVERY < 0 ? -EVERY : EVERY, double(c) / (50.0 * 96));
}

// Mixed stream: per rep 12 TMEM-A N=64 then 12 smem-A (SW128) N=96 UMMAs
// (MODE bit 0), optionally with warps 1-3 + 4-7 streaming tcgen05.ld (bit 1)
// or tcgen05.st (bit 2) on other columns, and warps streaming STS (bit 3).
template <int MODE>
__global__ void __launch_bounds__(256, 1) mixed_rate(int reps, unsigned long long* clk) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = align_smem_1024(raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 16; i += 256) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    stop = 0;
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (warp == 0) {
    const uint32_t td0 = __shfl_sync(0xffffffffu, tm, 0);
    const uint64_t bd = sdesc_planar(__shfl_sync(0xffffffffu, smem_u32(sm + 16384), 0), 1536);
    const uint64_t ad128 = sdesc_k128(__shfl_sync(0xffffffffu, smem_u32(sm), 0));
    constexpr uint32_t id64 = idesc_bf16_f32(128, 64), id96 = idesc_bf16_f32(128, 96);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int i = 0; i < 12; ++i)
        if (elect_one()) umma_bf16_ta(td0 + 32u * (i & 1), td0 + 256u + 8u * (i & 3), bd, id64, 1);
      if constexpr (MODE & 1) {
#pragma unroll
        for (int i = 0; i < 12; ++i)
          if (elect_one()) umma_bf16(td0 + 32u * (i & 1), ad128 + 2u * (i & 3), bd, id96, 1);
      }
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (lane == 0 && blockIdx.x == 0) clk[0] = static_cast<unsigned long long>(clock64() - t0);
    if (lane == 0) stop = 1;
  } else if (warp >= 4) {
    const uint32_t lf = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = c;
    float acc = 0.f;
    while (!stop) {
      if constexpr (MODE & 2) {
        tmem_ld32_raw(tm + lf + 320u, v);
        tmem_ld32_raw(tm + lf + 352u, v);
        tmem_ld_wait();
        acc += __uint_as_float(v[3]);
      }
      if constexpr (MODE & 4) {
        tmem_st32(tm + lf + 384u, v);
        tmem_st_wait();
      }
      if constexpr (MODE & 8) {
        uint4* d = reinterpret_cast<uint4*>(sm + 40960 + (warp - 4) * 4096);
        for (int k = 0; k < 8; ++k) d[k * 32 + lane] = make_uint4(k, lane, 1, 2);
      }
      if constexpr (MODE < 2) break;
    }
    if (acc == 1234.f) clk[1] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

template <int MODE>
static void run_mixed(unsigned long long* clk) {
  cudaFuncSetAttribute(mixed_rate<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  mixed_rate<MODE><<<148, 256, 70000>>>(100, clk);
  cudaDeviceSynchronize();
  unsigned long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  const double ideal = (MODE & 1) ? 12 * 32 + 12 * 56 : 12 * 32;
  printf("mixed mode %2d (%s%s%s%s): %.0f clk per rep (isolated-rate sum %.0f)\n", MODE,
         (MODE & 1) ? "TMEM-A N64 + smem-A N96" : "TMEM-A N64 only", (MODE & 2) ? ", +tcgen05.ld" : "",
         (MODE & 4) ? ", +tcgen05.st" : "", (MODE & 8) ? ", +STS" : "", double(c) / 100.0, ideal);
}

static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return static_cast<uint16_t>(u >> 16);  // exact for small integers
}

int main() {
  std::vector<float> A(kW * 128 * 16), B(kW * 96 * 16);
  srand(1);
  for (auto& a : A) a = static_cast<float>(rand() % 5 - 2);
  for (auto& b : B) b = static_cast<float>(rand() % 5 - 2);
  std::vector<uint16_t> hA(A.size()), hB(B.size());
  for (size_t i = 0; i < A.size(); ++i) hA[i] = f2bf(A[i]);
  for (size_t i = 0; i < B.size(); ++i) hB[i] = f2bf(B[i]);
  uint16_t *dA, *dB;
  float *dump, *sink;
  unsigned long long* clk;
  cudaMalloc(&dA, hA.size() * 2);
  cudaMalloc(&dB, hB.size() * 2);
  cudaMalloc(&dump, 128 * 224 * 4);
  cudaMalloc(&sink, 4);
  cudaMalloc(&clk, 148 * 8);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(overlap_test<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  cudaFuncSetAttribute(overlap_test<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  cudaFuncSetAttribute(overlap_test<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  // expected D
  std::vector<double> E(128 * 224, 0.0);
  for (int iw = 0; iw < kW; ++iw)
    for (int j = 0; j < 3; ++j) {
      const int blk = iw - 1 + j;
      if (blk < 0 || blk >= kW) continue;
      for (int m = 0; m < 128; ++m)
        for (int c = 0; c < 32; ++c) {
          double s = 0;
          for (int k = 0; k < 16; ++k) s += A[(iw * 128 + m) * 16 + k] * B[(iw * 96 + j * 32 + c) * 16 + k];
          E[m * 224 + blk * 32 + c] += s;
        }
    }
  for (int mode : {0, 2}) {
    if (mode == 0) overlap_test<0><<<1, 128, kSmem>>>(dA, dB, 1, 1, dump, clk);
    else overlap_test<2><<<1, 128, kSmem>>>(dA, dB, 1, 1, dump, clk);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("overlap mode %d: %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> D(128 * 224);
    cudaMemcpy(D.data(), dump, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (size_t i = 0; i < D.size(); ++i)
      if (D[i] != static_cast<float>(12.0 * E[i])) ++bad;
    printf("overlap correctness mode %d (%s): %d / %zu mismatches\n", mode,
           mode == 2 ? "A from TMEM" : "A from smem", bad, D.size());
  }
  for (int mode : {0, 1, 2}) {
    const int reps = 200, inner = 12;
    if (mode == 0) overlap_test<0><<<148, 128, kSmem>>>(dA, dB, reps, inner, dump, clk);
    else if (mode == 1) overlap_test<1><<<148, 128, kSmem>>>(dA, dB, reps, inner, dump, clk);
    else overlap_test<2><<<148, 128, kSmem>>>(dA, dB, reps, inner, dump, clk);
    cudaDeviceSynchronize();
    unsigned long long c;
    cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    const double n = static_cast<double>(reps) * kW * 12;
    printf("rate mode %d (%s): %.1f clk/UMMA (5 of 7 windows N=96, 2 N=64)\n", mode,
           mode == 0 ? "sliding windows, smem A" : mode == 1 ? "one D, smem A" : "sliding, TMEM A",
           static_cast<double>(c) / n);
  }
  run_commit<0>(clk); run_commit<12>(clk); run_commit<-12>(clk); run_commit<-4>(clk);
  run_mixed<0>(clk); run_mixed<1>(clk); run_mixed<2>(clk); run_mixed<3>(clk); run_mixed<4>(clk); run_mixed<5>(clk); run_mixed<8>(clk); run_mixed<9>(clk); run_mixed<15>(clk);
  run_fixed<16, 1>(clk); run_fixed<32, 1>(clk); run_fixed<48, 1>(clk); run_fixed<64, 1>(clk);
  run_fixed<96, 1>(clk); run_fixed<128, 1>(clk); run_fixed<32, 0>(clk); run_fixed<64, 0>(clk); run_fixed<96, 0>(clk);
  for (int st : {0, 1})
    for (int warps : {4, 8, 16})
      for (int batch : {1, 2, 4}) {
        const int reps = 4096;
        ld_rate<<<148, warps * 32>>>(reps, batch, st, clk, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("ld_rate: %s\n", cudaGetErrorString(e));
          return 1;
        }
        unsigned long long c;
        cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
        const double bytes = static_cast<double>(reps) * warps * 32 * 32 * 4;
        printf("tcgen05.%s x32: %2d warps, wait every %d: %.1f B/clk/SM (%.1f clk per warp-instruction)\n",
               st ? "st" : "ld", warps, batch, bytes / static_cast<double>(c),
               static_cast<double>(c) / reps);
      }
  return 0;
}
