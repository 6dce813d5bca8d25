// Design evidence, not product: issue-to-completion rate of back-to-back
// tcgen05.mma (M=128, K=16, bf16) for operand layouts the member kernels use.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_2208_14049_b200/csrc \
//        umma_rate.cu -o umma_rate
#include <cuda_runtime.h>

#include <cstdio>

#include "cuda/sm100.cuh"

using namespace es::sm100;

// layout 0: SW128 K-major (A and B); 1: planar no-swizzle (A and B);
// shift: A start moved by `shift` rows of 16 B (planar only).
__global__ void __launch_bounds__(128, 1) rate(int layout, int N, int shift, int reps,
                                               unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
    const uint32_t idesc = idesc_bf16_f32(128, N);
    uint64_t ad, bd;
    if (layout == 0) {
      ad = sdesc_k128(a);
      bd = sdesc_k128(b);
    } else {
      ad = sdesc_planar(a + shift * 16, 160 * 16);
      bd = sdesc_planar(b, N * 16);
    }
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) umma_bf16(tmem, ad, bd, idesc, r != 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = static_cast<unsigned long long>(t1 - t0);
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

// Descriptors recomputed per MMA (as the conv kernel's tap loop does): issued
// from lane 0 only (mode 0) or from a converged warp with elect.sync (mode 1).
__global__ void __launch_bounds__(128, 1) rate_varying(int mode, int N, int reps,
                                                       unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
  const uint32_t idesc = idesc_bf16_f32(128, N);
  if (mode == 0) {
    if (threadIdx.x == 0) {
      const long long t0 = clock64();
      for (int r = 0; r < reps; ++r) {
        const int t = r % 9, j = (r / 9) & 3;
        umma_bf16(tmem, sdesc_planar(a + (16 + (t / 3 - 1) * 9 + t % 3) * 16 + j * 2 * 2560, 2560),
                  sdesc_planar(b + t * 2048 + j * 256, N * 16), idesc, r != 0);
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      if (blockIdx.x == 0) out[0] = static_cast<unsigned long long>(clock64() - t0);
    }
  } else if (threadIdx.x < 32) {
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int t = r % 9, j = (r / 9) & 3;
      const uint64_t ad = sdesc_planar(a + (16 + (t / 3 - 1) * 9 + t % 3) * 16 + j * 2 * 2560, 2560);
      const uint64_t bd = sdesc_planar(b + t * 2048 + j * 256, N * 16);
      if (elect_one()) umma_bf16(tmem, ad, bd, idesc, r != 0);
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = static_cast<unsigned long long>(clock64() - t0);
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

// Descriptors from a per-tap table, loops unrolled (9 taps x 4 K steps):
// mode 2 = converged warp (warp index made provably uniform) + elect.sync,
// mode 3 = lane 0 only.
__global__ void __launch_bounds__(128, 1) rate_table(int mode, int N, int reps, int pad,
                                                     unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
  const uint32_t idesc = idesc_bf16_f32(128, N);
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const uint64_t ad0 = sdesc_planar(a + 16 * 16, 2560), bd0 = sdesc_planar(b, N * 16);
  int otab[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) otab[t] = (t / 3 - 1) * pad + (t % 3 - 1);
  auto body = [&](bool elect) {
    const long long t0 = clock64();
    for (int r = 0; r < reps; r += 36) {
#pragma unroll
      for (int t = 0; t < 9; ++t)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t ad = ad0 + static_cast<uint64_t>(otab[t] + j * 320);
          const uint64_t bd = bd0 + static_cast<uint64_t>(t * 4 * N + j * 2 * N);
          if (!elect || elect_one()) umma_bf16(tmem, ad, bd, idesc, (r | t | j) != 0);
        }
    }
    if (!elect || elect_one()) umma_commit(&bar);
    __syncwarp(elect ? 0xffffffffu : 1u);
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = static_cast<unsigned long long>(clock64() - t0);
  };
  if (mode == 2) {
    if (warp == 0) body(true);
  } else if (threadIdx.x == 0) {
    body(false);
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

// Independent accumulators: MMA r accumulates into chain r % chains (TMEM
// columns chain * N), so consecutive MMAs carry no accumulator dependency.
template <int CH>
__global__ void __launch_bounds__(128, 1) rate_chains(int N, int reps, unsigned long long* out,
                                                      int M = 128) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
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
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 64 * 1024);
    const uint32_t idesc = idesc_bf16_f32(M, N);
    const uint64_t ad = sdesc_planar(a, 160 * 16), bd = sdesc_planar(b, N * 16);
    const long long t0 = clock64();
    for (int r = 0; r < reps; r += CH) {
#pragma unroll
      for (int c = 0; c < CH; ++c)
        umma_bf16(tmem + static_cast<uint32_t>(c * N), ad, bd, idesc, r > 0);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0) out[0] = static_cast<unsigned long long>(clock64() - t0);
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// A operand from TMEM (tcgen05.mma ... [a_tmem]): only B is read from smem.
template <int CH>
__global__ void __launch_bounds__(128, 1) rate_ta(int N, int reps, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
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
    const uint32_t b = smem_u32(smem + 64 * 1024);
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint64_t bd = sdesc_planar(b, N * 16);
    const long long t0 = clock64();
    for (int r = 0; r < reps; r += CH) {
#pragma unroll
      for (int c = 0; c < CH; ++c)
        umma_bf16_ta(tmem + static_cast<uint32_t>(c * N), tmem + 256u + static_cast<uint32_t>(c * 8),
                     bd, idesc, r > 0);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0) out[0] = static_cast<unsigned long long>(clock64() - t0);
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// The conv kernel's split conv2 block: 3 dw shifts x 4 K steps, A planar
// (plane 4608 B, start moved by -1/0/+1 rows), B planar N = 96.
// rand_fill: operands filled with random bf16 in (-1, 1) instead of zeros
// (the tensor pipe's rate on real data, not on all-zero operands).
__global__ void __launch_bounds__(512, 1) rate_split(int N, int reps, int shift_on,
                                                     unsigned long long* out, int dcol = 0,
                                                     int boff = 0, int rand_fill = 0,
                                                     int idle_mode = 0) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) {
    uint32_t v = 0;
    if (rand_fill) {
      uint32_t h = (i + 1) * 2654435761u;
      h ^= h >> 15;
      h *= 2246822519u;
      h ^= h >> 13;
      // two bf16 with sign, exponent 0x7E or 0x7D (|x| in [0.25, 1)), random mantissa
      const uint32_t lo = ((h & 1u) << 15) | ((0x7Du + ((h >> 1) & 1u)) << 7) | ((h >> 2) & 0x7Fu);
      const uint32_t hi = (((h >> 9) & 1u) << 15) | ((0x7Du + ((h >> 10) & 1u)) << 7) | ((h >> 11) & 0x7Fu);
      v = lo | (hi << 16);
    }
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
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
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  __shared__ uint64_t idle_bar;
  if (threadIdx.x == 0) {
    mbar_init(&idle_bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp >= 4) {  // idle warps: 1 = suspended try_wait, 2 = spinning try_wait
    if (idle_mode == 1) mbar_sleep_wait(&idle_bar, 0);
    if (idle_mode == 2) mbar_wait(&idle_bar, 0);
  }
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 40 * 1024 + boff);
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint64_t ad0 = sdesc_planar(a + 16 * 16, 4608), bd0 = sdesc_planar(b, N * 16);
    const uint32_t dt = tmem + static_cast<uint32_t>(dcol);
    const long long t0 = clock64();
    for (int r = 0; r < reps; r += 12) {
      // rotate (idle_mode >= 3): each block reads another 8 KB window of A,
      // as the kernel does (a new grid block every time), not the same bytes
      const uint64_t rot = idle_mode >= 3 ? static_cast<uint64_t>(((r / 12) % 4) * 128) : 0;
#pragma unroll
      for (int dwi = 0; dwi < 3; ++dwi)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t ad = ad0 + rot + static_cast<uint64_t>((dwi - 1) * 8 * shift_on - shift_on + j * 576);
          const uint64_t bd = bd0 + static_cast<uint64_t>((dwi * 4 + j) * 2 * N);
          // idle_mode 4: the kernel's ring -- every block starts a fresh
          // accumulation in the next of 3 slots; 5: plus a commit per block
          const uint32_t dslot = idle_mode >= 4 ? dt + static_cast<uint32_t>(((r / 12) % 3) * 96) : dt;
          const uint32_t acc = idle_mode >= 4 ? ((dwi | j) != 0) : ((r | dwi | j) != 0);
          if (elect_one()) umma_bf16(dslot, ad, bd, idesc, acc);
        }
      if (idle_mode == 5 && elect_one()) umma_commit(&idle_bar);
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = static_cast<unsigned long long>(clock64() - t0);
    if (threadIdx.x == 0) mbar_arrive(&idle_bar);
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// The conv kernel's slot protocol without its data flow: warp 0 issues the
// split pattern into a ring of `slots` TMEM slots, committing c2_full[s] per
// block and waiting c2_empty[s] before reusing a slot; warp 1 (the
// "epilogue") waits c2_full[s] and arrives c2_empty[s] (optionally after a
// tcgen05.ld of the slot).
__global__ void __launch_bounds__(128, 1) rate_ring(int reps, int slots, int epi_ld,
                                                    unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t full[4], empty[4], done;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int blocks = reps / 12;
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 40 * 1024);
    const uint32_t idesc = idesc_bf16_f32(128, 96);
    const uint64_t ad0 = sdesc_planar(a + 16 * 16, 4608), bd0 = sdesc_planar(b, 96 * 16);
    const long long t0 = clock64();
    for (int blk = 0; blk < blocks; ++blk) {
      const int sl = blk % slots;
      mbar_wait(&empty[sl], (static_cast<uint32_t>(blk / slots) & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t d = tmem + 128u + static_cast<uint32_t>(sl * 96);
#pragma unroll
      for (int dwi = 0; dwi < 3; ++dwi)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t ad = ad0 + static_cast<uint64_t>((dwi - 1) * 8 - 1 + j * 576);
          const uint64_t bd = bd0 + static_cast<uint64_t>((dwi * 4 + j) * 2 * 96);
          if (elect_one()) umma_bf16(d, ad, bd, idesc, (dwi | j) != 0);
        }
      if (elect_one()) umma_commit(&full[sl]);
      __syncwarp();
    }
    mbar_wait(&done, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = static_cast<unsigned long long>(clock64() - t0);
  } else if (warp == 1) {
    for (int blk = 0; blk < blocks; ++blk) {
      const int sl = blk % slots;
      mbar_wait(&full[sl], static_cast<uint32_t>(blk / slots) & 1u);
      tc_fence_after();
      if (epi_ld) {
        uint32_t r[32];
        tmem_ld32_raw(tmem + 128u + static_cast<uint32_t>(sl * 96), r);
        tmem_ld_wait();
        if (r[0] == 0x12345678u && r[31] == 7u) out[1] = r[1];  // keep the load
      }
      tc_fence_before();
      __syncwarp();
      if (threadIdx.x == 32) mbar_arrive(&empty[sl]);
    }
    if (threadIdx.x == 32) mbar_arrive(&done);
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// The conv kernel's two-chain structure without its data: per tile, warp 1
// issues conv1 (2 UMMAs M=128 N=64) into ONE TMEM buffer (c1_full commit,
// waits c1_empty); an "epi1" warp waits c1_full, arrives c1_empty at once,
// waits a2_empty[t % nbuf_a2] and arrives a2_full[t % nbuf_a2]; warp 0
// (conv2) waits a2_full, issues 2 blocks x 12 UMMAs (N=96) into a 3-slot ring
// (c2_full per block, commits a2_empty after the tile); an "epi2" warp
// releases the slots.  mode bit 0: conv1 issued by warp 0 right before
// conv2 of the previous tile instead of by warp 1.
__global__ void __launch_bounds__(384, 1) rate_chain(int tiles, int mode, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t c1f, c1e, c1e8, a2f[2], a2e[2], c2f[3], c2e[3], done;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&c1f, 1);
    mbar_init(&c1e, 1);
    mbar_init(&c1e8, 8);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a2f[i], 1);
      mbar_init(&a2e[i], 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&c2f[i], 1);
      mbar_init(&c2e[i], 1);
    }
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const uint32_t a = smem_u32(smem), b = smem_u32(smem + 40 * 1024);
  const uint32_t id1 = idesc_bf16_f32(128, 64), id2 = idesc_bf16_f32(128, 96);
  const uint64_t ad0 = sdesc_planar(a + 16 * 16, 4608), bd0 = sdesc_planar(b, 96 * 16);
  const uint64_t a1d = sdesc_planar(a + 60 * 1024, 4096), w1d = sdesc_planar(b + 40 * 1024, 64 * 16);
  const bool fused = mode & 1;
  auto conv1 = [&](int t) {
    mbar_wait(&c1e, (static_cast<uint32_t>(t) & 1u) ^ 1u);
    tc_fence_after();
    for (int mb = 0; mb < 2; ++mb)
      if (elect_one()) umma_bf16(tmem + static_cast<uint32_t>(mb * 64), a1d + mb * 128, w1d, id1, 0);
    if (elect_one()) umma_commit(&c1f);
    __syncwarp();
  };
  if (warp == 0) {
    const long long t0 = clock64();
    if (fused) conv1(0);
    for (int t = 0; t < tiles; ++t) {
      if (fused && t + 1 < tiles) conv1(t + 1);
      const int ab = t & 1;
      mbar_wait(&a2f[ab], static_cast<uint32_t>(t >> 1) & 1u);
      tc_fence_after();
      for (int mb = 0; mb < 2; ++mb) {
        const int blk = t * 2 + mb, sl = blk % 3;
        mbar_wait(&c2e[sl], (static_cast<uint32_t>(blk / 3) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + 128u + static_cast<uint32_t>(sl * 96);
#pragma unroll
        for (int dwi = 0; dwi < 3; ++dwi)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t ad = ad0 + static_cast<uint64_t>(mb * 128 + (dwi - 1) * 8 - 1 + j * 576);
            const uint64_t bd = bd0 + static_cast<uint64_t>((dwi * 4 + j) * 2 * 96);
            if (elect_one()) umma_bf16(d, ad, bd, id2, (dwi | j) != 0);
          }
        if (elect_one()) {
          umma_commit(&c2f[sl]);
          if (mb == 1) umma_commit(&a2e[ab]);
        }
        __syncwarp();
      }
    }
    mbar_wait(&done, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = static_cast<unsigned long long>(clock64() - t0);
  } else if (warp == 1) {
    if (!fused)
      for (int t = 0; t < tiles; ++t) conv1(t);
  } else if (warp == 2 || warp >= 4) {  // epi1 (mode bit 2: 8 warps that tcgen05.ld conv1's TMEM)
    const bool ld = mode & 4;
    if (warp >= 4 && !ld) {
      // idle
    } else {
    for (int t = 0; t < tiles; ++t) {
      mbar_wait(&c1f, static_cast<uint32_t>(t) & 1u);
      tc_fence_after();
      if (ld && warp >= 4) {
        const int ew = warp - 4, q = warp & 3;
        uint32_t v0[32], v1[32];
        const uint32_t base = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>((ew >> 2) * 32);
        tmem_ld32_raw(base, v0);
        tmem_ld32_raw(base + 64u, v1);
        tmem_ld_wait();
        if (v0[3] == 0x7fffffffu && v1[5] == 3u) out[1] = v0[0];
      }
      tc_fence_before();
      if (ld) {
        // c1 buffer released by the 8 loading warps (count 8 via lane 0 of each)
        if (warp >= 4 && (threadIdx.x & 31) == 0) mbar_arrive(&c1e8);
      } else if (threadIdx.x == 64) {
        mbar_arrive(&c1e);
      }
      if (warp >= 4) continue;
      const int ab = t & 1;
      mbar_wait(&a2e[ab], (static_cast<uint32_t>(t >> 1) & 1u) ^ 1u);
      if (ld) mbar_wait(&c1e8, static_cast<uint32_t>(t) & 1u);  // the loads are done
      if (mode & 2) {  // the kernel's generic -> async proxy fence before the hand-off
        reinterpret_cast<volatile uint32_t*>(smem + 60 * 1024)[threadIdx.x] = t;
        fence_proxy_async_smem();
      }
      if (threadIdx.x == 64) {
        if (ld) mbar_arrive(&c1e);
        mbar_arrive(&a2f[ab]);
      }
    }
    }
  } else if (warp == 3) {  // epi2
    for (int blk = 0; blk < 2 * tiles; ++blk) {
      const int sl = blk % 3;
      mbar_wait(&c2f[sl], static_cast<uint32_t>(blk / 3) & 1u);
      tc_fence_before();
      if (threadIdx.x == 96) mbar_arrive(&c2e[sl]);
    }
    if (threadIdx.x == 96) mbar_arrive(&done);
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

__device__ __forceinline__ void tshift(uint32_t taddr) {
  asm volatile("tcgen05.shift.cta_group::1.down [%0];" ::"r"(taddr) : "memory");
}

// The conv kernel's split pipeline: per block 12 UMMAs (N = 96) into a ring
// slot, then 12 tcgen05.shift on an older slot (nshift = 0: UMMAs only).
__global__ void __launch_bounds__(128, 1) rate_mix(int reps, int nshift, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
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
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 40 * 1024);
    const uint32_t idesc = idesc_bf16_f32(128, 96);
    const uint64_t ad0 = sdesc_planar(a + 16 * 16, 4608), bd0 = sdesc_planar(b, 96 * 16);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t d = tmem + 128u + static_cast<uint32_t>((r % 3) * 96);
#pragma unroll
      for (int dhi = 0; dhi < 3; ++dhi)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t ad = ad0 + static_cast<uint64_t>((dhi - 1) * 8 - 1 + j * 576);
          const uint64_t bd = bd0 + static_cast<uint64_t>((dhi * 4 + j) * 2 * 96);
          if (elect_one()) umma_bf16(d, ad, bd, idesc, (dhi | j) != 0);
        }
      const uint32_t ds = tmem + 128u + static_cast<uint32_t>(((r + 2) % 3) * 96);
      for (int c = 0; c < 32 && nshift; c += 8) {
        if (elect_one()) tshift(ds + 32u + c);
        if (elect_one()) tshift(ds + 64u + c);
        if (elect_one()) tshift(ds + 64u + c);
      }
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = static_cast<unsigned long long>(clock64() - t0);
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// Two issuers as in the conv kernel: warp 0 issues each block's 12 UMMAs
// (ring of 3 slots, commit per block); warp 1 waits for a block's commit and
// issues its 12 shifts (+ commit).  Returns clk per block.
__global__ void __launch_bounds__(128, 1) rate_two_issuers(int reps, int shifts_by_warp1,
                                                           unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t done[3], sdone[3];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) {
      mbar_init(&done[i], 1);
      mbar_init(&sdone[i], 1);
    }
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const long long t0 = clock64();
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 40 * 1024);
    const uint32_t idesc = idesc_bf16_f32(128, 96);
    const uint64_t ad0 = sdesc_planar(a + 16 * 16, 4608), bd0 = sdesc_planar(b, 96 * 16);
    for (int r = 0; r < reps; ++r) {
      const int sl = r % 3;
      if (r >= 3) mbar_wait(&sdone[sl], static_cast<uint32_t>((r / 3) - 1) & 1u);  // slot free
      tc_fence_after();
      const uint32_t d = tmem + 128u + static_cast<uint32_t>(sl * 96);
#pragma unroll
      for (int dhi = 0; dhi < 3; ++dhi)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t ad = ad0 + static_cast<uint64_t>((dhi - 1) * 8 - 1 + j * 576);
          const uint64_t bd = bd0 + static_cast<uint64_t>((dhi * 4 + j) * 2 * 96);
          if (elect_one()) umma_bf16(d, ad, bd, idesc, (dhi | j) != 0);
        }
      if (elect_one()) umma_commit(&done[sl]);
      __syncwarp();
    }
  } else if (warp == 1) {
    for (int r = 0; r < reps; ++r) {
      const int sl = r % 3;
      mbar_wait(&done[sl], static_cast<uint32_t>(r / 3) & 1u);
      tc_fence_after();
      const uint32_t d = tmem + 128u + static_cast<uint32_t>(sl * 96);
      for (int c = 0; c < 32 && shifts_by_warp1; c += 8) {
        if (elect_one()) tshift(d + 32u + c);
        if (elect_one()) tshift(d + 64u + c);
        if (elect_one()) tshift(d + 64u + c);
      }
      if (elect_one()) umma_commit(&sdone[sl]);
      __syncwarp();
    }
    mbar_wait(&sdone[(reps - 1) % 3], static_cast<uint32_t>((reps - 1) / 3) & 1u);
    if (blockIdx.x == 0 && threadIdx.x == 32) out[0] = static_cast<unsigned long long>(clock64() - t0);
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

// The conv kernel's conv2 issuer: UMMAs of block r, then (after waiting for
// block r-1's commit) block r-1's 12 shifts, one warp.
__global__ void __launch_bounds__(128, 1) rate_issuer(int reps, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t done[3];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&done[i], 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 40 * 1024);
    const uint32_t idesc = idesc_bf16_f32(128, 96);
    const uint64_t ad0 = sdesc_planar(a + 16 * 16, 4608), bd0 = sdesc_planar(b, 96 * 16);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int sl = r % 3;
      const uint32_t d = tmem + 128u + static_cast<uint32_t>(sl * 96);
#pragma unroll
      for (int dhi = 0; dhi < 3; ++dhi)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t ad = ad0 + static_cast<uint64_t>((dhi - 1) * 8 - 1 + j * 576);
          const uint64_t bd = bd0 + static_cast<uint64_t>((dhi * 4 + j) * 2 * 96);
          if (elect_one()) umma_bf16(d, ad, bd, idesc, (dhi | j) != 0);
        }
      if (elect_one()) umma_commit(&done[sl]);
      __syncwarp();
      if (r > 0) {
        const int ps = (r - 1) % 3;
        mbar_wait(&done[ps], static_cast<uint32_t>((r - 1) / 3) & 1u);
        tc_fence_after();
        const uint32_t dp = tmem + 128u + static_cast<uint32_t>(ps * 96);
        for (int c = 0; c < 32; c += 8) {
          if (elect_one()) tshift(dp + 32u + c);
          if (elect_one()) tshift(dp + 64u + c);
          if (elect_one()) tshift(dp + 64u + c);
        }
      }
    }
    mbar_wait(&done[(reps - 1) % 3], static_cast<uint32_t>((reps - 1) / 3) & 1u);
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = static_cast<unsigned long long>(clock64() - t0);
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
  {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(rate_issuer, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    rate_issuer<<<148, 128, 100 * 1024>>>(60, d);
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    std::printf("conv2 issuer pattern: %.1f clk per block %s\n", double(c) / 60,
                cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
  }
  {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(rate_two_issuers, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int ns = 0; ns < 2; ++ns) {
      rate_two_issuers<<<148, 128, 100 * 1024>>>(60, ns, d);
      unsigned long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      std::printf("two issuers, shifts=%d: %.1f clk per block %s\n", ns, double(c) / 60,
                  cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(d);
  }
  {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(rate_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int ns = 0; ns < 2; ++ns) {
      rate_mix<<<148, 128, 100 * 1024>>>(60, ns, d);
      unsigned long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      std::printf("mix shifts=%d: %.1f clk per block (12 UMMA N=96%s) %s\n", ns, double(c) / 60,
                  ns ? " + 12 shifts" : "", cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(d);
  }
  {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(rate_split, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int N : {32, 96})
      for (int sh = 0; sh < 2; ++sh) {
        rate_split<<<148, 128, 100 * 1024>>>(N, 504, sh, d, 0, 0);
        unsigned long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        std::printf("split pattern N=%d shifts=%d: %6.1f clk/MMA %s\n", N, sh, double(c) / 504,
                    cudaGetErrorString(cudaGetLastError()));
      }
    for (int N : {32, 96, 128})
      for (int rf = 0; rf < 2; ++rf) {
        rate_split<<<148, 128, 100 * 1024>>>(N, 504, 1, d, 0, 0, rf);
        unsigned long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        std::printf("split pattern N=%d operands=%s: %6.1f clk/MMA %s\n", N, rf ? "random" : "zero",
                    double(c) / 504, cudaGetErrorString(cudaGetLastError()));
      }
    cudaFuncSetAttribute(rate_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int mode : {0, 1, 4, 5}) {
      unsigned long long* d3;
      cudaMalloc(&d3, 16);
      rate_chain<<<148, 384, 100 * 1024>>>(200, mode, d3);
      unsigned long long c = 0;
      cudaMemcpy(&c, d3, 8, cudaMemcpyDeviceToHost);
      std::printf("chain mode=%d (%s%s): %6.1f clk per tile (%5.1f per conv2 UMMA) %s\n", mode,
                  (mode & 1) ? "conv1 from the conv2 issuer" : "conv1 from its own warp",
                  (mode & 4) ? ", 8 epi1 warps tcgen05.ld conv1" : "", double(c) / 200,
                  double(c) / 200 / 24, cudaGetErrorString(cudaGetLastError()));
      cudaFree(d3);
    }
    cudaFuncSetAttribute(rate_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int slots : {2, 3, 4})
      for (int ld = 0; ld < 2; ++ld) {
        unsigned long long* d2;
        cudaMalloc(&d2, 16);
        rate_ring<<<148, 128, 100 * 1024>>>(1200, slots, ld, d2);
        unsigned long long c = 0;
        cudaMemcpy(&c, d2, 8, cudaMemcpyDeviceToHost);
        std::printf("ring slots=%d epilogue_ld=%d: %6.1f clk/MMA %s\n", slots, ld, double(c) / 1200,
                    cudaGetErrorString(cudaGetLastError()));
        cudaFree(d2);
      }
    for (int threads : {128, 480})
      for (int idle = 0; idle < 6; ++idle) {
        if (threads == 128 && idle && idle < 3) continue;
        rate_split<<<148, threads, 100 * 1024>>>(96, 504, 1, d, 0, 0, 1, idle);
        unsigned long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        std::printf("split N=96 threads=%d idle=%s: %6.1f clk/MMA %s\n", threads,
                    idle == 0 ? "exit" : idle == 1 ? "sleep-wait" : idle == 2 ? "spin-wait" : idle == 3 ? "rotating A" : idle == 4 ? "slot ring" : "ring+commit", double(c) / 504,
                    cudaGetErrorString(cudaGetLastError()));
      }
    for (int dcol : {0, 96, 256, 352})
      for (int boff : {0, 128, 512}) {
        rate_split<<<148, 128, 100 * 1024>>>(96, 504, 1, d, dcol, boff);
        unsigned long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        std::printf("split N=96 dcol=%d boff=%d: %6.1f clk/MMA %s\n", dcol, boff, double(c) / 504,
                    cudaGetErrorString(cudaGetLastError()));
      }
    cudaFree(d);
  }
  {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(rate_chains<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int N : {32, 64, 128, 256}) {
      rate_chains<1><<<148, 128, 100 * 1024>>>(N, 512, d, 64);
      unsigned long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      std::printf("M=64 N=%3d: %6.1f clk/MMA  (%5.0f MAC/clk) %s\n", N, double(c) / 512,
                  64.0 * N * 16 * 512 / double(c), cudaGetErrorString(cudaGetLastError()));
    }
    cudaFuncSetAttribute(rate_ta<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(rate_ta<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int N : {16, 32, 64, 128, 256})
      for (int ci = 0; ci < 2; ++ci) {
        if (N * (1 << ci) > 256) continue;
        (ci ? rate_ta<2> : rate_ta<1>)<<<148, 128, 100 * 1024>>>(N, 512, d);
        unsigned long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        std::printf("A=tmem chains=%d N=%3d: %6.1f clk/MMA  (%5.0f MAC/clk) %s\n", 1 << ci, N,
                    double(c) / 512, 128.0 * N * 16 * 512 / double(c),
                    cudaGetErrorString(cudaGetLastError()));
      }
    cudaFree(d);
  }
  {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    auto fns = {rate_chains<1>, rate_chains<2>, rate_chains<4>, rate_chains<8>};
    for (auto f : fns) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int N : {16, 32, 64, 96, 128})
      for (int ci = 0; ci < 4; ++ci) {
        const int chains = 1 << ci;
        if (N * chains > 512) continue;
        auto f = ci == 0 ? rate_chains<1> : ci == 1 ? rate_chains<2> : ci == 2 ? rate_chains<4> : rate_chains<8>;
        f<<<148, 128, 100 * 1024>>>(N, 512, d, 128);
        unsigned long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        std::printf("chains=%d N=%3d: %6.1f clk/MMA  (%5.0f MAC/clk) %s\n", chains, N,
                    double(c) / 512, 128.0 * N * 16 * 512 / double(c),
                    cudaGetErrorString(cudaGetLastError()));
      }
    cudaFree(d);
  }
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int reps = 512;
  for (int layout = 0; layout < 2; ++layout)
    for (int N : {32, 64, 128, 256})
      for (int shift : {0, 1, 3}) {
        if (layout == 0 && shift) continue;
        rate<<<148, 128, 100 * 1024>>>(layout, N, shift, reps, d);
        unsigned long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        std::printf("%-7s N=%3d shift=%d: %6.1f clk/MMA  (%5.0f MAC/clk) %s\n",
                    layout ? "planar" : "sw128", N, shift, double(c) / reps,
                    128.0 * N * 16 * reps / double(c), cudaGetErrorString(cudaGetLastError()));
      }
  cudaFuncSetAttribute(rate_varying, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int N : {32, 64, 128}) {
      rate_varying<<<148, 128, 100 * 1024>>>(mode, N, reps, d);
      unsigned long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      std::printf("varying desc, %s N=%3d: %6.1f clk/MMA %s\n", mode ? "warp+elect" : "lane0     ", N,
                  double(c) / reps, cudaGetErrorString(cudaGetLastError()));
    }
  cudaFuncSetAttribute(rate_table, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int mode = 2; mode < 4; ++mode)
    for (int N : {32, 64, 128}) {
      rate_table<<<148, 128, 100 * 1024>>>(mode, N, 504, 9, d);
      unsigned long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      std::printf("tap table, %s N=%3d: %6.1f clk/MMA %s\n", mode == 2 ? "warp+elect" : "lane0     ",
                  N, double(c) / 504, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
