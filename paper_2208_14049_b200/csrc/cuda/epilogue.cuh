// Shared epilogue step of the TMEM-resident member kernels: fp32 hidden
// pre-activations -> +bias, ReLU, bf16 -> written back into the same TMEM
// columns as the A operand of layer 2.
#pragma once

#include <cuda_bf16.h>

#include "sm100.cuh"

namespace es {

__device__ __forceinline__ uint32_t pack_relu_bf16x2(uint32_t lo_bits, uint32_t hi_bits, float blo,
                                                     float bhi) {
  const float lo = fmaxf(__uint_as_float(lo_bits) + blo, 0.0f);
  const float hi = fmaxf(__uint_as_float(hi_bits) + bhi, 0.0f);
  __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);  // .x (low half) = lo
  return *reinterpret_cast<uint32_t*>(&p);
}

// bf16x2 {relu(lo + blo), relu(hi + bhi)} with one cvt.rn.relu (the same bits
// as fmaxf then round-to-nearest-even for every finite input).
__device__ __forceinline__ uint32_t add_relu_bf16x2(uint32_t lo_bits, uint32_t hi_bits, float blo,
                                                    float bhi) {
  const float lo = __uint_as_float(lo_bits) + blo;
  const float hi = __uint_as_float(hi_bits) + bhi;
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// 32 fp32 columns -> 16 bf16 pairs in TMEM; biases as float4 loads (`bias`
// 16-byte aligned).
__device__ __forceinline__ void relu_bf16_chunk(const uint32_t (&r)[32], const float* bias,
                                                uint32_t dst) {
  uint32_t p[16];
  const float4* b4 = reinterpret_cast<const float4*>(bias);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 bv = b4[j];
    p[2 * j] = add_relu_bf16x2(r[4 * j], r[4 * j + 1], bv.x, bv.y);
    p[2 * j + 1] = add_relu_bf16x2(r[4 * j + 2], r[4 * j + 3], bv.z, bv.w);
  }
  sm100::tmem_st16(dst, p);
}

// This warp's 32 lanes, fp32 columns [base, base + ncols) -> bf16 pairs at
// [base, base + ncols/2).  ncols is a multiple of 64.  The load of chunk i+1 is
// in flight while chunk i is converted; every store lands on columns whose
// fp32 values were already read (chunk i writes [16i, 16i+16) <= 32i).
__device__ __forceinline__ void hidden_to_bf16(uint32_t base, const float* bias, int ncols) {
  uint32_t ra[32], rb[32];
  const int chunks = ncols / 32;
  sm100::tmem_ld32_raw(base, ra);
  sm100::tmem_ld_wait();
  for (int i = 0; i < chunks; i += 2) {
    sm100::tmem_ld32_raw(base + 32u * (i + 1), rb);
    relu_bf16_chunk(ra, bias + 32 * i, base + 16u * i);
    sm100::tmem_ld_wait();
    if (i + 2 < chunks) sm100::tmem_ld32_raw(base + 32u * (i + 2), ra);
    relu_bf16_chunk(rb, bias + 32 * (i + 1), base + 16u * (i + 1));
    sm100::tmem_ld_wait();
  }
  sm100::tmem_st_wait();
}

// Layer-2 accumulators: `parts` independent 16-column partial sums (so the
// dependent UMMA chain is parts times shorter), reduced here in fixed order.
__device__ __forceinline__ void read_d2(uint32_t addr, int parts, float (&z)[16]) {
  sm100::tmem_ld16(addr, z);
  for (int p = 1; p < parts; ++p) {
    float t[16];
    sm100::tmem_ld16(addr + 16u * p, t);
#pragma unroll
    for (int c = 0; c < 16; ++c) z[c] += t[c];
  }
}

}  // namespace es
