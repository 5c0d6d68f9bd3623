// Device-side building blocks of the AMSP step kernels (sm_100a).
//
// The element math is the one defined in oracle/amsp_oracle.c (header
// comment): every operation is an explicitly rounded binary32 intrinsic so
// nvcc cannot contract or reorder it, which makes the GPU result bit-equal
// to the -ffp-contract=off CPU oracle.
#pragma once

#include <cuda_bf16.h>
#include <cstdint>

#include "kernels.h"

namespace amsp {


// ---------------------------------------------------------------- counters

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ((h >> 40) - 2^23) * 2^-23: exact in binary32, in [-1, 1).
__device__ __forceinline__ float unit_from_key(uint64_t key) {
  const int32_t q = static_cast<int32_t>(splitmix64(key) >> 40) - (1 << 23);
  return __fmul_rn(static_cast<float>(q), 1.0f / 8388608.0f);
}

// Micro-batch mu of step t (mu = 0 is the single-micro-batch key).
__device__ __forceinline__ uint64_t grad_key(uint64_t seed, uint32_t step, uint32_t mb,
                                             uint32_t rank, uint64_t index) {
  return seed ^ (static_cast<uint64_t>(step) << 48) ^ (static_cast<uint64_t>(mb) << 44) ^
         (static_cast<uint64_t>(rank) << 40) ^ index;
}

__device__ __forceinline__ float grad_value(uint64_t seed, uint32_t step, uint32_t mb,
                                            uint32_t rank, uint64_t index) {
  return __fmul_rn(unit_from_key(grad_key(seed, step, mb, rank, index)), 0.0078125f);
}

__device__ __forceinline__ float master_init(uint64_t seed, uint64_t index) {
  return __fmul_rn(0.02f, unit_from_key(seed ^ (0xFFFFull << 48) ^ index));
}

// ---------------------------------------------------------------- bf16

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ float bf16_at(uint16_t h) {
  return __uint_as_float(static_cast<uint32_t>(h) << 16);
}

// Round-to-nearest-even pack; .x (lo) lands at the lower address.
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  uint32_t u;
  memcpy(&u, &h, sizeof(u));
  return u;
}

__device__ __forceinline__ uint16_t to_bf16(float x) {
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  uint16_t u;
  memcpy(&u, &h, sizeof(u));
  return u;
}

// ---------------------------------------------------------------- memory
// 128-bit streaming accesses. Gradients are read-only for the kernel's
// lifetime (possibly from a peer GPU over NVLink): non-coherent path, no L1
// allocation. Optimizer state is read then written by the same thread.

__device__ __forceinline__ uint4 ld_ro_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float4 ld_state_v4(const float* p) {
  float4 r;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream_v4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// Streaming (evict-first) 128-bit store for outputs nobody re-reads soon.
__device__ __forceinline__ void st_stream_u4(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// Read-only 128-bit fp32 load (non-coherent path, no L1 allocation).
__device__ __forceinline__ float4 ld_ro_f4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// ---------------------------------------------------------------- AdamW

__device__ __forceinline__ void adamw(const AdamScalars& s, float g, float& p,
                                      float& m, float& v) {
  const float mm = __fadd_rn(__fmul_rn(s.beta1, m), __fmul_rn(s.omb1, g));
  const float vv =
      __fadd_rn(__fmul_rn(s.beta2, v), __fmul_rn(__fmul_rn(s.omb2, g), g));
  const float d = __fadd_rn(__fmul_rn(__fsqrt_rn(vv), s.inv_sqrt_bc2), s.eps);
  float pp = __fmul_rn(p, s.decay);
  pp = __fsub_rn(pp, __fmul_rn(s.step_size, __fdiv_rn(mm, d)));
  m = mm;
  v = vv;
  p = pp;
}

}  // namespace amsp
