// bs_device.cuh: device helpers shared by the SpMV and SpMM kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "bs.h"

namespace bsk {

// N bytes loaded as one streaming vector load. Packed weights are read exactly once per call, so
// they bypass L1 (L1::no_allocate) and do not displace x in L2.
template <int NBYTES>
struct Vec;
template <>
struct Vec<1> {
  uint32_t w[1];
  __device__ __forceinline__ void load(const void* p) {
    uint16_t t;
    asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(t) : "l"(p));
    w[0] = t;
  }
};
template <>
struct Vec<2> {
  uint32_t w[1];
  __device__ __forceinline__ void load(const void* p) {
    uint16_t t;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(t) : "l"(p));
    w[0] = t;
  }
};
template <>
struct Vec<4> {
  uint32_t w[1];
  __device__ __forceinline__ void load(const void* p) {
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(w[0]) : "l"(p));
  }
};
template <>
struct Vec<8> {
  uint32_t w[2];
  __device__ __forceinline__ void load(const void* p) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "l"(p));
  }
};
template <>
struct Vec<16> {
  uint32_t w[4];
  __device__ __forceinline__ void load(const void* p) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "l"(p));
  }
};

// Element i of a vector of 8-bit or 16-bit lanes packed in 32-bit words (i is a compile-time
// constant after unrolling, so these become PRMT/BFE or register-half selects).
template <int N>
__device__ __forceinline__ uint32_t get_u8(const Vec<N>& v, int i) { return (v.w[i >> 2] >> (8 * (i & 3))) & 0xffu; }
template <int N>
__device__ __forceinline__ uint32_t get_u16(const Vec<N>& v, int i) { return (v.w[i >> 1] >> (16 * (i & 1))) & 0xffffu; }

// acc += w * x with fp32 accumulation. For f16/bf16 both factors stay 16-bit; sm_100's mixed
// FMA (FHFMA) forms the exact product and rounds once into fp32.
template <int DT>
__device__ __forceinline__ void fma_acc(float& acc, uint32_t w, uint32_t x);
template <>
__device__ __forceinline__ void fma_acc<BS_F16>(float& acc, uint32_t w, uint32_t x) {
  const uint16_t a = (uint16_t)w, b = (uint16_t)x;
  asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(a), "h"(b));
}
template <>
__device__ __forceinline__ void fma_acc<BS_BF16>(float& acc, uint32_t w, uint32_t x) {
  const uint16_t a = (uint16_t)w, b = (uint16_t)x;
  asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(acc) : "h"(a), "h"(b));
}
template <>
__device__ __forceinline__ void fma_acc<BS_F32>(float& acc, uint32_t w, uint32_t x) {
  acc = fmaf(__uint_as_float(w), __uint_as_float(x), acc);
}

// fp32 -> storage bits of D, round to nearest even.
template <int DT>
__device__ __forceinline__ uint32_t from_float(float f);
template <>
__device__ __forceinline__ uint32_t from_float<BS_F16>(float f) { return __half_as_ushort(__float2half_rn(f)); }
template <>
__device__ __forceinline__ uint32_t from_float<BS_BF16>(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }
template <>
__device__ __forceinline__ uint32_t from_float<BS_F32>(float f) { return __float_as_uint(f); }

// 16-bit storage -> fp32 (exact).
template <int DT>
__device__ __forceinline__ float to_float(uint32_t bits);
template <>
__device__ __forceinline__ float to_float<BS_F16>(uint32_t b) { return __half2float(__ushort_as_half((uint16_t)b)); }
template <>
__device__ __forceinline__ float to_float<BS_BF16>(uint32_t b) { return __uint_as_float(b << 16); }
template <>
__device__ __forceinline__ float to_float<BS_F32>(uint32_t b) { return __uint_as_float(b); }

template <int DT>
struct DTraits {
  using raw_t = uint16_t;
  static constexpr int kBytes = 2;
};
template <>
struct DTraits<BS_F32> {
  using raw_t = uint32_t;
  static constexpr int kBytes = 4;
};

__device__ __forceinline__ uint32_t lds_u16(uint32_t saddr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ void lds_v4(uint32_t saddr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(saddr));
}
__device__ __forceinline__ void sts_u32(uint32_t saddr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(saddr), "r"(v));
}
__device__ __forceinline__ void sts_u16(uint32_t saddr, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(saddr), "h"(v));
}
__device__ __forceinline__ void sts_v4(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c), "r"(d));
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace bsk
