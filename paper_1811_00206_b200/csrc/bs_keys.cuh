// bs_keys.cuh: the magnitude key of docs/layout.md "Canonical form", shared by the pruning kernels
// (prune.cu) and the pattern kernels (patterns.cu). The key of a value is its abs bit pattern as an
// unsigned integer, with every NaN folded onto one key just above +Inf: for IEEE formats the unsigned
// order of these keys is the |w| order, -0 and +0 tie, and all NaNs are equal and above everything.
#pragma once

#include <stdint.h>

#include "bs.h"

namespace bsk {

template <int DT>
struct KeyOf;
template <>
struct KeyOf<BS_F32> {
  using raw_t = uint32_t;
  static constexpr int kBits = 31;
  __host__ __device__ static constexpr uint32_t key(uint32_t u) {
    uint32_t a = u & 0x7fffffffu;
    return a > 0x7f800000u ? 0x7f800001u : a;
  }
};
template <>
struct KeyOf<BS_F16> {
  using raw_t = uint16_t;
  static constexpr int kBits = 15;
  __host__ __device__ static constexpr uint32_t key(uint32_t u) {
    uint32_t a = u & 0x7fffu;
    return a > 0x7c00u ? 0x7c01u : a;
  }
};
template <>
struct KeyOf<BS_BF16> {
  using raw_t = uint16_t;
  static constexpr int kBits = 15;
  __host__ __device__ static constexpr uint32_t key(uint32_t u) {
    uint32_t a = u & 0x7fffu;
    return a > 0x7f80u ? 0x7f81u : a;
  }
};

}  // namespace bsk
