// bs_tc.cuh: Blackwell async-pipeline helpers shared by the tensor-core kernels (spmm.cu K6,
// spmm24.cu K5): mbarriers, bulk / tensor (TMA) copies, UMMA shared-memory descriptors, tensor maps.
#pragma once

#include <cuda.h>
#include <stdint.h>

#include "bs_common.cuh"

namespace bsk_tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(bar), "r"(parity)
                 : "memory");
  }
}

// global -> shared bulk copy (16-byte aligned source, destination and size), completes on `bar`
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// 2-D tensor copy (TMA) of one box at coordinates (c0 = inner / column, c1 = row)
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: 8-row × 128-byte atoms, SBO = 1024 B between
// 8-row groups, LBO unused (1), version 1 (bits 46-47), layout type 2 (bits 61-63). Advancing K by 16
// 16-bit elements inside the atom adds 2 (32 bytes >> 4) to the start address field.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}

// byte offset of 16-bit element (row, col) in a K-major SWIZZLE_128B tile of 64 columns
__device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t col) {
  return row * 128 + ((((col >> 3) ^ (row & 7)) & 7) << 4) + (col & 7) * 2;
}

// kind::f16 instruction descriptor: fp32 accumulate (bit 4), A/B format f16 (0) or bf16 (1) at bits
// 7 / 10, K-major A and B, N >> 3 at bit 17, M >> 4 at bit 24; bit 2 selects the sparse (.sp) form.
__host__ __device__ inline uint32_t idesc_f16(int dt_bf16, int M, int N, bool sparse) {
  const uint32_t fmt = dt_bf16 ? 1u : 0u;
  return (sparse ? (1u << 2) : 0u) | (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// Thread-block clusters (split-K partial sums through distributed shared memory).
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float4 ld_cluster_f4(uint32_t local_addr, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(ra) : "memory");
  return v;
}

// CTA pairs (cta_group::2): the address of `local_addr` in CTA `rank` of the cluster, and an mbarrier
// arrive there. Relaxed: a release at cluster scope compiles to a MEMBAR that waits for every load the
// thread has in flight (the metadata prefetch: ncu showed 46 % membar stalls); the arrive only counts,
// and the tensor-memory stores it announces are ordered by tcgen05.wait::st + fence::before_thread_sync.
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local_addr, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(rank));
  return ra;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-D tensor copy into this CTA's shared memory that completes on an mbarrier of either CTA of the pair
__device__ __forceinline__ void tma_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}

// 4-D tensor copy in im2col mode (implicit im2col for convolution): a column of pixels × channels of an
// NHWC tensor starting at base pixel (w, h, n), channel c, each pixel displaced by the filter offset
// (dw, dh); pixels outside the tensor read as zeros
__device__ __forceinline__ void tma_im2col_4d(uint32_t dst, const CUtensorMap* map, int c, int w, int h, int n,
                                              uint16_t dw, uint16_t dh, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(dst),
      "l"((uint64_t)map), "r"(c), "r"(w), "r"(h), "r"(n), "r"(bar), "h"(dw), "h"(dh)
      : "memory");
}

// Layer epilogue of the tensor-core products (bs_conv2d, bs_spmm_fused): v + bias[row] (16-bit D), then
// ReLU / sigmoid / tanh (bs_act), in fp32 before the one rounding; the expressions of bs_spmv_fused.
template <int DT>
__device__ __forceinline__ float act_epilogue(float v, const void* bias, int act, int64_t row) {
  if (bias) v += bsk::to_float<DT>(__ldg((const uint16_t*)bias + row));
  switch (act) {
    case BS_ACT_RELU: return fmaxf(v, 0.f);
    case BS_ACT_SIGMOID: return 1.f / (1.f + expf(-v));
    case BS_ACT_TANH: return tanhf(v);
    default: return v;
  }
}

// im2col copy completing on an mbarrier of either CTA of a pair (the K5 CTA-pair kernel)
__device__ __forceinline__ void tma_im2col_4d_pair(uint32_t dst, const CUtensorMap* map, int c, int w, int h, int n,
                                                   uint16_t dw, uint16_t dh, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(dst),
      "l"((uint64_t)map), "r"(c), "r"(w), "r"(h), "r"(n), "r"(bar_cluster), "h"(dw), "h"(dh)
      : "memory");
}

// Implicit im2col geometry of a tensor-core SpMM over a convolution (bs_conv2d): the X column starting at
// pixel p of K-columns [col0, col0 + 64) is 64 channels of one filter tap
struct ConvX {
  int conv, C, KW, OW, OHW, pad;
  __device__ __forceinline__ void coords(int64_t p, int col0, int& c, int& w, int& h, int& n, uint16_t& dw,
                                         uint16_t& dh) const {
    const int tap = col0 / C;
    c = col0 - tap * C;
    const int dy = tap / KW, dx = tap - dy * KW;
    n = (int)(p / OHW);
    const int pix = (int)(p - (int64_t)n * OHW);
    const int oy = pix / OW, ox = pix - oy * OW;
    w = ox - pad;
    h = oy - pad;
    dw = (uint16_t)dx;
    dh = (uint16_t)dy;
  }
};

}  // namespace bsk_tc

// Im2col tensor map of an NHWC 16-bit tensor [Nimg][H][W][C] for a kh × kw, stride-1 convolution with
// symmetric padding `pad`: columns of `pixels` output positions × 64 channels, 128-byte swizzle (the X tile
// layout of K6). Returns false if the driver entry point is missing or the encoding is rejected.
bool bsk_make_map_im2col(CUtensorMap* m, int dt, const void* in, int64_t Nimg, int64_t H, int64_t W, int64_t C, int kh,
                         int kw, int pad, int pixels);

// 2-D tensor map of a row-major [rows][cols] 16-bit matrix (dt f16 / bf16) with row stride `ld`
// elements; box of bc columns × br rows, 128-byte swizzle, zero fill out of bounds. Returns false if
// the driver entry point is missing or the encoding is rejected (alignment, strides).
bool bsk_make_map_2d(CUtensorMap* m, int dt, const void* base, int64_t cols, int64_t rows, int64_t ld, int bc, int br);
