// spmm.cu: bs_spmm, Y = W_bs · X for a batch of N columns (Fig. `benchmark`(b), batch 8).
//
// K6, tensor cores (f16/bf16, SPMM layout, B | 64). Per CTA: one 128-row tile of W and up to 256
// batch columns, streamed over K in chunks of 64 columns.
//   - A producer lane bulk-copies each (tile, chunk) blob of packed W (docs/layout.md SPMM) into a
//     shared-memory ring (cp.async.bulk + mbarrier).
//   - Four "decompress" warps rebuild the dense 128×64 A tile in shared memory. Thread r owns row r:
//     it clears the row, then scatters the row's kept values to their columns (the paper's balanced
//     rows make this the same work for every thread). The same warps stage the 64-column
//     chunk of X as the N×64 B tile. Both tiles are in the canonical K-major SWIZZLE_128B layout of
//     the UMMA descriptors. A fence.proxy.async makes the stores visible to the tensor core.
//   - One elected thread issues tcgen05.mma.cta_group::1.kind::f16 (M = 128, N = padded batch,
//     K = 16, ×4 per chunk) with the fp32 accumulator in tensor memory. A/B are double-buffered, and
//     tcgen05.commit → mbarrier hands buffers back.
//   - The epilogue warps read the accumulator with tcgen05.ld (32x32b) and store Y rows [N][M] in D.
// Dense flops are spent on the decompressed tile, but only packed bytes cross HBM.
// Column n of Y depends only on column n of X, and the accumulation order over K is fixed.
//
// CUDA-core fallback (f32, or B not dividing 64): one thread per (row, batch column) walks the row's
// blobs in chunk order with fp32 FMAs.
#include "bs_common.cuh"
#include "bs_device.cuh"

namespace {

constexpr int BM = 128;     // rows per tile (MMA M)
constexpr int KC = 64;      // columns per chunk (one SWIZZLE_128B atom of 16-bit values)
constexpr int NSB = 4;      // blob ring stages
constexpr int kThreads = 192;  // warp 0 producer, warp 1 MMA/TMEM, warps 2..5 decompress + epilogue

struct TcArgs {
  const uint8_t* W;   // packed SPMM layout
  const void* X;
  void* Y;
  int64_t M, K, NB, N, ldx, ldy;
  int B, k, CB, NC;   // block width, kept per block, blocks per chunk, chunks
  int is;             // index bytes
  int64_t tile_stride;
  int BN;             // padded batch columns handled per CTA (multiple of 16, <= 256)
  int blob_max;       // bytes of one full blob (128 rows, CB blocks)
  int xvec;           // X rows 16-byte aligned (LDG.128 staging)
  uint32_t idesc;     // tcgen05 instruction descriptor
  int tmem_cols;
};

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
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: 8-row x 128-byte atoms, SBO = 1024 B between
// 8-row groups, LBO unused (1), version 1 (bits 46-47), layout type 2 (bits 61-63).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
// byte offset of element (row, col) in a K-major SWIZZLE_128B tile of 64 16-bit columns
__device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t col) {
  return row * 128 + ((((col >> 3) ^ (row & 7)) & 7) << 4) + (col & 7) * 2;
}

template <int DT, int IS>
__global__ void __launch_bounds__(kThreads, 1) spmm_tc_kernel(TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[2 * NSB + 5];
  __shared__ uint32_t tmem_holder;
  using raw_t = uint16_t;
  constexpr int ES = 2;
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sA = smem_u32(smem);                         // 2 x 16 KB
  const uint32_t sB = sA + 2 * BM * 128;                      // 2 x BN*128
  const uint32_t sR = sB + 2 * a.BN * 128;                    // NSB x blob_max
  const uint32_t b_full = smem_u32(&bars[0]), b_empty = smem_u32(&bars[NSB]);
  const uint32_t a_full = smem_u32(&bars[2 * NSB]), m_done = smem_u32(&bars[2 * NSB + 2]);
  const uint32_t acc_full = smem_u32(&bars[2 * NSB + 4]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile = blockIdx.x;
  const int64_t m0 = tile * BM;
  const int64_t mt = (a.M - m0) < BM ? (a.M - m0) : BM;
  const int64_t n0 = (int64_t)blockIdx.y * a.BN;
  const uint8_t* tile_base = a.W + tile * a.tile_stride;
  auto blob_bytes = [&](int64_t cb) {
    return (uint32_t)(bsk::align_up(mt * cb * a.k * ES, 16) + bsk::align_up(mt * cb * a.k * IS, 16));
  };
  const uint32_t blobCB = blob_bytes(a.CB);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSB; ++s) {
      mbar_init(b_full + 8 * s, 1);
      mbar_init(b_empty + 8 * s, 128);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(a_full + 8 * s, 128);
      mbar_init(m_done + 8 * s, 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // tensor-memory accumulator: 128 lanes x tmem_cols fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_d = tmem_holder;

  if (warp == 0) {
    // ---- producer: bulk-copy blobs (tile, chunk) into the ring
    if (lane == 0) {
      for (int c = 0; c < a.NC; ++c) {
        const int s = c % NSB;
        if (c >= NSB) mbar_wait(b_empty + 8 * s, (uint32_t)(((c / NSB) - 1) & 1));
        const int64_t cb = (a.NB - (int64_t)a.CB * c) < a.CB ? (a.NB - (int64_t)a.CB * c) : a.CB;
        const uint32_t bytes = blob_bytes(cb);
        mbar_expect_tx(b_full + 8 * s, bytes);
        bulk_g2s(sR + s * a.blob_max, tile_base + (int64_t)c * blobCB, bytes, b_full + 8 * s);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: one elected thread
    if (lane == 0) {
      for (int c = 0; c < a.NC; ++c) {
        const int ab = c & 1;
        mbar_wait(a_full + 8 * ab, (uint32_t)((c >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t da = sw128_desc(sA + ab * BM * 128), db = sw128_desc(sB + ab * a.BN * 128);
#pragma unroll
        for (int kk = 0; kk < KC / 16; ++kk) {
          const uint32_t acc = (c > 0 || kk > 0) ? 1u : 0u;
          // advance 16 elements (32 bytes = 2 units of 16 B) along K inside the swizzle atom
          asm volatile(
              "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
              "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(a.idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(m_done + 8 * ab)
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(acc_full)
                   : "memory");
    }
  } else {
    // ---- decompress + stage X (128 threads, u = row of the tile)
    const int u = threadIdx.x - 64;
    for (int c = 0; c < a.NC; ++c) {
      const int s = c % NSB, ab = c & 1;
      const int64_t cb = (a.NB - (int64_t)a.CB * c) < a.CB ? (a.NB - (int64_t)a.CB * c) : a.CB;
      if (c >= 2) mbar_wait(m_done + 8 * ab, (uint32_t)(((c >> 1) - 1) & 1));  // MMA done with buffer ab
      mbar_wait(b_full + 8 * s, (uint32_t)((c / NSB) & 1));
      // A row u: clear, then scatter the row's cb·k kept values
      const uint32_t arow = sA + ab * BM * 128;
#pragma unroll
      for (int j = 0; j < 8; ++j) bsk::sts_v4(arow + u * 128 + j * 16, 0u, 0u, 0u, 0u);
      if (u < mt) {
        const uint32_t bv = sR + s * a.blob_max;
        const uint32_t bi = bv + (uint32_t)bsk::align_up(mt * cb * a.k * ES, 16);
        const int n_e = (int)cb * a.k;
        for (int e = 0; e < n_e; ++e) {
          const uint32_t pos = (uint32_t)u * n_e + e;
          const uint32_t w = bsk::lds_u16(bv + pos * 2);
          uint32_t o;
          if (IS == 1) {
            uint16_t b8;
            asm volatile("ld.shared.u8 %0, [%1];" : "=h"(b8) : "r"(bi + pos));
            o = b8;
          } else {
            o = bsk::lds_u16(bi + pos * 2);
          }
          const uint32_t col = (uint32_t)(e / a.k) * a.B + o;
          bsk::sts_u16(arow + sw128_off(u, col), (uint16_t)w);
        }
      }
      // B tile: X columns [c·64, c·64 + 64) of batch rows n0 .. n0 + BN (zeros outside X)
      const uint32_t brow = sB + ab * a.BN * 128;
      const int64_t kc0 = (int64_t)c * KC;
      const int64_t kvalid = (a.K - kc0) < KC ? (a.K - kc0) : KC;
      for (int p = u; p < a.BN * 8; p += 128) {
        const int n = p >> 3, j = p & 7;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        const int64_t ng = n0 + n;
        if (ng < a.N) {
          const raw_t* xs = (const raw_t*)a.X + ng * a.ldx + kc0 + j * 8;
          if (a.xvec && j * 8 + 8 <= kvalid) {
            v = __ldg((const uint4*)xs);
          } else {
            uint32_t h[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) h[e] = (j * 8 + e < kvalid) ? (uint32_t)__ldg(xs + e) : 0u;
            v = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
          }
        }
        bsk::sts_v4(brow + n * 128 + ((((uint32_t)j ^ (uint32_t)(n & 7)) & 7) << 4), v.x, v.y, v.z, v.w);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> tensor core
      mbar_arrive(a_full + 8 * ab);
      mbar_arrive(b_empty + 8 * s);
    }
    // ---- epilogue: TMEM -> registers -> Y (row m = 32·(warp % 4) + lane)
    mbar_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int q = warp & 3;
    const int64_t m = 32 * q + lane;
    for (int nb = 0; nb < a.BN; nb += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tmem_d + ((uint32_t)(32 * q) << 16) + (uint32_t)nb));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (m < mt) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int64_t ng = n0 + nb + e;
          if (ng < a.N) ((raw_t*)a.Y)[ng * a.ldy + m0 + m] = (raw_t)bsk::from_float<DT>(__uint_as_float(r[e]));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(a.tmem_cols));
  }
}

// CUDA-core fallback on the SPMM layout: thread per (row, batch column), chunks in order.
template <int DT, int IS>
__global__ void spmm_cc_kernel(const uint8_t* __restrict__ W, const void* __restrict__ X, void* __restrict__ Y,
                               int64_t M, int64_t NB, int64_t N, int64_t ldx, int64_t ldy, int B, int k, int CB,
                               int64_t tile_stride) {
  using raw_t = typename bsk::DTraits<DT>::raw_t;
  constexpr int ES = bsk::DTraits<DT>::kBytes;
  const int64_t total = M * N;
  const int64_t NC = (NB + CB - 1) / CB;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = g % M, n = g / M;
    const int64_t t = r / BM, rl = r - t * BM;
    const int64_t mt = (M - BM * t) < BM ? (M - BM * t) : BM;
    const int64_t blobCB = bsk::align_up(mt * CB * k * ES, 16) + bsk::align_up(mt * CB * k * IS, 16);
    const raw_t* xn = (const raw_t*)X + n * ldx;
    float acc = 0.f;
    for (int64_t c = 0; c < NC; ++c) {
      const int64_t cb = (NB - CB * c) < CB ? (NB - CB * c) : CB;
      const uint8_t* blob = W + t * tile_stride + c * blobCB;
      const raw_t* bv = (const raw_t*)blob;
      const uint8_t* bi = blob + bsk::align_up(mt * cb * k * ES, 16);
      for (int64_t e = rl * cb * k; e < (rl + 1) * cb * k; ++e) {
        const int64_t j = (e - rl * cb * k) / k;
        const uint32_t o = IS == 1 ? bi[e] : ((const uint16_t*)bi)[e];
        const int64_t col = (CB * c + j) * B + o;
        bsk::fma_acc<DT>(acc, bv[e], xn[col]);
      }
    }
    ((raw_t*)Y)[n * ldy + r] = (raw_t)bsk::from_float<DT>(acc);
  }
}

template <int DT, int IS>
cudaError_t launch_tc(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx, void* Y,
                      int64_t ldy, cudaStream_t s) {
  TcArgs a;
  a.W = (const uint8_t*)packed;
  a.X = X;
  a.Y = Y;
  a.M = g.M; a.K = g.K; a.NB = g.NB; a.N = N; a.ldx = ldx; a.ldy = ldy;
  a.B = g.B; a.k = g.k; a.CB = g.V; a.NC = (int)g.NBf; a.is = g.is; a.tile_stride = g.offB;
  int64_t BN = (N + 15) / 16 * 16;
  if (BN > 256) BN = 256;
  a.BN = (int)BN;
  a.blob_max = (int)(bsk::align_up((int64_t)BM * g.V * g.k * 2, 16) + bsk::align_up((int64_t)BM * g.V * g.k * g.is, 16));
  a.xvec = (((uintptr_t)X & 15) == 0) && (ldx % 8 == 0);
  const uint32_t fmt = DT == BS_BF16 ? 1u : 0u;
  a.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  int cols = 32;
  while (cols < BN) cols <<= 1;
  a.tmem_cols = cols;
  const int64_t smem = 1024 + 2LL * BM * 128 + 2LL * BN * 128 + (int64_t)NSB * a.blob_max;
  auto kern = spmm_tc_kernel<DT, IS>;
  static int configured = 0;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         bsk::dev_props().smem_optin - 1024);
    if (e != cudaSuccess) return e;
    configured = 1;
  }
  if (smem > bsk::dev_props().smem_optin - 1024) return cudaErrorNotSupported;
  dim3 grid((unsigned)g.P, (unsigned)((N + BN - 1) / BN));
  kern<<<grid, kThreads, (size_t)smem, s>>>(a);
  return cudaGetLastError();
}

template <int DT, int IS>
cudaError_t launch_cc(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx, void* Y,
                      int64_t ldy, cudaStream_t s) {
  const int64_t total = g.M * N;
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)bsk::dev_props().sms * 32) blocks = (int64_t)bsk::dev_props().sms * 32;
  spmm_cc_kernel<DT, IS><<<(unsigned)blocks, 256, 0, s>>>((const uint8_t*)packed, X, Y, g.M, g.NB, N, ldx, ldy, g.B,
                                                          g.k, g.V, g.offB);
  return cudaGetLastError();
}

}  // namespace

// Returns cudaErrorNotSupported when the caller should fall back to column-at-a-time SpMV
// (SPMV layout).
cudaError_t bsk_launch_spmm(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx, void* Y,
                            int64_t ldy, cudaStream_t s) {
  if (g.layout != BS_LAYOUT_SPMM) return cudaErrorNotSupported;
  if (g.k == 0) {  // W_bs = 0
    for (int64_t n = 0; n < N; ++n) {
      cudaError_t e = cudaMemsetAsync((char*)Y + (size_t)(n * ldy) * g.es, 0, (size_t)g.M * g.es, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  const bool tc = g.es == 2 && (64 % g.B) == 0;
  if (tc) {
    cudaError_t e = g.dt == BS_BF16 ? (g.is == 1 ? launch_tc<BS_BF16, 1>(g, packed, X, N, ldx, Y, ldy, s)
                                                 : launch_tc<BS_BF16, 2>(g, packed, X, N, ldx, Y, ldy, s))
                                    : (g.is == 1 ? launch_tc<BS_F16, 1>(g, packed, X, N, ldx, Y, ldy, s)
                                                 : launch_tc<BS_F16, 2>(g, packed, X, N, ldx, Y, ldy, s));
    if (e != cudaErrorNotSupported) return e;
  }
  switch (g.dt) {
    case BS_F32: return g.is == 1 ? launch_cc<BS_F32, 1>(g, packed, X, N, ldx, Y, ldy, s) : launch_cc<BS_F32, 2>(g, packed, X, N, ldx, Y, ldy, s);
    case BS_F16: return g.is == 1 ? launch_cc<BS_F16, 1>(g, packed, X, N, ldx, Y, ldy, s) : launch_cc<BS_F16, 2>(g, packed, X, N, ldx, Y, ldy, s);
    default: return g.is == 1 ? launch_cc<BS_BF16, 1>(g, packed, X, N, ldx, Y, ldy, s) : launch_cc<BS_BF16, 2>(g, packed, X, N, ldx, Y, ldy, s);
  }
}
