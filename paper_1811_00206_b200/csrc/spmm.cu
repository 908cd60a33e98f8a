// spmm.cu: bs_spmm, Y = W_bs · X for a batch of N columns (Fig. `benchmark`(b), batch 8).
//
// K6, tensor cores (f16/bf16, SPMM layout, B | 64). Per CTA: one 128-row tile of W, up to 256 batch
// columns, and a contiguous range of the 64-column K chunks (split-K over a thread-block cluster).
//   - Warp 0, one lane: per chunk, a bulk copy of the packed (tile, chunk) blob (docs/layout.md SPMM)
//     and a TMA tensor copy of the BN × 64 X tile (128-byte swizzle, zero fill past N and K) into an
//     NSB-stage ring (mbarrier complete_tx), 4..16 stages deep.
//   - Warps 2..17: two groups of 8 warps, alternating chunks, rebuild the dense 128 × 64 A tile in one
//     of NA = 4 buffers: a linear zero fill, a named barrier, then an entry-parallel scatter: thread
//     t takes blob entries t, t+256, ... (consecutive lanes read consecutive values and indices:
//     conflict-free; four entries' loads in flight before their stores) and stores each value
//     at (row, (entry's block)·B + index) of the K-major SWIZZLE_128B tile. The balanced rows give every
//     chunk the same entry count per row, so (row, block) follow from the entry number by a
//     running quotient. fence.proxy.async publishes the stores to the tensor core.
//   - Warp 1, one lane: 4 × tcgen05.mma.cta_group::1.kind::f16 (M = 128, N = BN, K = 16) per chunk into
//     the fp32 accumulator in tensor memory; tcgen05.commit frees the blob/X stage and the A buffer.
//   - Epilogue: tcgen05.ld (32x32b) → Y [N][M]. With split-K (cluster of S CTAs along K), each CTA
//     parks its fp32 partial tile in shared memory, and after a cluster barrier CTA j sums slice j of
//     the tile over the S partials in rank order through distributed shared memory (ld.shared::cluster).
// S depends only on M and K (never on N), and the accumulation order over K is fixed, so column n of Y
// depends only on column n of X: batch sharding reproduces the unsharded columns bit for bit.
// Dense flops are spent on the decompressed tile; only packed bytes cross HBM.
//
// CUDA-core fallback (f32, B not dividing 64, unaligned X): one thread per (row, batch column) walks
// the row's blobs in chunk order with fp32 FMAs.
#include "bs_common.cuh"
#include "bs_device.cuh"
#include "bs_tc.cuh"

namespace {

using namespace bsk_tc;

constexpr int BM = 128;          // rows per tile (MMA M)
constexpr int KC = 64;           // columns per chunk (one SWIZZLE_128B atom of 16-bit values)
constexpr int NA = 4;            // dense A tile buffers
constexpr int kMaxStages = 16;   // blob + X tile ring stages (runtime NSB: even, 4..16)
constexpr int kDecomp = 256;     // threads per decompress group (8 warps)
constexpr int kGroups = 2;       // decompress groups, alternating chunks
constexpr int kThreads = 64 + kGroups * kDecomp;
constexpr int kMaxCluster = 8;   // split-K factor (portable cluster size)

struct TcArgs {
  const uint8_t* W;   // packed SPMM layout
  void* Y;
  int64_t M, NB, N, ldy;
  int B, k, CB, NC;   // block width, kept per block, blocks per chunk, chunks per row tile
  int64_t tile_stride;
  int BN, S, NSB;     // batch columns per CTA (multiple of 16), split-K cluster size, ring stages
  int blob_max;       // bytes of a full blob (128 rows, CB blocks)
  uint32_t idesc;
  int tmem_cols;
};

template <int DT>
__global__ void __launch_bounds__(kThreads, 1) spmm_tc_kernel(const __grid_constant__ CUtensorMap tX, TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[2 * kMaxStages + 2 * NA + 1];
  __shared__ uint32_t tmem_holder;
  __shared__ uint8_t ctab[64];  // entry number within a row's chunk run -> block offset (entry / k)·B
  using raw_t = uint16_t;
  constexpr int ES = 2;
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int NSB = a.NSB;
  const uint32_t sA = smem_u32(smem);                          // NA × 16 KB dense A tiles
  const uint32_t XSZ = (uint32_t)a.BN * 128;                   // X tile: BN rows × 128 B
  const uint32_t sX = sA + NA * BM * 128;                      // NSB × XSZ
  const uint32_t sR = sX + (uint32_t)NSB * XSZ;                // NSB × blob_max
  const uint32_t full = smem_u32(&bars[0]), empty = smem_u32(&bars[kMaxStages]);
  const uint32_t a_full = smem_u32(&bars[2 * kMaxStages]), a_empty = smem_u32(&bars[2 * kMaxStages + NA]);
  const uint32_t acc_full = smem_u32(&bars[2 * kMaxStages + 2 * NA]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.S;
  const int rank = S > 1 ? (int)cluster_rank() : 0;
  const int64_t tile = blockIdx.x / S;
  const int64_t m0 = tile * BM;
  const int64_t mt = (a.M - m0) < BM ? (a.M - m0) : BM;
  const int64_t n0 = (int64_t)blockIdx.y * a.BN;
  const int c0 = (int)((int64_t)rank * a.NC / S), c1 = (int)((int64_t)(rank + 1) * a.NC / S);
  const int nloc = c1 - c0;  // >= 1 (S <= NC)
  const uint8_t* tile_base = a.W + tile * a.tile_stride;
  const int k = a.k;
  auto blob_bytes = [&](int64_t cb) {
    return (uint32_t)(bsk::align_up(mt * cb * k * ES, 16) + bsk::align_up(mt * cb * k, 16));
  };
  const uint32_t blobCB = blob_bytes(a.CB);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSB; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
    }
    for (int s = 0; s < NA; ++s) {
      mbar_init(a_full + 8 * s, kDecomp);  // one decompress group
      mbar_init(a_empty + 8 * s, 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x >= 64 && threadIdx.x < 128) {
    const int q = threadIdx.x - 64;
    ctab[q] = (uint8_t)(q < a.CB * k ? (q / k) * a.B : 0);
  }
  if (warp == 1) {  // tensor-memory accumulator: 128 lanes × tmem_cols fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_d = tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ---- producer
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tX) : "memory");
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nloc; ++i) {
        const int c = c0 + i;
        if (i >= NSB) mbar_wait(empty + 8 * s, ph ^ 1u);
        const int64_t cb = (a.NB - (int64_t)a.CB * c) < a.CB ? (a.NB - (int64_t)a.CB * c) : a.CB;
        const uint32_t bytes = blob_bytes(cb);
        mbar_expect_tx(full + 8 * s, bytes + XSZ);
        bulk_g2s(sR + (uint32_t)s * (uint32_t)a.blob_max, tile_base + (int64_t)c * blobCB, bytes, full + 8 * s);
        tma_2d(sX + (uint32_t)s * XSZ, &tX, c * KC, (int)n0, full + 8 * s);
        if (++s == NSB) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nloc; ++i) {
        const int ab = i & (NA - 1);
        mbar_wait(full + 8 * s, ph);
        mbar_wait(a_full + 8 * ab, (uint32_t)(i / NA) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t da = sw128_desc(sA + (uint32_t)ab * BM * 128), db = sw128_desc(sX + (uint32_t)s * XSZ);
#pragma unroll
        for (int kk = 0; kk < KC / 16; ++kk) {
          const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
          asm volatile(
              "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
              "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(a.idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(empty + 8 * s)
                     : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(a_empty + 8 * ab)
                     : "memory");
        if (++s == NSB) { s = 0; ph ^= 1u; }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(acc_full)
                   : "memory");
    }
  } else {
    // ---- decompress: group grp (8 warps) rebuilds chunks i = grp, grp + 2, ...; thread t = 0..255.
    // Entry e of a chunk sits in row e / rk at run position e % rk (rk = entries per row); thread t
    // walks e = t, t + 256, ... keeping (row, position) by a running quotient. Full chunks and the
    // last (shorter) chunk of the row tile each get their constants once.
    const int grp = (threadIdx.x - 64) / kDecomp, t = (threadIdx.x - 64) % kDecomp;
    struct CG {
      int rk, dq, dr, r0, e0, n_e, ioff;
    };
    auto mk = [&](int rk) {
      CG g;
      g.rk = rk; g.dq = kDecomp / rk; g.dr = kDecomp % rk; g.r0 = t / rk; g.e0 = t % rk;
      g.n_e = (int)mt * rk; g.ioff = (int)bsk::align_up((int64_t)g.n_e * ES, 16);
      return g;
    };
    const CG gF = mk(a.CB * k), gL = mk((int)(a.NB - (int64_t)a.CB * (a.NC - 1)) * k);
    const int ilast = a.NC - 1 - c0;  // local index of the row tile's last chunk (may be >= nloc)
    uint8_t* const ring = smem + (sR - sA);
    int s = grp;  // ring stage of chunk i (NSB is even, so group grp keeps stages of its parity)
    uint32_t ph = 0;
    for (int i = grp; i < nloc; i += kGroups) {
      const int ab = i & (NA - 1);
      const uint32_t aph = (uint32_t)(i / NA) & 1u;
      const uint32_t aT = sA + (uint32_t)ab * BM * 128;
      uint8_t* const aTp = smem + ab * BM * 128;
      if (i >= NA) mbar_wait(a_empty + 8 * ab, aph ^ 1u);  // MMA done with this A tile
#pragma unroll
      for (int q = 0; q < 4; ++q) bsk::sts_v4(aT + q * 4096 + t * 16, 0u, 0u, 0u, 0u);
      const CG& G = i == ilast ? gL : gF;
      const int rk = G.rk, dq = G.dq, dr = G.dr, n_e = G.n_e;
      int r = G.r0, rem = G.e0;
      mbar_wait(full + 8 * s, ph);
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(kDecomp) : "memory");  // zero fill before any scatter
      const uint8_t* blob = ring + s * a.blob_max;
      const uint16_t* bv = (const uint16_t*)blob;
      const uint8_t* bi = blob + G.ioff;
      for (int e0 = t; e0 < n_e; e0 += 4 * kDecomp) {
        uint16_t w[4];
        uint8_t o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // loads first: four entries in flight
          const int e = e0 + u * kDecomp;
          w[u] = e < n_e ? bv[e] : (uint16_t)0;
          o[u] = e < n_e ? bi[e] : (uint8_t)0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (e0 + u * kDecomp < n_e) {
            const uint32_t col = (uint32_t)ctab[rem] + o[u];
            *(uint16_t*)(aTp + sw128_off((uint32_t)r, col)) = w[u];
          }
          rem += dr;
          r += dq;
          if (rem >= rk) { rem -= rk; ++r; }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> tensor core
      mbar_arrive(a_full + 8 * ab);
      s += kGroups;
      if (s >= NSB) { s -= NSB; ph ^= 1u; }
    }
    // ---- epilogue: TMEM -> registers. Warp w reads lane quarter w % 4 (rows 32·(w % 4) + lane) and
    // column part (w - 2) / 4 of NP parts.
    mbar_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int q = warp & 3, part = (warp - 2) >> 2;
    const int NP = a.BN % 32 == 0 ? 4 : 2;  // parts of BN / NP columns, a multiple of 8
    const int m = 32 * q + lane;
    float* red = (float*)smem;  // split-K partial tile [BN][128] (the rings are idle now)
    if (part < NP) {
      const int pw = a.BN / NP;
      for (int nb = part * pw; nb < (part + 1) * pw; nb += 8) {
        uint32_t rr[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(rr[0]), "=r"(rr[1]), "=r"(rr[2]), "=r"(rr[3]), "=r"(rr[4]), "=r"(rr[5]), "=r"(rr[6]), "=r"(rr[7])
                     : "r"(tmem_d + ((uint32_t)(32 * q) << 16) + (uint32_t)nb));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (S > 1) {
#pragma unroll
          for (int e = 0; e < 8; ++e) red[(nb + e) * BM + m] = __uint_as_float(rr[e]);
        } else if (m < mt) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int64_t ng = n0 + nb + e;
            if (ng < a.N) ((raw_t*)a.Y)[ng * a.ldy + m0 + m] = (raw_t)bsk::from_float<DT>(__uint_as_float(rr[e]));
          }
        }
      }
    }
  }
  if (S > 1) {
    cluster_sync_all();  // every partial tile is parked
    if (warp >= 2) {
      const int t = threadIdx.x - 64;
      const int U = a.BN * BM / 4;  // float4 units of the tile
      const int u0 = (int)((int64_t)rank * U / S), u1 = (int)((int64_t)(rank + 1) * U / S);
      for (int u = u0 + t; u < u1; u += kGroups * kDecomp) {
        const uint32_t la = sA + (uint32_t)u * 16;
        float4 v = ld_cluster_f4(la, 0);
        for (int p = 1; p < S; ++p) {  // fixed rank order: partials over consecutive K ranges
          const float4 w = ld_cluster_f4(la, (uint32_t)p);
          v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
        }
        const int n = u >> 5, row = (u & 31) * 4;
        const int64_t ng = n0 + n;
        if (ng < a.N) {
          raw_t* yp = (raw_t*)a.Y + ng * a.ldy + m0 + row;
          const float f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (row + e < mt) yp[e] = (raw_t)bsk::from_float<DT>(f[e]);
        }
      }
    }
    cluster_sync_all();  // peers' shared memory stays alive until every slice is read
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

// Split-K factor for a row-tile count and chunk count: enough clusters to cover the SMs once, never
// more chunks than exist. Depends only on (M, K), never on N.
int split_k(int64_t tiles, int64_t NC) {
  int64_t S = bsk::dev_props().sms / tiles;
  if (S > kMaxCluster) S = kMaxCluster;
  if (S > NC / 6) S = NC / 6;  // at least 6 chunks per CTA: fixed costs stay amortised
  return S < 1 ? 1 : (int)S;
}

template <int DT>
cudaError_t launch_tc(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx, void* Y,
                      int64_t ldy, cudaStream_t s) {
  if (((uintptr_t)X & 15) != 0 || (ldx % 8) != 0) return cudaErrorNotSupported;  // TMA: 16-byte rows
  TcArgs a;
  a.W = (const uint8_t*)packed;
  a.Y = Y;
  a.M = g.M; a.NB = g.NB; a.N = N; a.ldy = ldy;
  a.B = g.B; a.k = g.k; a.CB = g.V; a.NC = (int)g.NBf; a.tile_stride = g.offB;
  a.blob_max = (int)(bsk::align_up((int64_t)BM * g.V * g.k * 2, 16) + bsk::align_up((int64_t)BM * g.V * g.k, 16));
  a.S = split_k(g.P, g.NBf);
  auto kern = spmm_tc_kernel<DT>;
  static int static_smem = -1;
  if (static_smem < 0) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             bsk::dev_props().smem_optin - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
    static_smem = (int)fa.sharedSizeBytes;
  }
  // NA dense A tiles + NSB stages of (X tile, blob): BN as large as 4 stages allow (<= 256), then as
  // many stages as fit (deep rings keep enough bytes in flight when blobs are small)
  const int64_t avail = bsk::dev_props().smem_optin - static_smem - 1024;  // 1024: alignment slack
  const int64_t ring = avail - (int64_t)NA * BM * 128;
  int64_t bn_max = ((ring / 4 - a.blob_max) / 128) / 16 * 16;
  if (bn_max > 256) bn_max = 256;
  if (bn_max < 16) return cudaErrorNotSupported;
  int64_t BN = (N + 15) / 16 * 16;
  if (BN > bn_max) BN = bn_max;
  a.BN = (int)BN;
  a.idesc = idesc_f16(DT == BS_BF16, BM, (int)BN, false);
  int cols = 32;
  while (cols < BN) cols <<= 1;
  a.tmem_cols = cols;
  int64_t nsb = ring / (BN * 128 + a.blob_max);
  if (nsb > kMaxStages) nsb = kMaxStages;
  nsb &= ~1LL;  // even: each decompress group keeps to one stage parity
  if (nsb < 4) return cudaErrorNotSupported;
  a.NSB = (int)nsb;
  const int64_t smem = 1024 + (int64_t)NA * BM * 128 + nsb * (BN * 128 + a.blob_max);
  if (a.S > 1 && BN * BM * 4 > smem - 1024) return cudaErrorNotSupported;  // partial tile must fit
  CUtensorMap tX;
  if (!bsk_make_map_2d(&tX, DT, X, g.K, N, ldx, KC, (int)BN)) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(g.P * a.S), (unsigned)((N + BN - 1) / BN));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tX, a);
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
    cudaError_t e = g.dt == BS_BF16 ? launch_tc<BS_BF16>(g, packed, X, N, ldx, Y, ldy, s)
                                    : launch_tc<BS_F16>(g, packed, X, N, ldx, Y, ldy, s);
    if (e != cudaErrorNotSupported) return e;
  }
  switch (g.dt) {
    case BS_F32: return g.is == 1 ? launch_cc<BS_F32, 1>(g, packed, X, N, ldx, Y, ldy, s) : launch_cc<BS_F32, 2>(g, packed, X, N, ldx, Y, ldy, s);
    case BS_F16: return g.is == 1 ? launch_cc<BS_F16, 1>(g, packed, X, N, ldx, Y, ldy, s) : launch_cc<BS_F16, 2>(g, packed, X, N, ldx, Y, ldy, s);
    default: return g.is == 1 ? launch_cc<BS_BF16, 1>(g, packed, X, N, ldx, Y, ldy, s) : launch_cc<BS_BF16, 2>(g, packed, X, N, ldx, Y, ldy, s);
  }
}
