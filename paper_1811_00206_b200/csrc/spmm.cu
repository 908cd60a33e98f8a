// spmm.cu: bs_spmm, Y = W_bs · X for a batch of N columns (Fig. `benchmark`(b), batch 8).
//
// K6, tensor cores (f16/bf16, SPMM layout, B | 64). Per CTA: one 128-row tile of W, up to 256 batch
// columns, and a contiguous range of the 64-column K chunks (split-K over a thread-block cluster).
//   - Warps 0..3, one lane each, chunks in turn: a bulk copy of the packed (tile, chunk) blob
//     (docs/layout.md SPMM) and a TMA tensor copy of the BN × 64 X tile (128-byte swizzle, zero fill
//     past N and K) into a ring of NSB = 4, 8, 12 or 16 stages (mbarrier complete_tx).
//   - Warps 6..21: four groups of 4 warps, chunks in turn, rebuild the dense 128 × 64 A tile in one of
//     NA = 4 or 8 buffers. A thread owns (row, block) units (at least 8 columns): it zero-fills the
//     unit's 16-byte pieces of the K-major SWIZZLE_128B tile, then stores each kept value at
//     (row, block·B + index). The balanced rows give every unit the same k entries per block,
//     contiguous in the blob. The same thread zero-fills and scatters, so no barrier is needed;
//     fence.proxy.async publishes the stores to the tensor core.
//   - Warps 4 and 5, one lane each, alternating chunks: 4 × tcgen05.mma.cta_group::1.kind::f16
//     (M = 128, N = BN, K = 16) per chunk into two fp32 accumulators in tensor memory (summed
//     acc0 + acc1 in the epilogue). tcgen05.commit frees the blob/X stage and the A buffer. Measured
//     with clock64, one issuing thread spends ~650 cycles per chunk (MMA issues ~80 cycles each,
//     commits ~90, waits ~80 even when ready), which alone bounded the kernel at N <= 32; a second
//     issuer gave 1.5x, a third and fourth nothing more.
//   - Every stage and A buffer belongs to one producer, one group and one MMA warp (NSB, NA multiples
//     of 4), which use it strictly in turn: mbarrier parity waits alias when a waiter runs two phases
//     ahead (odd ring depths faulted on stale blob indices).
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

#ifdef BS_TRACE_K6
// Debug timeline (tools/k6_trace_probe.py): %globaltimer at phase boundaries, per CTA.
__device__ unsigned long long g_k6_trace[4096 * 16];
extern "C" int bs_k6_trace_read(void* host, int n) { return (int)cudaMemcpyFromSymbol(host, g_k6_trace, (size_t)n * 8); }
#define K6_MARK(i)                                                                                              \
  do {                                                                                                          \
    unsigned long long t_;                                                                                      \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                                      \
    const unsigned cta_ = blockIdx.x + gridDim.x * blockIdx.y;                                                  \
    if (cta_ < 4096) g_k6_trace[cta_ * 16 + (i)] = t_;                                                          \
  } while (0)
// cycle accounting of the waits (clock64; globaltimer ticks are too coarse for ~200 ns chunks)
#define K6_TIC(t) t = clock64()
#define K6_TOC(acc, t) acc += clock64() - (t)
#define K6_STORE(i, v)                                                                                          \
  do {                                                                                                          \
    const unsigned cta_ = blockIdx.x + gridDim.x * blockIdx.y;                                                  \
    if (cta_ < 4096) g_k6_trace[cta_ * 16 + (i)] = (unsigned long long)(v);                                     \
  } while (0)
#else
#define K6_MARK(i) \
  do {             \
  } while (0)
#define K6_TIC(t) (void)0
#define K6_TOC(acc, t) (void)0
#define K6_STORE(i, v) (void)0
#endif

namespace {

using namespace bsk_tc;

constexpr int BM = 128;          // rows per tile (MMA M)
constexpr int KC = 64;           // columns per chunk (one SWIZZLE_128B atom of 16-bit values)
constexpr int kMaxNA = 8;        // dense A tile buffers (runtime NA: 4 or 8)
constexpr int kMaxStages = 16;   // blob + X tile ring stages (runtime NSB: 4, 8, 12 or 16)
constexpr int kDecomp = 128;     // threads per decompress group (4 warps)
constexpr int kGroups = 4;       // decompress groups, chunks in turn (4 chunks rebuilt concurrently)
constexpr int kProducers = 4;    // producer warps: one bulk copy takes ~0.3 us to issue (measured)
constexpr int kMmaWarp = kProducers;  // first MMA warp
constexpr int kMmaWarps = 2;          // MMA issuers (a tcgen05.mma issue costs ~80 cycles: one thread cannot keep up with N <= 32)
constexpr int kFirstDecomp = 32 * (kProducers + kMmaWarps);
constexpr int kThreads = kFirstDecomp + kGroups * kDecomp;
// split-K factor: at most 4 CTAs per cluster. Clusters of 8 CTAs with ~200 KB of shared memory each did not
// all fit at once (conv4_2: 16 clusters, CTAs starting up to 28 us late, tools/k6_trace_probe.py); S = 4
// fits and took conv3_3 26.6 -> 14.3 us.
constexpr int kMaxCluster = 4;

struct TcArgs {
  const uint8_t* W;   // packed SPMM layout
  void* Y;
  int64_t M, NB, N, ldy;
  int B, k, CB, NC;   // block width, kept per block, blocks per chunk, chunks per row tile
  int64_t tile_stride;
  int BN, S, NSB, NA; // batch columns per CTA (multiple of 16), split-K cluster size, ring stages, A buffers
  int blob_max;       // bytes of a full blob (128 rows, CB blocks)
  uint32_t idesc;
  int tmem_cols, acc_cols;  // allocated columns; columns per accumulator (one per MMA warp)
  int colfast;        // grid order (bsk::tc_cols_fast)
  // implicit im2col (bs_conv2d): X is the im2col of an NHWC input, loaded by TMA in im2col mode
  int conv, cC, cKW, cOW, cOHW, cPad;
  const void* bias;   // bs_conv2d: optional per-row (output channel) bias of D, Eq. 1's +B
  int act;            // bs_conv2d: bs_act after the bias, in fp32 before the one rounding (as bs_spmv_fused)
};

// Layer epilogue of bs_conv2d / bs_spmm_fused (bsk_tc::act_epilogue)
template <int DT>
__device__ __forceinline__ float tc_epilogue(float v, const TcArgs& a, int64_t row) {
  return act_epilogue<DT>(v, a.bias, a.act, row);
}

template <int DT>
__global__ void __launch_bounds__(kThreads, 1) spmm_tc_kernel(const __grid_constant__ CUtensorMap tX, TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[2 * kMaxStages + 2 * kMaxNA + 1];
  __shared__ uint32_t tmem_holder;
  using raw_t = uint16_t;
  constexpr int ES = 2;
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int NSB = a.NSB, NA = a.NA;
  const uint32_t sA = smem_u32(smem);                          // NA × 16 KB dense A tiles
  const uint32_t XSZ = (uint32_t)a.BN * 128;                   // X tile: BN rows × 128 B
  const uint32_t sX = sA + NA * BM * 128;                      // NSB × XSZ
  const uint32_t sR = sX + (uint32_t)NSB * XSZ;                // NSB × blob_max
  const uint32_t full = smem_u32(&bars[0]), empty = smem_u32(&bars[kMaxStages]);
  const uint32_t a_full = smem_u32(&bars[2 * kMaxStages]), a_empty = smem_u32(&bars[2 * kMaxStages + kMaxNA]);
  const uint32_t acc_full = smem_u32(&bars[2 * kMaxStages + 2 * kMaxNA]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lg_na = NA == 8 ? 3 : 2;
  const int S = a.S;
  const int rank = S > 1 ? (int)cluster_rank() : 0;
  const int64_t tile = a.colfast ? blockIdx.y : blockIdx.x / S;
  const int64_t m0 = tile * BM;
  const int64_t mt = (a.M - m0) < BM ? (a.M - m0) : BM;
  const int64_t n0 = (int64_t)(a.colfast ? blockIdx.x / S : blockIdx.y) * a.BN;
  const int c0 = (int)((int64_t)rank * a.NC / S), c1 = (int)((int64_t)(rank + 1) * a.NC / S);
  const int nloc = c1 - c0;  // >= 1 (S <= NC)
  const uint8_t* tile_base = a.W + tile * a.tile_stride;
  const int k = a.k;
  auto blob_bytes = [&](int64_t cb) {
    return (uint32_t)(bsk::align_up(mt * cb * k * ES, 16) + bsk::align_up(mt * cb * k, 16));
  };
  const uint32_t blobCB = blob_bytes(a.CB);

  if (threadIdx.x == 0) K6_MARK(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSB; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
    }
    for (int s = 0; s < NA; ++s) {
      mbar_init(a_full + 8 * s, kDecomp);  // one decompress group
      mbar_init(a_empty + 8 * s, 1);
    }
    mbar_init(acc_full, kMmaWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {  // tensor-memory accumulator: 128 lanes × tmem_cols fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // PDL: the set-up above (barriers, TMEM allocation) overlapped the previous kernel's tail; every global
  // access below waits for it (W may have just been packed, X written, Y read)
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tmem_d = tmem_holder;
  if (threadIdx.x == 0) K6_MARK(1);

  if (warp < kProducers) {
    if (lane == 0) {  // ---- producers: warp w issues chunks i = w, w + 4, ...
      if (warp == 0) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tX) : "memory");
      int s = warp % NSB;
      uint32_t ph = 0;
      [[maybe_unused]] long long tw_ = 0, c_empty = 0;
      for (int i = warp; i < nloc; i += kProducers) {
        const int c = c0 + i;
        K6_TIC(tw_);
        if (i >= NSB) mbar_wait(empty + 8 * s, ph ^ 1u);
        K6_TOC(c_empty, tw_);
        const int64_t cb = (a.NB - (int64_t)a.CB * c) < a.CB ? (a.NB - (int64_t)a.CB * c) : a.CB;
        const uint32_t bytes = blob_bytes(cb);
        mbar_expect_tx(full + 8 * s, bytes + XSZ);
        bulk_g2s(sR + (uint32_t)s * (uint32_t)a.blob_max, tile_base + (int64_t)c * blobCB, bytes, full + 8 * s);
        if (a.conv) {  // chunk c = 64 channels of one filter tap (dy, dx); the column tile starts at pixel n0
          const int col0 = c * KC, tap = col0 / a.cC, coff = col0 - tap * a.cC;
          const int dy = tap / a.cKW, dx = tap - dy * a.cKW;
          const int img = (int)(n0 / a.cOHW), pix = (int)(n0 - (int64_t)img * a.cOHW);
          const int oy = pix / a.cOW, ox = pix - oy * a.cOW;
          tma_im2col_4d(sX + (uint32_t)s * XSZ, &tX, coff, ox - a.cPad, oy - a.cPad, img, (uint16_t)dx, (uint16_t)dy,
                        full + 8 * s);
        } else {
          tma_2d(sX + (uint32_t)s * XSZ, &tX, c * KC, (int)n0, full + 8 * s);
        }
        s += kProducers;
        if (s >= NSB) { s -= NSB; ph ^= 1u; }
      }
      if (warp == 0) K6_STORE(9, c_empty);
    }
  } else if (warp < kFirstDecomp / 32) {
    if (lane == 0) {  // ---- MMA issuers: warp j issues chunks i = j, j + kMmaWarps, ... into accumulator j
      const int j = warp - kMmaWarp;
      const uint32_t acc_j = tmem_d + (uint32_t)(j * a.acc_cols);
      int s = j % NSB;
      uint32_t ph = 0;
      [[maybe_unused]] long long tw_ = 0, c_full = 0, c_afull = 0, c_issue = 0;
      for (int i = j; i < nloc; i += kMmaWarps) {
        const int ab = i & (NA - 1);
        K6_TIC(tw_);
        mbar_wait(full + 8 * s, ph);
        K6_TOC(c_full, tw_);
        K6_TIC(tw_);
        mbar_wait(a_full + 8 * ab, (uint32_t)(i >> lg_na) & 1u);
        K6_TOC(c_afull, tw_);
        K6_TIC(tw_);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t da = sw128_desc(sA + (uint32_t)ab * BM * 128), db = sw128_desc(sX + (uint32_t)s * XSZ);
#pragma unroll
        for (int kk = 0; kk < KC / 16; ++kk) {
          const uint32_t acc = (i >= kMmaWarps || kk > 0) ? 1u : 0u;
          asm volatile(
              "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(acc_j),
              "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(a.idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(empty + 8 * s)
                     : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(a_empty + 8 * ab)
                     : "memory");
        K6_TOC(c_issue, tw_);
        s += kMmaWarps;
        if (s >= NSB) { s -= NSB; ph ^= 1u; }
      }
      if (j == 0) {
        K6_STORE(10, c_full);
        K6_STORE(11, c_afull);
        K6_STORE(12, c_issue);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(acc_full)
                   : "memory");
    }
  } else {
    // ---- decompress: group grp (4 warps) rebuilds chunks i = grp, grp + 4, ...; thread t = 0..127.
    // Work unit = (row r, U = max(B, 8) columns): its U / 8 16-byte pieces of the K-major SWIZZLE_128B
    // tile and its entries (blocks u·BPU .. u·BPU + BPU - 1, contiguous in the blob). The owner zero-fills
    // its pieces and then scatters its entries, so program order alone orders the two (no barrier).
    // Entries are read 8 at a time (16-byte value load, 8-byte index load) when k % 8 == 0.
    const int grp = (threadIdx.x - kFirstDecomp) / kDecomp, t = (threadIdx.x - kFirstDecomp) % kDecomp;
    const int U = a.B >= 8 ? a.B : 8, BPU = U / a.B, PPU = U / 8;
    const int lg_upr = 31 - __clz(KC / U);  // units per row: 1, 2, 4 or 8 (U divides 64)
    const int nunits = BM << lg_upr;
    const bool vec8 = (k & 7) == 0;
    const int ilast = a.NC - 1 - c0;  // local index of the row tile's last chunk (may be >= nloc)
    const int cbF = a.CB, cbL = (int)(a.NB - (int64_t)a.CB * (a.NC - 1));
    int s = grp;  // ring stage of chunk i
    uint32_t ph = 0;
    [[maybe_unused]] long long tw_ = 0, c_aempty = 0, c_dfull = 0, c_work = 0;
    for (int i = grp; i < nloc; i += kGroups) {
      const int ab = i & (NA - 1);
      const uint32_t aph = (uint32_t)(i >> lg_na) & 1u;
      const uint32_t aT = sA + (uint32_t)ab * BM * 128;
      const int cb = i == ilast ? cbL : cbF;
      const int n_e = (int)mt * cb * k;
      K6_TIC(tw_);
      if (i >= NA) mbar_wait(a_empty + 8 * ab, aph ^ 1u);  // MMA done with this A tile
      K6_TOC(c_aempty, tw_);
      K6_TIC(tw_);
      mbar_wait(full + 8 * s, ph);
      K6_TOC(c_dfull, tw_);
      K6_TIC(tw_);
      if (t == 0 && grp == 0 && i == 0) K6_MARK(2);
      // 32-bit shared addresses (a generic pointer here would compile to LD.E with 64-bit math)
      const uint32_t bv = sR + (uint32_t)s * (uint32_t)a.blob_max;
      const uint32_t bi = bv + (((uint32_t)n_e * ES + 15u) & ~15u);
      for (int unit = t; unit < nunits; unit += kDecomp) {
        const int r = unit >> lg_upr, u = unit & ((1 << lg_upr) - 1);
        const uint32_t rowb = aT + (uint32_t)r * 128;
        for (int p = 0; p < PPU; ++p)
          bsk::sts_v4(rowb + ((((uint32_t)(u * PPU + p)) ^ (uint32_t)(r & 7)) << 4), 0u, 0u, 0u, 0u);
        if (r >= mt) continue;
        const int j0 = u * BPU, j1 = (j0 + BPU) < cb ? (j0 + BPU) : cb;
        for (int j = j0; j < j1; ++j) {
          const int e0 = (r * cb + j) * k;
          const uint32_t cbase = (uint32_t)(j * a.B);
          auto put = [&](uint32_t w, uint32_t o) {
            const uint32_t col = cbase + o;
            bsk::sts_u16(rowb + ((((col >> 3) ^ (uint32_t)r) & 7) << 4) + (col & 7) * 2, (uint16_t)w);
          };
          if (vec8) {
            for (int e = e0; e < e0 + k; e += 8) {
              uint32_t ww[4], ii[2];
              bsk::lds_v4(bv + 2u * (uint32_t)e, ww[0], ww[1], ww[2], ww[3]);
              asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(ii[0]), "=r"(ii[1]) : "r"(bi + (uint32_t)e));
#pragma unroll
              for (int q = 0; q < 8; ++q) put((ww[q >> 1] >> (16 * (q & 1))) & 0xFFFFu, (ii[q >> 2] >> (8 * (q & 3))) & 0xFFu);
            }
          } else {
            for (int e = e0; e < e0 + k; ++e) {
              uint16_t o8;
              asm volatile("ld.shared.u8 %0, [%1];" : "=h"(o8) : "r"(bi + (uint32_t)e));
              put(bsk::lds_u16(bv + 2u * (uint32_t)e), o8);
            }
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> tensor core
      mbar_arrive(a_full + 8 * ab);
      K6_TOC(c_work, tw_);
      s += kGroups;
      if (s >= NSB) { s -= NSB; ph ^= 1u; }
    }
    if (t == 0 && grp == 0) {
      K6_STORE(13, c_aempty);
      K6_STORE(14, c_dfull);
      K6_STORE(15, c_work);
    }
    // ---- epilogue: TMEM -> registers. Warp w reads lane quarter w % 4 (rows 32·(w % 4) + lane) and
    // column part (w - 2) / 4 of NP parts.
    if (t == 0 && grp == 0) K6_MARK(3);
    mbar_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (t == 0 && grp == 0) K6_MARK(4);
    const int q = warp & 3, part = (warp - kFirstDecomp / 32) >> 2;
    const int NP = a.BN % 32 == 0 ? 4 : 2;  // parts of BN / NP columns, a multiple of 8
    const int m = 32 * q + lane;
    // split-K partial tile [BN][128] fp32 at sA (the rings are idle now)
    if (part < NP) {
      const int pw = a.BN / NP;
      for (int nb = part * pw; nb < (part + 1) * pw; nb += 8) {
        // accumulator j holds chunks i = j mod kMmaWarps; summed ((acc0 + acc1) + acc2) + ..., a fixed order
        uint32_t rr[8];
        const uint32_t ta = tmem_d + ((uint32_t)(32 * q) << 16) + (uint32_t)nb;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(rr[0]), "=r"(rr[1]), "=r"(rr[2]), "=r"(rr[3]), "=r"(rr[4]), "=r"(rr[5]), "=r"(rr[6]), "=r"(rr[7])
                     : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int jacc = 1; jacc < kMmaWarps && jacc < nloc; ++jacc) {
          uint32_t r1[8];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(r1[0]), "=r"(r1[1]), "=r"(r1[2]), "=r"(r1[3]), "=r"(r1[4]), "=r"(r1[5]), "=r"(r1[6]), "=r"(r1[7])
                       : "r"(ta + (uint32_t)(jacc * a.acc_cols)));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int e = 0; e < 8; ++e) rr[e] = __float_as_uint(__uint_as_float(rr[e]) + __uint_as_float(r1[e]));
        }
        if (S > 1) {
#pragma unroll
          for (int e = 0; e < 8; ++e) bsk::sts_u32(sA + (uint32_t)(((nb + e) * BM + m) * 4), rr[e]);
        } else if (m < mt) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int64_t ng = n0 + nb + e;
            if (ng < a.N)
              ((raw_t*)a.Y)[ng * a.ldy + m0 + m] = (raw_t)bsk::from_float<DT>(tc_epilogue<DT>(__uint_as_float(rr[e]), a, m0 + m));
          }
        }
      }
    }
  }
  if (threadIdx.x == kFirstDecomp) K6_MARK(5);
  if (S > 1) {
    cluster_sync_all();  // every partial tile is parked
    if (threadIdx.x == kFirstDecomp) K6_MARK(6);
    if (warp >= kFirstDecomp / 32) {
      const int t = threadIdx.x - kFirstDecomp;
      const int U = a.BN * BM / 4;  // float4 units of the tile
      const int u0 = (int)((int64_t)rank * U / S), u1 = (int)((int64_t)(rank + 1) * U / S);
      // two units per thread and round with all their S remote loads in flight before the first add (a
      // load-add chain per unit was latency-bound: ~4.6 us of conv4_2's epilogue, tools/k6_trace_probe.py);
      // then the fixed rank order: partials over consecutive K ranges
      constexpr int UU = 2, NTH = kGroups * kDecomp;
      for (int ub = u0 + t; ub < u1; ub += UU * NTH) {
        float4 w[UU][kMaxCluster];
#pragma unroll
        for (int j = 0; j < UU; ++j)
#pragma unroll
          for (int p = 0; p < kMaxCluster; ++p)
            if (p < S && ub + j * NTH < u1) w[j][p] = ld_cluster_f4(sA + (uint32_t)(ub + j * NTH) * 16, (uint32_t)p);
#pragma unroll
        for (int j = 0; j < UU; ++j) {
          const int u = ub + j * NTH;
          if (u >= u1) break;
          float4 v = w[j][0];
#pragma unroll
          for (int p = 1; p < kMaxCluster; ++p)
            if (p < S) { v.x += w[j][p].x; v.y += w[j][p].y; v.z += w[j][p].z; v.w += w[j][p].w; }
          const int n = u >> 5, row = (u & 31) * 4;
          const int64_t ng = n0 + n;
          if (ng < a.N) {
            raw_t* yp = (raw_t*)a.Y + ng * a.ldy + m0 + row;
            const float f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (row + e < mt) yp[e] = (raw_t)bsk::from_float<DT>(tc_epilogue<DT>(f[e], a, m0 + row + e));
          }
        }
      }
    }
    if (threadIdx.x == kFirstDecomp) K6_MARK(7);
    cluster_sync_all();  // peers' shared memory stays alive until every slice is read
  }
  if (threadIdx.x == kFirstDecomp) K6_MARK(8);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == kMmaWarp) {
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
  // 3 (not 6) chunks per CTA at least: CTC W_hh (K = 1024) N = 8..256 7-9% faster, nothing slower (A/B)
  const int mc = bsk::splitk_min_chunks(3);
  if (S > NC / mc) S = NC / mc;  // at least mc chunks per CTA: fixed costs stay amortised
  return S < 1 ? 1 : (int)S;
}

struct ConvGeom {  // implicit im2col input of bsk_launch_conv (NHWC, stride 1)
  int64_t Nimg, H, W, C;
  int kh, kw, pad;
};

template <int DT>
cudaError_t launch_tc(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx, void* Y,
                      int64_t ldy, cudaStream_t s, const ConvGeom* cv = nullptr, const void* bias = nullptr,
                      int act = 0) {
  if (!cv && (((uintptr_t)X & 15) != 0 || (ldx % 8) != 0)) return cudaErrorNotSupported;  // TMA: 16-byte rows
  TcArgs a;
  a.conv = cv != nullptr;
  a.bias = bias;
  a.act = act;
  if (cv) {
    a.cC = (int)cv->C;
    a.cKW = cv->kw;
    a.cOW = (int)(cv->W + 2 * cv->pad - cv->kw + 1);
    a.cOHW = (int)((cv->H + 2 * cv->pad - cv->kh + 1) * a.cOW);
    a.cPad = cv->pad;
  }
  a.W = (const uint8_t*)packed;
  a.Y = Y;
  a.M = g.M; a.NB = g.NB; a.N = N; a.ldy = ldy;
  a.B = g.B; a.k = g.k; a.CB = g.V; a.NC = (int)g.NBf; a.tile_stride = g.offB;
  a.blob_max = (int)(bsk::align_up((int64_t)BM * g.V * g.k * 2, 16) + bsk::align_up((int64_t)BM * g.V * g.k, 16));
  a.S = split_k(g.P, g.NBf);
  auto kern = spmm_tc_kernel<DT>;
  cudaError_t perr = cudaSuccess;
  const int static_smem = bsk::prepare_func((const void*)kern, &perr);
  if (static_smem < 0) return perr;
  // NA dense A tiles + NSB stages of (X tile, blob): BN as large as 4 stages allow with NA = 4 (<= 256);
  // NA = 8 when 8 stages still fit (more chunks in flight hide the MMA completion latency), else 4.
  const int64_t avail = bsk::dev_props().smem_optin - static_smem - 1024;  // 1024: alignment slack
  int64_t bn_max = (((avail - 4LL * BM * 128) / 4 - a.blob_max) / 128) / 16 * 16;
  if (bn_max > 512 / kMmaWarps) bn_max = 512 / kMmaWarps;  // kMmaWarps accumulators in 512 TMEM columns
  if (bn_max < 16) return cudaErrorNotSupported;
  int64_t BN = (N + 15) / 16 * 16;
  if (BN > bn_max) BN = bn_max;
  // conv5_x: 4 row tiles × S = 4 × 1 column tile left 132 SMs idle (20.6 -> 13.2 us). Only below a quarter
  // of the SMs: each column tile decompresses its A chunks again, and K6 is shared-memory bound (conv4_2
  // at 64 -> 144 CTAs: 17.5 -> 23.9 us)
  BN = bsk::fill_bn(N, BN, g.P * a.S, 16, 4);
  a.BN = (int)BN;
  a.idesc = idesc_f16(DT == BS_BF16, BM, (int)BN, false);
  int cols = 32;
  while (cols < BN) cols <<= 1;
  a.acc_cols = cols;
  a.tmem_cols = cols * kMmaWarps;  // <= 512 (BN <= 256)
  a.NA = (avail - 8LL * BM * 128) / (BN * 128 + a.blob_max) >= 8 ? 8 : 4;
  const int64_t ring = avail - (int64_t)a.NA * BM * 128;
  int64_t nsb = ring / (BN * 128 + a.blob_max);
  if (nsb > kMaxStages) nsb = kMaxStages;
  // A multiple of 4 (= producers = decompress groups, a multiple of the MMA warps): then every stage
  // belongs to one producer, one group and one MMA warp, which use it strictly in turn, so no waiter
  // is ever two phases ahead of a barrier (mbarrier parity waits alias beyond one phase; odd depths
  // faulted on stale blob indices).
  nsb &= ~3LL;
  if (nsb < 4) return cudaErrorNotSupported;
  a.NSB = (int)nsb;
  const int64_t smem = 1024 + (int64_t)a.NA * BM * 128 + nsb * (BN * 128 + a.blob_max);
  if (a.S > 1 && BN * BM * 4 > smem - 1024) return cudaErrorNotSupported;  // partial tile must fit
  CUtensorMap tX;
  if (cv) {
    if (!bsk_make_map_im2col(&tX, DT, X, cv->Nimg, cv->H, cv->W, cv->C, cv->kh, cv->kw, cv->pad, (int)BN))
      return cudaErrorNotSupported;
  } else if (!bsk_make_map_2d(&tX, DT, X, g.K, N, ldx, KC, (int)BN)) {
    return cudaErrorNotSupported;
  }
  cudaLaunchConfig_t cfg = {};
  // column tiles adjacent only when W exceeds half of L2 (fc6, 31 MB, ran 10 % slower at N = 128 with them)
  a.colfast = bsk::tc_cols_fast() && g.P <= 65535 && g.total > (int64_t)bsk::dev_props().l2_bytes / 2;
  const unsigned nct = (unsigned)((N + BN - 1) / BN);
  cfg.gridDim = a.colfast ? dim3(nct * (unsigned)a.S, (unsigned)g.P) : dim3((unsigned)(g.P * a.S), nct);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)a.S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
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

// Convolution with implicit im2col (bs_conv2d): Y [pixels][Cout] = W_bs · im2col(in)ᵀ with the X tiles loaded
// straight from the NHWC input by TMA in im2col mode (no im2col kernel, no [pixels][kh·kw·C] intermediate).
// Eligible: SPMM layout, 16-bit, B | 64, C % 64 == 0 (a 64-column chunk is one filter tap), stride 1,
// symmetric padding, a 16-byte aligned input; cudaErrorNotSupported otherwise.
cudaError_t bsk_launch_conv(const bsk::Geom& g, const void* packed, const void* in, int64_t Nimg, int64_t H, int64_t W,
                            int64_t C, int kh, int kw, int pad, const void* bias, int act, void* Y, cudaStream_t s) {
  if (g.layout != BS_LAYOUT_SPMM || g.es != 2 || (64 % g.B) != 0 || g.k == 0) return cudaErrorNotSupported;
  if (C % 64 != 0 || g.K != (int64_t)kh * kw * C || ((uintptr_t)in & 15) != 0) return cudaErrorNotSupported;
  if (pad > 127 || kh > 128 || kw > 128) return cudaErrorNotSupported;
  const int64_t OH = H + 2 * pad - kh + 1, OW = W + 2 * pad - kw + 1;
  if (OH < 1 || OW < 1) return cudaErrorNotSupported;
  const int64_t N = Nimg * OH * OW;
  if (N >= (1LL << 31)) return cudaErrorNotSupported;
  const ConvGeom cv{Nimg, H, W, C, kh, kw, pad};
  return g.dt == BS_BF16 ? launch_tc<BS_BF16>(g, packed, in, N, g.K, Y, g.M, s, &cv, bias, act)
                         : launch_tc<BS_F16>(g, packed, in, N, g.K, Y, g.M, s, &cv, bias, act);
}

// Y = act(W_bs·X + bias) on the tensor cores (SPMM layout, 16-bit, B | 64, aligned X): K6 with the layer
// epilogue of bs_conv2d. cudaErrorNotSupported otherwise.
cudaError_t bsk_launch_spmm_fused(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx,
                                  void* Y, int64_t ldy, const void* bias, int act, cudaStream_t s) {
  if (g.layout != BS_LAYOUT_SPMM || g.es != 2 || (64 % g.B) != 0 || g.k == 0) return cudaErrorNotSupported;
  return g.dt == BS_BF16 ? launch_tc<BS_BF16>(g, packed, X, N, ldx, Y, ldy, s, nullptr, bias, act)
                         : launch_tc<BS_F16>(g, packed, X, N, ldx, Y, ldy, s, nullptr, bias, act);
}

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
