// spmm24.cu: K5, the 2:4 path (B = 4, k = 2: the shape of Fig. 2, at 50%) on Blackwell sparse
// tensor cores, plus its CUDA-core SpMV/SpMM (2-bit metadata, 2.25 B per nonzero at f16).
//
// The SP24 layout (docs/layout.md) is already the operand format of a 2:4 sparse MMA: the kept values
// form the compressed A (M × K/2, row-major) and the block nibbles idx0 | idx1 << 2 form the metadata
// (M × K/8 bytes). Per CTA: a 128-row tile of W, BN <= 128 batch columns and a contiguous range of the
// 128-column K chunks (split-K over a cluster of S CTAs, S from M and K only; the S fp32 partial tiles
// are summed in rank order through distributed shared memory, as in K6).
//   - One producer lane issues TMA tensor copies (cp.async.bulk.tensor.2d, 128-byte swizzle): the
//     compressed A chunk (128 rows × 64 values) and the X chunk (BN rows × 2 atoms of 64 columns).
//   - 128 threads (thread = row) copy their 16 metadata bytes of the chunk into tensor memory with
//     tcgen05.st (one 32-bit column per K = 32 step, 16-bit halves exchanged between rows r and r ^ 8).
//   - One thread issues 4 × tcgen05.mma.sp.cta_group::1.kind::f16 (M = 128, N = BN, K = 32) into an
//     fp32 accumulator in tensor memory; tcgen05.commit releases the stage.
//   - Epilogue: tcgen05.ld → Y [N][M].
// No decompression: the tensor core consumes the packed bytes directly.

#include "bs_common.cuh"
#include "bs_device.cuh"
#include "bs_tc.cuh"

#ifdef BS_TRACE_K5
// Debug timeline (tools/k6_trace_probe.py --k5): %globaltimer at phase boundaries, per CTA.
__device__ unsigned long long g_k5_trace[4096 * 16];
extern "C" int bs_k5_trace_read(void* host, int n) { return (int)cudaMemcpyFromSymbol(host, g_k5_trace, (size_t)n * 8); }
#define K5_MARK(i)                                                                                              \
  do {                                                                                                          \
    unsigned long long t_;                                                                                      \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                                      \
    const unsigned cta_ = blockIdx.x + gridDim.x * blockIdx.y;                                                  \
    if (cta_ < 4096) g_k5_trace[cta_ * 16 + (i)] = t_;                                                          \
  } while (0)
#else
#define K5_MARK(i) \
  do {             \
  } while (0)
#endif

namespace {

constexpr int BM = 128;
constexpr int KCH = 128;  // original columns per chunk (64 compressed values: one 128-byte swizzle atom)
constexpr int kMaxStages = 8;  // pipeline stages (runtime NST: as many as shared memory holds, 2..8)
constexpr int kMaxSplit = 4;   // split-K cluster size cap (as K6: clusters of 8 large-smem CTAs may not all fit)

struct Sp24Args {
  const uint8_t* meta;  // M × K/8 bytes
  void* Y;
  int64_t M, K, N, ldy;
  int BN, NC;           // batch columns per CTA (multiple of 16), chunks per row tile
  int S;                // split-K cluster size
  int NST;              // pipeline stages
  uint32_t idesc;
  int tmem_cols, meta_col, acc_stride;  // allocated TMEM columns; first metadata column; columns per accumulator
  int meta_cols;        // TMEM metadata columns per row tile: NST stages × 4 K-steps × mstride
  int mstride;          // TMEM columns between the metadata of consecutive K = 32 steps
  int colfast;          // grid order (bsk::tc_cols_fast)
  const void* bias;     // bs_spmm_fused: per-row bias of D or NULL
  int act;              // bs_spmm_fused: bs_act
  bsk_tc::ConvX cx;     // bs_conv2d: implicit im2col (cx.conv != 0; C % 64 == 0)
};

using namespace bsk_tc;

// RT row tiles of 128 rows per CTA (RT = 2: M = 256 per CTA, two accumulators in TMEM that share every
// X tile, which halves the X traffic from L2 on layers with many row tiles; each row's sum is the same
// sequence of M = 128 MMAs either way).
template <int DT, int RT>
__global__ void __launch_bounds__(64 + 128 * RT, 1) spmm24_kernel(const __grid_constant__ CUtensorMap tA,
                                                                  const __grid_constant__ CUtensorMap tX, Sp24Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[3 * kMaxStages + 1];
  using raw_t = uint16_t;
  __shared__ uint32_t tmem_holder;
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t ASZ = BM * 128;                 // compressed A chunk of one row tile: 128 rows × 128 B
  const uint32_t BSZ = 2u * (uint32_t)a.BN * 128;  // X chunk: 2 atoms of BN rows × 128 B
  const int NST = a.NST;
  const uint32_t sA = smem_u32(smem), sB = sA + NST * RT * ASZ;
  const uint32_t full = smem_u32(&bars[0]), empty = smem_u32(&bars[kMaxStages]);
  const uint32_t meta_ok = smem_u32(&bars[2 * kMaxStages]), acc_full = smem_u32(&bars[3 * kMaxStages]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.S;
  const int rank = S > 1 ? (int)cluster_rank() : 0;
  const int64_t m0 = (int64_t)(a.colfast ? blockIdx.y : blockIdx.x / S) * (BM * RT);
  const int64_t mrows = (a.M - m0) < BM * RT ? (a.M - m0) : BM * RT;  // rows of this CTA
  const int rtl = (int)((mrows + BM - 1) / BM);                       // live row tiles (1..RT)
  const int64_t n0 = (int64_t)(a.colfast ? blockIdx.x / S : blockIdx.y) * a.BN;
  const int c0 = (int)((int64_t)rank * a.NC / S), nloc = (int)((int64_t)(rank + 1) * a.NC / S) - c0;  // >= 1

  if (threadIdx.x == 0) K5_MARK(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
      mbar_init(meta_ok + 8 * s, 4 * RT);  // one arrive per metadata warp
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tX) : "memory");
  }
  if (warp == 1) {
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
  const uint32_t tmem = tmem_holder;
  if (threadIdx.x == 0) K5_MARK(1);

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nloc; ++i) {
        const int c = c0 + i;
        if (i >= NST) mbar_wait(empty + 8 * s, ph ^ 1u);
        mbar_expect_tx(full + 8 * s, (uint32_t)rtl * ASZ + BSZ);
        for (int t = 0; t < rtl; ++t) tma_2d(sA + (s * RT + t) * ASZ, &tA, c * (KCH / 2), (int)(m0 + t * BM), full + 8 * s);
        if (a.cx.conv) {  // implicit im2col: each 64-column atom is 64 channels of one filter tap
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            int cc, w, hh, nn;
            uint16_t dw, dh;
            a.cx.coords(n0, c * KCH + 64 * h2, cc, w, hh, nn, dw, dh);
            tma_im2col_4d(sB + s * BSZ + (uint32_t)h2 * (uint32_t)a.BN * 128, &tX, cc, w, hh, nn, dw, dh, full + 8 * s);
          }
        } else {
          tma_2d(sB + s * BSZ, &tX, c * KCH, (int)n0, full + 8 * s);
          tma_2d(sB + s * BSZ + (uint32_t)a.BN * 128, &tX, c * KCH + 64, (int)n0, full + 8 * s);
        }
        if (++s == NST) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- sparse MMA issuer
      int s = 0;
      uint32_t par = 0;
      for (int i = 0; i < nloc; ++i) {
        mbar_wait(full + 8 * s, par);
        if (i == 0) K5_MARK(2);
        mbar_wait(meta_ok + 8 * s, par);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          if (t < rtl) {
            const uint64_t da = sw128_desc(sA + (s * RT + t) * ASZ);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              // A: 16 compressed values (32 B) per K = 32 step; B: 32 columns (64 B) per step, atom j / 2
              const uint64_t db = sw128_desc(sB + s * BSZ + (uint32_t)(j >> 1) * (uint32_t)a.BN * 128) + (uint64_t)((j & 1) * 4);
              const uint32_t te = tmem + (uint32_t)(a.meta_col + t * a.meta_cols) + (uint32_t)((s * 4 + j) * a.mstride);
              const uint32_t acc = (i > 0 || j > 0) ? 1u : 0u;
              asm volatile(
                  "{ .reg .pred p; setp.ne.b32 p, %5, 0;\n\t"
                  "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %4, p; }" ::"r"(tmem + (uint32_t)(t * a.acc_stride)),
                  "l"(da + (uint64_t)(j * 2)), "l"(db), "r"(te), "r"(a.idesc), "r"(acc));
            }
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(empty + 8 * s)
                     : "memory");
        if (++s == NST) { s = 0; par ^= 1u; }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(acc_full)
                   : "memory");
    }
  } else {
    // ---- metadata → tensor memory (thread = row); then the epilogue. A row's 16 metadata bytes of a
    // chunk are loaded two chunks ahead, so the global latency overlaps the MMAs. Warp w >= 2 serves row
    // tile (w - 2) / 4 and TMEM lane quarter w % 4 (the quarter a warp may access).
    const int q = warp & 3;  // TMEM lane quarter of this warp: rows 32q .. 32q + 31 of its tile
    const int t = (warp - 2) >> 2;
    const int64_t row = 32 * q + lane;  // in the tile
    const int64_t trow = (int64_t)t * BM + row;  // in the CTA's rows
    const uint8_t* mrow = a.meta + (m0 + trow) * (a.K / 8) + (int64_t)c0 * 16;
    auto ldm = [&](int i) {
      return (trow < mrows && i < nloc) ? __ldg((const uint4*)(mrow + (int64_t)i * 16)) : make_uint4(0u, 0u, 0u, 0u);
    };
    uint4 m_cur = ldm(0), m_nxt = ldm(1);
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nloc; ++i) {
      if (i >= NST) mbar_wait(empty + 8 * s, ph ^ 1u);
      const uint4 m = m_cur;
      m_cur = m_nxt;
      m_nxt = ldm(i + 2);
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a.meta_col + t * a.meta_cols) + (uint32_t)(s * 4 * a.mstride);
      const uint32_t mw[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        // The sparse MMA reads the metadata of row r, K-half h (16 bits: 4 groups) from TMEM lane
        // (r % 8) + 8·h + 16·(r / 16), halfword (r / 8) % 2 (measured: tools/sp24_probe.py). So rows r
        // and r ^ 8 (lanes of this warp) swap halves: lane r % 16 < 8 keeps both rows' K-half 0, the
        // other lane both rows' K-half 1.
        const uint32_t oth = __shfl_xor_sync(0xffffffffu, mw[j], 8);
        const uint32_t w = (lane & 8) ? ((oth >> 16) | (mw[j] & 0xFFFF0000u)) : ((mw[j] & 0xFFFFu) | (oth << 16));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr + (uint32_t)(j * a.mstride)),
                     "r"(w)
                     : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(meta_ok + 8 * s);
      if (++s == NST) { s = 0; ph ^= 1u; }
    }
    if (threadIdx.x == 64) K5_MARK(3);
    mbar_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 64) K5_MARK(4);
    // split-K partial tile [BN][128·RT] fp32 at sA (the rings are idle now)
    const int64_t mt = mrows - (int64_t)t * BM;  // rows of this warp's tile (may be <= 0)
    for (int nb = 0; nb < a.BN; nb += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(t * a.acc_stride + nb)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (S > 1) {
#pragma unroll
        for (int e = 0; e < 8; ++e) bsk::sts_u32(sA + (uint32_t)(((nb + e) * (BM * RT) + trow) * 4), r[e]);
      } else if (row < mt) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int64_t ng = n0 + nb + e;
          if (ng < a.N)
            ((raw_t*)a.Y)[ng * a.ldy + m0 + trow] =
                (raw_t)bsk::from_float<DT>(act_epilogue<DT>(__uint_as_float(r[e]), a.bias, a.act, m0 + trow));
        }
      }
    }
  }
  if (threadIdx.x == 64) K5_MARK(5);
  if (S > 1) {  // fixed-order sum of the S partial tiles through distributed shared memory
    cluster_sync_all();
    if (threadIdx.x == 64) K5_MARK(6);
    if (warp >= 2) {
      const int t = threadIdx.x - 64;
      constexpr int RW = BM * RT / 4;  // float4 units per partial-tile column
      const int U = a.BN * RW;
      const int u0 = (int)((int64_t)rank * U / S), u1 = (int)((int64_t)(rank + 1) * U / S);
      // four units per thread and round, all their S remote loads in flight before the first add: a
      // load-add chain per unit was latency-bound (CTC N = 256: 4.1 us, tools/k6_trace_probe.py --k5)
      constexpr int UU = 4;
      const int NTH = 128 * RT;
      for (int ub = u0 + t; ub < u1; ub += UU * NTH) {
        float4 w[UU][kMaxSplit];
#pragma unroll
        for (int j = 0; j < UU; ++j)
#pragma unroll
          for (int p = 0; p < kMaxSplit; ++p)
            if (p < S && ub + j * NTH < u1) w[j][p] = ld_cluster_f4(sA + (uint32_t)(ub + j * NTH) * 16, (uint32_t)p);
#pragma unroll
        for (int j = 0; j < UU; ++j) {
          const int u = ub + j * NTH;
          if (u >= u1) break;
          float4 v = w[j][0];
#pragma unroll
          for (int p = 1; p < kMaxSplit; ++p)  // the fixed rank order (as K6)
            if (p < S) { v.x += w[j][p].x; v.y += w[j][p].y; v.z += w[j][p].z; v.w += w[j][p].w; }
          const int n = u / RW, r4 = (u - n * RW) * 4;
          const int64_t ng = n0 + n;
          if (ng < a.N) {
            raw_t* yp = (raw_t*)a.Y + ng * a.ldy + m0 + r4;
            const float f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (r4 + e < mrows) yp[e] = (raw_t)bsk::from_float<DT>(act_epilogue<DT>(f[e], a.bias, a.act, m0 + r4 + e));
          }
        }
      }
    }
    if (threadIdx.x == 64) K5_MARK(7);
    cluster_sync_all();
  }
  if (threadIdx.x == 64) K5_MARK(8);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
  }
}

// CTA pair (cta_group::2, cluster of 2, S = 1): M = 256 rows per pair, 128 per CTA (its compressed A rows
// and their metadata in its own shared and tensor memory), N_t = BN <= 256 batch columns, BN / 2 X rows per
// CTA. The leader (rank 0) issues tcgen05.mma.sp.cta_group::2 (M = 256, N = BN, K = 32), which reads both
// CTAs' operands and accumulates each CTA's 128 rows in its own TMEM. Both CTAs' TMA copies complete on the
// leader's full barrier; the peer's metadata threads arrive on the leader's meta barrier; the MMA commits
// multicast to both CTAs' empty / acc barriers. X traffic from L2 is half of the single-CTA M = 128 tile's.
template <int DT>
__global__ void __launch_bounds__(192, 1) spmm24_pair_kernel(const __grid_constant__ CUtensorMap tA,
                                                             const __grid_constant__ CUtensorMap tX, Sp24Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[3 * kMaxStages + 1];
  using raw_t = uint16_t;
  __shared__ uint32_t tmem_holder;
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int BNh = a.BN / 2;
  const uint32_t ASZ = BM * 128;                 // compressed A chunk: 128 rows × 128 B
  const uint32_t BSZ = 2u * (uint32_t)BNh * 128;  // this CTA's X chunk: 2 atoms of BN/2 rows × 128 B
  const int NST = a.NST;
  const uint32_t sA = smem_u32(smem), sB = sA + NST * ASZ;
  const uint32_t full = smem_u32(&bars[0]), empty = smem_u32(&bars[kMaxStages]);
  const uint32_t meta_ok = smem_u32(&bars[2 * kMaxStages]), acc_full = smem_u32(&bars[3 * kMaxStages]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_rank();  // 0: leader
  const int64_t pt = a.colfast ? blockIdx.y : blockIdx.x >> 1;
  const int64_t ct = a.colfast ? blockIdx.x >> 1 : blockIdx.y;
  const int64_t m0 = pt * (2 * BM) + rank * BM;  // this CTA's rows
  const int64_t mt = (a.M - m0) < BM ? (a.M - m0) : BM;  // may be <= 0 (the pair's second half past M)
  const int64_t n0 = ct * a.BN;
  const int nloc = a.NC;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full + 8 * s, 2);        // leader: its arrive.expect_tx + the peer's arrive
      mbar_init(empty + 8 * s, 1);       // one multicast commit
      mbar_init(meta_ok + 8 * s, 8);     // leader: both CTAs' metadata warps
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tX) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();  // both CTAs' barriers are initialised before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;");
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tmem = tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs): copies complete on the leader's full barrier
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nloc; ++i) {
        if (i >= NST) mbar_wait(empty + 8 * s, ph ^ 1u);
        const uint32_t lf = mapa_u32(full + 8 * s, 0);
        if (rank == 0) mbar_expect_tx(full + 8 * s, 2u * (ASZ + BSZ));
        else mbar_arrive_cluster(lf);
        tma_2d_pair(sA + s * ASZ, &tA, i * (KCH / 2), (int)m0, lf);
        if (a.cx.conv) {
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            int cc, w, hh, nn;
            uint16_t dw, dh;
            a.cx.coords(n0 + rank * BNh, i * KCH + 64 * h2, cc, w, hh, nn, dw, dh);
            tma_im2col_4d_pair(sB + s * BSZ + (uint32_t)h2 * (uint32_t)BNh * 128, &tX, cc, w, hh, nn, dw, dh, lf);
          }
        } else {
          tma_2d_pair(sB + s * BSZ, &tX, i * KCH, (int)(n0 + rank * BNh), lf);
          tma_2d_pair(sB + s * BSZ + (uint32_t)BNh * 128, &tX, i * KCH + 64, (int)(n0 + rank * BNh), lf);
        }
        if (++s == NST) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---- sparse MMA issuer (leader)
      int s = 0;
      uint32_t par = 0;
      for (int i = 0; i < nloc; ++i) {
        mbar_wait(full + 8 * s, par);
        mbar_wait(meta_ok + 8 * s, par);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t da = sw128_desc(sA + s * ASZ);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t db = sw128_desc(sB + s * BSZ + (uint32_t)(j >> 1) * (uint32_t)BNh * 128) + (uint64_t)((j & 1) * 4);
          const uint32_t te = tmem + (uint32_t)a.meta_col + (uint32_t)((s * 4 + j) * a.mstride);
          const uint32_t acc = (i > 0 || j > 0) ? 1u : 0u;
          asm volatile(
              "{ .reg .pred p; setp.ne.b32 p, %5, 0;\n\t"
              "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%3], %4, p; }" ::"r"(tmem),
              "l"(da + (uint64_t)(j * 2)), "l"(db), "r"(te), "r"(a.idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(empty + 8 * s),
                     "h"((uint16_t)3)
                     : "memory");
        if (++s == NST) { s = 0; par ^= 1u; }
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(acc_full),
                   "h"((uint16_t)3)
                   : "memory");
    }
  } else {
    // ---- metadata → this CTA's tensor memory (thread = row), as in spmm24_kernel; then the epilogue
    const int q = warp & 3;
    const int64_t row = 32 * q + lane;
    const uint8_t* mrow = a.meta + (m0 + row) * (a.K / 8);
    auto ldm = [&](int i) {
      return (row < mt && i < nloc) ? __ldg((const uint4*)(mrow + (int64_t)i * 16)) : make_uint4(0u, 0u, 0u, 0u);
    };
    const uint32_t lm = mapa_u32(meta_ok, 0);
    uint4 m_cur = ldm(0), m_nxt = ldm(1);
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nloc; ++i) {
      if (i >= NST) mbar_wait(empty + 8 * s, ph ^ 1u);
      const uint4 m = m_cur;
      m_cur = m_nxt;
      m_nxt = ldm(i + 2);
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)a.meta_col + (uint32_t)(s * 4 * a.mstride);
      const uint32_t mw[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t oth = __shfl_xor_sync(0xffffffffu, mw[j], 8);
        const uint32_t w = (lane & 8) ? ((oth >> 16) | (mw[j] & 0xFFFF0000u)) : ((mw[j] & 0xFFFFu) | (oth << 16));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr + (uint32_t)(j * a.mstride)),
                     "r"(w)
                     : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(lm + 8u * (uint32_t)s);
      if (++s == NST) { s = 0; ph ^= 1u; }
    }
    mbar_wait(acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int nb = 0; nb < a.BN; nb += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)nb));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < mt) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int64_t ng = n0 + nb + e;
          if (ng < a.N)
            ((raw_t*)a.Y)[ng * a.ldy + m0 + row] =
                (raw_t)bsk::from_float<DT>(act_epilogue<DT>(__uint_as_float(r[e]), a.bias, a.act, m0 + row));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();  // the leader's MMAs have read the peer's shared memory; both TMEM halves are drained
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
  }
}

// CUDA-core 2:4 product (any N, any dtype): warp per (row, batch column); lane l walks block pairs.
template <int DT>
__global__ void sp24_cc_kernel(const uint8_t* __restrict__ vals, const uint8_t* __restrict__ meta,
                               const void* __restrict__ X, void* __restrict__ Y, int64_t M, int64_t K, int64_t N,
                               int64_t ldx, int64_t ldy) {
  using raw_t = typename bsk::DTraits<DT>::raw_t;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t NB = K / 4;
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < M * N; w += nwarps) {
    const int64_t r = w % M, n = w / M;
    const raw_t* vr = (const raw_t*)vals + r * (K / 2);
    const uint8_t* mr = meta + r * (NB / 2);
    const raw_t* xn = (const raw_t*)X + n * ldx;
    float acc = 0.f;
    for (int64_t b = lane; b < NB; b += 32) {
      const uint32_t nib = (mr[b >> 1] >> (4 * (b & 1))) & 0xF;
      bsk::fma_acc<DT>(acc, vr[2 * b], xn[4 * b + (nib & 3)]);
      bsk::fma_acc<DT>(acc, vr[2 * b + 1], xn[4 * b + (nib >> 2)]);
    }
    acc = bsk::warp_sum_f(acc);
    if (lane == 0) ((raw_t*)Y)[n * ldy + r] = (raw_t)bsk::from_float<DT>(acc);
  }
}

// Batch-1 2:4 SpMV, 16-bit values (HBM-bound): a warp per row; lane l takes groups of 4 blocks
// (16 columns) g = l, l + 32, ...: one 16-byte load of the group's 8 kept values, one 2-byte load of its
// 4 metadata nibbles, two 16-byte loads of x (L1/L2-resident), then 8 FHFMAs on the selected halves.
// Two groups are loaded before either is used. Requires K % 16 == 0 and a 16-byte aligned x.
template <int DT>
__global__ void __launch_bounds__(256) sp24_spmv16_kernel(const uint16_t* __restrict__ vals,
                                                          const uint8_t* __restrict__ meta,
                                                          const uint16_t* __restrict__ x, uint16_t* __restrict__ y,
                                                          int64_t M, int64_t K) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t NG = K / 16;  // groups of 4 blocks per row
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < M; r += nwarps) {
    const uint4* vr = (const uint4*)(vals + r * (K / 2));
    const uint16_t* mr = (const uint16_t*)(meta + r * (K / 8));
    const uint4* xv = (const uint4*)x;
    float acc0 = 0.f, acc1 = 0.f;
    auto group = [&](float& acc, uint4 w, uint32_t nib, uint4 xa, uint4 xb) {
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
      const uint32_t xx[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // block q: x halves in words 2q, 2q + 1
        const uint32_t n4 = (nib >> (4 * q)) & 0xFu;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t o = h == 0 ? (n4 & 3u) : (n4 >> 2);
          const uint32_t xw = (o & 2u) ? xx[2 * q + 1] : xx[2 * q];
          bsk::fma_acc<DT>(acc, (ww[q] >> (16 * h)) & 0xFFFFu, (xw >> (16 * (o & 1u))) & 0xFFFFu);
        }
      }
    };
    int64_t g = lane;
    for (; g + 32 < NG; g += 64) {
      const uint4 w0 = __ldcs(vr + g), w1 = __ldcs(vr + g + 32);
      const uint32_t n0 = __ldcs(mr + g), n1 = __ldcs(mr + g + 32);
      const uint4 x0a = __ldg(xv + 2 * g), x0b = __ldg(xv + 2 * g + 1);
      const uint4 x1a = __ldg(xv + 2 * (g + 32)), x1b = __ldg(xv + 2 * (g + 32) + 1);
      group(acc0, w0, n0, x0a, x0b);
      group(acc1, w1, n1, x1a, x1b);
    }
    if (g < NG) group(acc0, __ldcs(vr + g), __ldcs(mr + g), __ldg(xv + 2 * g), __ldg(xv + 2 * g + 1));
    const float tot = bsk::warp_sum_f(acc0 + acc1);
    if (lane == 0) y[r] = (uint16_t)bsk::from_float<DT>(tot);
  }
}

struct Conv24 {  // implicit im2col input (bs_conv2d on SP24)
  int64_t Nimg, H, W, C;
  int kh, kw, pad;
};

template <int DT>
cudaError_t launch_tc24(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx, void* Y,
                        int64_t ldy, cudaStream_t s, const void* bias = nullptr, int act = 0,
                        const Conv24* cv = nullptr) {
  int BN = (int)((N + 15) / 16 * 16);
  static const int bn_max = [] {  // BS_K5_BN_MAX: tuning knob (128 or 256); BN only partitions columns
    const char* e = getenv("BS_K5_BN_MAX");
    const int v = e && e[0] ? atoi(e) : 128;
    return v >= 256 ? 256 : 128;
  }();
  if (BN > bn_max) BN = bn_max;  // 128 keeps a 4-stage ring; 256 leaves 2 stages
  const int64_t tiles = (g.M + BM - 1) / BM;
  // RT = 2 (two row tiles per CTA sharing each X tile) when the layer has enough row tiles and enough
  // columns that X traffic matters: A/B in DESIGN.md §4 K5. BS_K5_RT forces 1 or 2. BN <= 128 (TMEM:
  // two accumulators + metadata).
  static const int rt_env = [] {
    const char* e = getenv("BS_K5_RT");
    return e && e[0] ? atoi(e) : 0;
  }();
  int RT = rt_env == 1 || rt_env == 2 ? rt_env : ((tiles >= 64 && N > 64) ? 2 : 1);
  if (RT == 2 && BN > 128) BN = 128;
  // CTA pairs (M = 256 per pair, BN <= 256) whenever split-K is off (S = 1: >= 75 row tiles on 148 SMs);
  // bit-identical to the single-CTA kernel (tools/k5_pair_check.py, test_k5_pair_*). BS_K5_PAIR=0: off.
  static const int pair_env = [] {
    const char* e = getenv("BS_K5_PAIR");
    return e && e[0] ? atoi(e) : 1;
  }();
  const bool pair = pair_env == 1 && bsk::dev_props().sms / tiles <= 1;
  if (pair) {
    RT = 1;
    BN = (int)((N + 31) / 32 * 32);
    if (BN > 256) BN = 256;
  }
  {  // narrower column tiles when the row tiles × split leave SMs idle (bsk::fill_bn; S as computed below)
    int64_t Sf = pair ? 1 : bsk::dev_props().sms / tiles;
    if (Sf > kMaxSplit) Sf = kMaxSplit;
    if (Sf > (g.K / KCH) / bsk::splitk_min_chunks(6)) Sf = (g.K / KCH) / bsk::splitk_min_chunks(6);
    if (Sf < 1) Sf = 1;
    const int64_t rows_per_cta = pair ? BM : (int64_t)BM * RT;
    BN = (int)bsk::fill_bn(N, BN, (g.M + rows_per_cta - 1) / rows_per_cta * Sf, pair ? 32 : 16, 2);  // CTC N = 64: 64 -> 128 CTAs
  }
  CUtensorMap tA, tX;
  const uint8_t* base = (const uint8_t*)packed;
  if (!bsk_make_map_2d(&tA, DT, base + g.offA, g.K / 2, g.M, g.K / 2, 64, BM)) return cudaErrorNotSupported;
  if (cv) {
    if (!bsk_make_map_im2col(&tX, DT, X, cv->Nimg, cv->H, cv->W, cv->C, cv->kh, cv->kw, cv->pad, pair ? BN / 2 : BN))
      return cudaErrorNotSupported;
  } else if (!bsk_make_map_2d(&tX, DT, X, g.K, N, ldx, 64, pair ? BN / 2 : BN)) {
    return cudaErrorNotSupported;
  }
  Sp24Args a;
  a.bias = bias;
  a.act = act;
  a.cx.conv = cv != nullptr;
  if (cv) {
    a.cx.C = (int)cv->C;
    a.cx.KW = cv->kw;
    a.cx.OW = (int)(cv->W + 2 * cv->pad - cv->kw + 1);
    a.cx.OHW = (int)((cv->H + 2 * cv->pad - cv->kh + 1) * a.cx.OW);
    a.cx.pad = cv->pad;
  }
  a.meta = base + g.offB;
  a.Y = Y;
  a.M = g.M; a.K = g.K; a.N = N; a.ldy = ldy;
  a.BN = BN;
  a.NC = (int)(g.K / KCH);
  a.idesc = idesc_f16(DT == BS_BF16, pair ? 2 * BM : BM, BN, true);
  a.mstride = 4;  // the metadata address of each K = 32 step must be 4-column aligned (stride 1 faults)
  int p2 = 32;
  while (p2 < BN) p2 <<= 1;
  a.acc_stride = p2;
  const int64_t stage = (int64_t)RT * BM * 128 + 2LL * (pair ? BN / 2 : BN) * 128;
  int64_t nst = (bsk::dev_props().smem_optin - 2048) / stage;
  static const int st_env = [] {  // BS_K5_STAGES: cap on the ring depth (A/B)
    const char* e = getenv("BS_K5_STAGES");
    return e && e[0] ? atoi(e) : kMaxStages;
  }();
  if (nst > st_env) nst = st_env;
  if (nst > kMaxStages) nst = kMaxStages;
  if (nst < 2) return cudaErrorNotSupported;
  a.NST = (int)nst;
  a.meta_cols = (int)nst * 4 * a.mstride;
  const int tot = RT * (p2 + a.meta_cols);
  int cols = 32;
  while (cols < tot) cols <<= 1;
  a.meta_col = RT * p2;
  a.tmem_cols = cols;
  if (a.tmem_cols > 512) return cudaErrorNotSupported;
  const int64_t smem = 1024 + nst * stage;
  int64_t S = bsk::dev_props().sms / tiles;  // split-K: from M and K only (never N, never RT)
  if (S > kMaxSplit) S = kMaxSplit;
  // 6: a deeper split helped N <= 128 by 7% but cost 60% at N = 256 (A/B on CTC W_ih)
  const int mc = bsk::splitk_min_chunks(6);
  if (S > a.NC / mc) S = a.NC / mc;  // at least mc chunks per CTA: fixed costs stay amortised
  if (S < 1) S = 1;
  a.S = (int)S;
  if (S > 1 && (int64_t)BN * BM * RT * 4 > nst * stage) return cudaErrorNotSupported;  // partial tile must fit
  if (pair) a.S = (int)(S = 1);
  const void* kern = pair ? (const void*)spmm24_pair_kernel<DT>
                          : RT == 2 ? (const void*)spmm24_kernel<DT, 2> : (const void*)spmm24_kernel<DT, 1>;
  cudaError_t perr = cudaSuccess;
  const int static_smem = bsk::prepare_func(kern, &perr);
  if (static_smem < 0) return perr;
  if (smem > bsk::dev_props().smem_optin - static_smem) return cudaErrorNotSupported;
  const int64_t ctiles = pair ? (g.M + 2 * BM - 1) / (2 * BM) : (g.M + BM * RT - 1) / (BM * RT);
  const unsigned cl = pair ? 2u : (unsigned)S;  // cluster size along x
  cudaLaunchConfig_t cfg = {};
  a.colfast = bsk::tc_cols_fast() && ctiles <= 65535;
  const unsigned nct = (unsigned)((N + BN - 1) / BN);
  cfg.gridDim = a.colfast ? dim3(nct * cl, (unsigned)ctiles) : dim3((unsigned)ctiles * cl, nct);
  cfg.blockDim = dim3(pair ? 192 : 64 + 128 * RT);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  void* args[] = {(void*)&tA, (void*)&tX, (void*)&a};
  return cudaLaunchKernelExC(&cfg, kern, args);
}

template <int DT>
cudaError_t launch_cc24(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx, void* Y,
                        int64_t ldy, cudaStream_t s) {
  const uint8_t* base = (const uint8_t*)packed;
  int64_t blocks = (g.M * N + 7) / 8;
  if (blocks > (int64_t)bsk::dev_props().sms * 16) blocks = (int64_t)bsk::dev_props().sms * 16;
  sp24_cc_kernel<DT><<<(unsigned)blocks, 256, 0, s>>>(base + g.offA, base + g.offB, X, Y, g.M, g.K, N, ldx, ldy);
  return cudaGetLastError();
}

}  // namespace

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)p;
  }
  return fn;
}

bool bsk_make_map_2d(CUtensorMap* m, int dt, const void* base, int64_t cols, int64_t rows, int64_t ld, int bc, int br) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
  cuuint32_t es[2] = {1, 1};
  const CUtensorMapDataType t = dt == BS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  return fn(m, t, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

bool bsk_make_map_im2col(CUtensorMap* m, int dt, const void* in, int64_t Nimg, int64_t H, int64_t W, int64_t C, int kh,
                         int kw, int pad, int pixels) {
  static EncodeIm2colFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeIm2colFn)p;
  }
  if (!fn) return false;
  // dims innermost first: C, W, H, N. The base pixels of the output positions run over
  // [-pad, extent - 1 + pad - (k - 1)] in each spatial dimension (stride 1).
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)Nimg};
  cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)(W * C * 2), (cuuint64_t)(H * W * C * 2)};
  int lower[2] = {-pad, -pad};
  int upper[2] = {pad - (kw - 1), pad - (kh - 1)};
  cuuint32_t es[4] = {1, 1, 1, 1};
  const CUtensorMapDataType t = dt == BS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  return fn(m, t, 4, const_cast<void*>(in), dims, strides, lower, upper, 64, (cuuint32_t)pixels, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// bs_conv2d on the SP24 layout: K5 with its X atoms loaded by TMA in im2col mode (as bsk_launch_conv for K6).
cudaError_t bsk_launch_conv24(const bsk::Geom& g, const void* packed, const void* in, int64_t Nimg, int64_t H, int64_t W,
                              int64_t C, int kh, int kw, int pad, const void* bias, int act, void* Y, cudaStream_t s) {
  if (g.layout != BS_LAYOUT_SP24 || g.es != 2 || g.K % KCH != 0) return cudaErrorNotSupported;
  if (C % 64 != 0 || g.K != (int64_t)kh * kw * C || ((uintptr_t)in & 15) != 0) return cudaErrorNotSupported;
  if (pad > 127 || kh > 128 || kw > 128) return cudaErrorNotSupported;
  const int64_t OH = H + 2 * pad - kh + 1, OW = W + 2 * pad - kw + 1;
  if (OH < 1 || OW < 1) return cudaErrorNotSupported;
  const int64_t N = Nimg * OH * OW;
  if (N >= (1LL << 31)) return cudaErrorNotSupported;
  const Conv24 cv{Nimg, H, W, C, kh, kw, pad};
  return g.dt == BS_BF16 ? launch_tc24<BS_BF16>(g, packed, in, N, g.K, Y, g.M, s, bias, act, &cv)
                         : launch_tc24<BS_F16>(g, packed, in, N, g.K, Y, g.M, s, bias, act, &cv);
}

// Y = act(W·X + bias) on the sparse tensor cores (bs_spmm_fused, SP24 layout); NotSupported when the operands
// do not allow the tensor-core path.
cudaError_t bsk_launch_sp24_fused(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx, void* Y,
                                  int64_t ldy, const void* bias, int act, cudaStream_t s) {
  const bool tc = g.es == 2 && g.K % KCH == 0 && ((uintptr_t)X & 15) == 0 && (ldx % 8) == 0;
  if (!tc) return cudaErrorNotSupported;
  return g.dt == BS_BF16 ? launch_tc24<BS_BF16>(g, packed, X, N, ldx, Y, ldy, s, bias, act)
                         : launch_tc24<BS_F16>(g, packed, X, N, ldx, Y, ldy, s, bias, act);
}

// Y = W·X for W in SP24 layout.
//   spmv (bs_spmv, N = 1): the HBM-bound CUDA-core SpMV with 16-byte loads.
//   otherwise (bs_spmm): the sparse tensor cores whenever the operands allow it (f16/bf16, K % 128 == 0,
//   16-byte aligned X rows), at every N including 1, so a column's summation order does not depend on N
//   and batch-sharded products reproduce the unsharded columns (include/bs.h). Operands the tensor path
//   cannot take (f32, unaligned X) use the scalar CUDA-core kernel at every N.
cudaError_t bsk_launch_sp24(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx, void* Y,
                            int64_t ldy, cudaStream_t s, bool spmv) {
  const bool aligned = ((uintptr_t)X & 15) == 0;
  if (spmv && g.es == 2 && g.K % 16 == 0 && aligned) {  // batch 1: HBM-bound SpMV
    const uint8_t* base = (const uint8_t*)packed;
    int64_t blocks = (g.M + 7) / 8;
    if (blocks > (int64_t)bsk::dev_props().sms * 8) blocks = (int64_t)bsk::dev_props().sms * 8;
    auto kern = g.dt == BS_BF16 ? sp24_spmv16_kernel<BS_BF16> : sp24_spmv16_kernel<BS_F16>;
    kern<<<(unsigned)blocks, 256, 0, s>>>((const uint16_t*)(base + g.offA), base + g.offB, (const uint16_t*)X,
                                          (uint16_t*)Y, g.M, g.K);
    return cudaGetLastError();
  }
  const bool tc = !spmv && g.es == 2 && g.K % KCH == 0 && aligned && (ldx % 8) == 0;
  if (tc) {
    cudaError_t e = g.dt == BS_BF16 ? launch_tc24<BS_BF16>(g, packed, X, N, ldx, Y, ldy, s)
                                    : launch_tc24<BS_F16>(g, packed, X, N, ldx, Y, ldy, s);
    if (e != cudaErrorNotSupported) return e;
  }
  switch (g.dt) {
    case BS_F32: return launch_cc24<BS_F32>(g, packed, X, N, ldx, Y, ldy, s);
    case BS_F16: return launch_cc24<BS_F16>(g, packed, X, N, ldx, Y, ldy, s);
    default: return launch_cc24<BS_BF16>(g, packed, X, N, ldx, Y, ldy, s);
  }
}
