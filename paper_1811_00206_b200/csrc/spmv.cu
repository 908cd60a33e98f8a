// spmv.cu: K3 bs_spmv, y = W_bs · x for a balanced-sparse W in the SPMV (or SPMM) layout.
//
// Paper design (Fig. 3): one thread per block partition; every thread gets the same
// work because every block keeps k entries; x is "rearranged and stored in shared memory to
// avoid bank conflicts". The B200 version:
//   - A warp walks a contiguous range of rows. Lane l owns the blocks b ≡ l (mod 32), V of them per
//     panel of 32·V blocks (docs/layout.md). The warp's packed values and indices form contiguous
//     runs of "steps" (32·V entries each).
//   - Those runs reach shared memory through the TMA bulk-copy engine (cp.async.bulk, SASS UBLKCP).
//     Each warp owns a ring of NS stages of up to Q steps. Lane 0 refills a stage as soon as the
//     warp has consumed it, and mbarriers with transaction counts signal arrival. So the bytes in
//     flight do not depend on register pressure or on the compute phase (tools/membench.cu:
//     >= 6.9 TB/s at 64 KB in flight per SM).
//   - x is staged per CTA in a block-interleaved order of 32-bit slots: element (b, o) of a chunk
//     goes to word (gl·B + o)·32 + (b & 31), with gl = (b>>5) - first group of the chunk. 16-bit
//     values sit zero-extended in the low half. Lane l only ever touches bank l, whatever the
//     indices are, so every gather is conflict-free by construction. The slot address is one
//     IMAD of the index byte (extracted by one PRMT): 4 instructions per nonzero including the
//     FHFMA.
//   - K is processed in chunks of whole panels when x does not fit in shared memory (65536 columns
//     of 16-bit x take 256 KB as slots). Each (row, chunk) partial is reduced by the warp and added
//     in chunk order. The tail blocks (T < 32·V per row, region VB) are a last pass with direct loads.
//   - f16/bf16 products are one FHFMA (exact 16x16 product, fp32 accumulate). Each lane keeps V
//     independent accumulators. They are summed in a fixed order and reduced with a warp butterfly.
//     Chunking depends only on (K, B, dtype), never on the row range, so row-sharded results are
//     bit-identical to unsharded ones.
//   - The grid is persistent, one 512-thread CTA per SM. Each CTA owns a contiguous, balanced row range.
#include "bs_common.cuh"
#include "bs_device.cuh"

namespace {

constexpr int kNT = 512;                 // threads per CTA (16 warps)
constexpr int kXBudget = 128 * 1024;     // bytes of x slots per chunk
constexpr int kMaxChunks = 8;

struct SpmvArgs {
  const uint8_t* VA;
  const uint8_t* VB;
  const uint8_t* IA;
  const uint8_t* IB;
  const void* x;
  void* y;
  int64_t M, NB, NBf, T;
  int B, k;
  int NS;          // ring stages per warp
  int xbytes;      // smem bytes reserved for x slots (max over chunks)
  int nchunks;     // panel chunks
  int PC;          // panels per chunk (the last may be shorter)
  int tail_in_last;  // tail groups are staged with the last panel chunk
  int xvec;        // x is 16-byte aligned and B allows 16-byte staging loads
};

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// Byte i (compile-time after unrolling) of w, zero-extended: one PRMT.
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int i) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "r"(0x4440 | i));
  return r;
}

// Stage the x columns of groups [g0, g1) into 32-bit slots: word (gl·B + o)·32 + l, gl = g - g0.
// Warp w fills groups g0+w, g0+w+NW, ...; lane l copies block g·32 + l into its own bank column.
template <int ES>
__device__ __forceinline__ void stage_x(const SpmvArgs& a, uint32_t sx, int64_t g0, int64_t g1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t gstride = (uint32_t)a.B * 128;
  for (int64_t g = g0 + warp; g < g1; g += nw) {
    const int64_t b = g * 32 + lane;
    if (b >= a.NB) continue;
    const uint32_t col = sx + (uint32_t)(g - g0) * gstride + lane * 4;  // + o*128
    if (ES == 2) {
      const uint16_t* xs = (const uint16_t*)a.x + b * a.B;
      if (a.xvec) {  // B % 8 == 0 and 16-byte aligned: 8 halves per load
        for (int q = 0; q < a.B / 8; ++q) {
          const uint4 v = __ldg((const uint4*)xs + q);
          const uint32_t c0 = col + q * 8 * 128;
          bsk::sts_u32(c0 + 0 * 128, v.x & 0xffffu);
          bsk::sts_u32(c0 + 1 * 128, v.x >> 16);
          bsk::sts_u32(c0 + 2 * 128, v.y & 0xffffu);
          bsk::sts_u32(c0 + 3 * 128, v.y >> 16);
          bsk::sts_u32(c0 + 4 * 128, v.z & 0xffffu);
          bsk::sts_u32(c0 + 5 * 128, v.z >> 16);
          bsk::sts_u32(c0 + 6 * 128, v.w & 0xffffu);
          bsk::sts_u32(c0 + 7 * 128, v.w >> 16);
        }
      } else {
        for (int o = 0; o < a.B; ++o) bsk::sts_u32(col + o * 128, (uint32_t)__ldg(xs + o));
      }
    } else {
      const uint32_t* xs = (const uint32_t*)a.x + b * a.B;
      if (a.xvec) {  // B % 4 == 0 and aligned
        for (int q = 0; q < a.B / 4; ++q) {
          const uint4 v = __ldg((const uint4*)xs + q);
          const uint32_t c0 = col + q * 4 * 128;
          bsk::sts_u32(c0 + 0 * 128, v.x);
          bsk::sts_u32(c0 + 1 * 128, v.y);
          bsk::sts_u32(c0 + 2 * 128, v.z);
          bsk::sts_u32(c0 + 3 * 128, v.w);
        }
      } else {
        for (int o = 0; o < a.B; ++o) bsk::sts_u32(col + o * 128, __ldg(xs + o));
      }
    }
  }
}

template <int DT>
__device__ __forceinline__ uint32_t lds_x(uint32_t addr) {
  return bsk::DTraits<DT>::kBytes == 2 ? bsk::lds_u16(addr) : bsk::lds_u32(addr);
}

// Per-lane accumulators -> warp total: fixed-order sum over v, then a butterfly.
template <int V>
__device__ __forceinline__ float warp_total(float (&acc)[V]) {
  float sum = acc[0];
#pragma unroll
  for (int v = 1; v < V; ++v) sum += acc[v];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  return bsk::warp_sum_f(sum);
}

// One CTA per SM, kNT/32 warps. Warp rows [wr0, wr1). For panel chunk c (panels [c·PC, c·PC+np)),
// each row contributes a segment of L = np·k consecutive steps. The ring streams the segments of
// all chunks in order; a stage never crosses a segment.
template <int DT, int V, int IS, int Q, int BT, bool MULTI>
__global__ void __launch_bounds__(kNT, 1) spmv_kernel(SpmvArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kNT / 32][4];
  using raw_t = typename bsk::DTraits<DT>::raw_t;
  constexpr int ES = bsk::DTraits<DT>::kBytes;
  constexpr int P = 32 * V;
  constexpr uint32_t SVB = Q * P * ES;  // values bytes per stage
  constexpr uint32_t SIB = Q * P * IS;  // index bytes per stage
  constexpr uint32_t SB = SVB + SIB;
  const int B = BT > 0 ? BT : a.B;
  const uint32_t GSW = (uint32_t)B * 128;  // bytes per group of 32 blocks (32-bit slots)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kNT / 32;
  const int64_t rb = (int64_t)blockIdx.x * a.M / gridDim.x;
  const int64_t re = (int64_t)(blockIdx.x + 1) * a.M / gridDim.x;
  const int64_t wr0 = rb + (int64_t)warp * (re - rb) / nw;
  const int64_t nrows = rb + (int64_t)(warp + 1) * (re - rb) / nw - wr0;
  const int64_t S = a.NBf * a.k;  // full-panel steps per row
  const int NS = a.NS;
  const uint32_t sx = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t ring = sx + a.xbytes + (uint32_t)(warp * NS) * SB;
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[warp][0]);
  float* part = (float*)(smem + a.xbytes + (size_t)nw * NS * SB) - rb;  // fp32 row partials (MULTI)

  // ---- producer cursor (lane 0): (chunk, row, step-in-segment) of the next stage to load
  int pc = 0;
  int64_t pr = 0, ps = 0;
  auto seg_len = [&](int c) -> int64_t {
    const int64_t p0 = (int64_t)c * a.PC;
    const int64_t np = (a.NBf - p0) < a.PC ? (a.NBf - p0) : a.PC;
    return np * a.k;
  };
  int64_t pL = seg_len(0);
  const bool have_panels = S > 0 && nrows > 0;
  auto issue = [&](uint32_t st) {  // load the next stage into ring slot st
    const int64_t n = (pL - ps) < Q ? (pL - ps) : Q;
    const int64_t step0 = (wr0 + pr) * S + (int64_t)pc * a.PC * a.k + ps;
    const uint32_t bv = (uint32_t)n * (P * ES), bi = (uint32_t)n * (P * IS);
    const uint32_t bar = bar0 + st * 8;
    mbar_expect_tx(bar, bv + bi);
    bulk_g2s(ring + st * SB, a.VA + step0 * (P * ES), bv, bar);
    bulk_g2s(ring + st * SB + SVB, a.IA + step0 * (P * IS), bi, bar);
    ps += n;
    if (ps == pL) {
      ps = 0;
      if (++pr == nrows) { pr = 0; ++pc; if (pc < a.nchunks) pL = seg_len(pc); }
    }
  };
  if (lane == 0) {
    for (int st = 0; st < NS; ++st) mbar_init(bar0 + st * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (have_panels)
      for (int st = 0; st < NS && pc < a.nchunks; ++st) issue((uint32_t)st);
  }
  __syncwarp();

  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;

  // ---- consumer
  int64_t consumed = 0;
  for (int c = 0; c < a.nchunks; ++c) {
    const int64_t g0 = (int64_t)c * a.PC * V;
    const bool last = c == a.nchunks - 1;
    const int64_t g1 = last && a.tail_in_last ? (a.NB + 31) / 32 : g0 + (seg_len(c) / (a.k > 0 ? a.k : 1)) * V;
    if (c > 0) __syncthreads();  // all warps are done with the previous chunk's x
    stage_x<ES>(a, sx, g0, g1);
    __syncthreads();
    if (!have_panels) continue;
    const int64_t L = seg_len(c);
    const uint32_t pstep = V * GSW;
    const int k = a.k;
    for (int64_t i = 0; i < nrows; ++i) {
      uint32_t pb = sx + lane * 4;  // slot base of the current panel within the chunk
      int t = 0;
      for (int64_t s0 = 0; s0 < L; s0 += Q) {
        const uint32_t st = (uint32_t)(consumed % NS);
        mbar_wait(bar0 + st * 8, (uint32_t)((consumed / NS) & 1));
        const uint32_t sv = ring + st * SB + lane * (V * ES);
        const uint32_t si = ring + st * SB + SVB + lane * (V * IS);
        const int nq = (L - s0) < Q ? (int)(L - s0) : Q;
        auto step = [&](int q) {
          uint32_t wv[(V * ES + 3) / 4], iv[(V * IS + 3) / 4];
          const uint32_t av = sv + q * (P * ES), ai = si + q * (P * IS);
          if constexpr (V * ES == 16) bsk::lds_v4(av, wv[0], wv[1], wv[2], wv[3]);
          else if constexpr (V * ES == 8) asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(wv[0]), "=r"(wv[1]) : "r"(av));
          else if constexpr (V * ES == 4) wv[0] = bsk::lds_u32(av);
          else wv[0] = bsk::lds_u16(av);
          if constexpr (V * IS == 16) bsk::lds_v4(ai, iv[0], iv[1], iv[2], iv[3]);
          else if constexpr (V * IS == 8) asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(iv[0]), "=r"(iv[1]) : "r"(ai));
          else if constexpr (V * IS == 4) iv[0] = bsk::lds_u32(ai);
          else if constexpr (V * IS == 2) iv[0] = bsk::lds_u16(ai);
          else { uint16_t b8; asm volatile("ld.shared.u8 %0, [%1];" : "=h"(b8) : "r"(ai)); iv[0] = b8; }
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const uint32_t o = IS == 1 ? byte_of(iv[v >> 2], v & 3) : (iv[v >> 1] >> (16 * (v & 1))) & 0xffffu;
            const uint32_t xv = lds_x<DT>(pb + o * 128 + v * GSW);
            const uint32_t w = ES == 2 ? (wv[v >> 1] >> (16 * (v & 1))) & 0xffffu : wv[v];
            bsk::fma_acc<DT>(acc[v], w, xv);
          }
          if (++t == k) { t = 0; pb += pstep; }
        };
        if (nq == Q) {  // full stage: no per-step predicate
#pragma unroll
          for (int q = 0; q < Q; ++q) step(q);
        } else {
#pragma unroll
          for (int q = 0; q < Q; ++q)
            if (q < nq) step(q);
        }
        __syncwarp();  // every lane is done with stage st
        ++consumed;
        if (lane == 0 && pc < a.nchunks) issue(st);
      }
      const int64_t r = wr0 + i;
      const float tot = warp_total<V>(acc);
      if (lane == 0) {
        if (MULTI) part[r] = c == 0 ? tot : part[r] + tot;
        else ((raw_t*)a.y)[r] = (raw_t)bsk::from_float<DT>(tot);
      }
    }
  }

  // ---- tail blocks (region VB, (t, v, lane) order), direct loads; x of the tail groups is staged
  if (a.T > 0 && a.k > 0) {
    const int64_t gt0 = a.NBf * V, gt1 = (a.NB + 31) / 32;
    uint32_t tbase;
    if (a.tail_in_last) {
      tbase = sx + (uint32_t)(gt0 - (int64_t)(a.nchunks - 1) * a.PC * V) * GSW;
    } else {
      __syncthreads();
      stage_x<ES>(a, sx, gt0, gt1);
      __syncthreads();
      tbase = sx;
    }
    const int Vt = (int)((a.T + 31) / 32);
    const raw_t* vb = (const raw_t*)a.VB;
    for (int64_t i = 0; i < nrows; ++i) {
      const int64_t r = wr0 + i;
      const int64_t f0 = r * a.k * a.T;
      for (int tt = 0; tt < a.k; ++tt) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int bl = v * 32 + lane;
          if (v < Vt && bl < a.T) {
            const int64_t e = f0 + (int64_t)tt * a.T + bl;
            const uint32_t w = vb[e];
            const uint32_t o = IS == 1 ? (uint32_t)a.IB[e] : (uint32_t)((const uint16_t*)a.IB)[e];
            const uint32_t xv = lds_x<DT>(tbase + lane * 4 + o * 128 + v * GSW);
            bsk::fma_acc<DT>(acc[v], w, xv);
          }
        }
      }
      const float tot = warp_total<V>(acc);
      if (lane == 0) {
        const float y = S > 0 ? part[r] + tot : tot;
        ((raw_t*)a.y)[r] = (raw_t)bsk::from_float<DT>(y);
      }
    }
  } else if (S == 0) {  // k == 0: y = 0
    for (int64_t i = lane; i < nrows; i += 32) ((raw_t*)a.y)[wr0 + i] = (raw_t)bsk::from_float<DT>(0.f);
  } else if (MULTI) {
    __syncwarp();
    for (int64_t i = lane; i < nrows; i += 32) ((raw_t*)a.y)[wr0 + i] = (raw_t)bsk::from_float<DT>(part[wr0 + i]);
  }
}

template <int V, int ES>
struct StageSteps {  // Q: 2 KB of values per stage
  static constexpr int value = 2048 / (32 * V * ES) < 1 ? 1 : 2048 / (32 * V * ES);
};

template <int DT, int V, int IS, int BT, bool MULTI>
cudaError_t launch_cfg(const SpmvArgs& a0, cudaStream_t s) {
  constexpr int ES = bsk::DTraits<DT>::kBytes;
  constexpr int Q = StageSteps<V, ES>::value;
  constexpr int SB = Q * 32 * V * (ES + IS);
  static int static_smem = -1;  // per instantiation: static smem (the mbarriers)
  auto kern = spmv_kernel<DT, V, IS, Q, BT, MULTI>;
  const auto& dp = bsk::dev_props();
  if (static_smem < 0) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dp.smem_optin - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
    static_smem = (int)fa.sharedSizeBytes;
  }
  SpmvArgs a = a0;
  int64_t grid = dp.sms;
  const int64_t need = (a.M + (kNT / 32) - 1) / (kNT / 32);
  if (grid > need) grid = need;
  const int64_t scratch = MULTI ? ((a.M + grid - 1) / grid + 1) * 4 : 0;
  const int64_t avail = dp.smem_optin - static_smem - a.xbytes - scratch;
  int NS = (int)(avail / ((kNT / 32) * (int64_t)SB));
  if (NS > 4) NS = 4;
  if (NS < 1) return cudaErrorInvalidConfiguration;
  a.NS = NS;
  const int64_t smem_all = a.xbytes + (int64_t)(kNT / 32) * NS * SB + scratch;
  kern<<<(unsigned)grid, kNT, (size_t)smem_all, s>>>(a);
  return cudaGetLastError();
}

template <int DT, int V, int IS>
cudaError_t launch_t(const SpmvArgs& a, cudaStream_t s) {
  const bool multi = a.nchunks > 1 || a.T > 0;
  if (a.B == 32 && IS == 1) return multi ? launch_cfg<DT, V, IS, 32, true>(a, s) : launch_cfg<DT, V, IS, 32, false>(a, s);
  return multi ? launch_cfg<DT, V, IS, 0, true>(a, s) : launch_cfg<DT, V, IS, 0, false>(a, s);
}

template <int DT, int IS>
cudaError_t dispatch_v(const bsk::Geom& g, const SpmvArgs& a, cudaStream_t s) {
  switch (g.V) {
    case 1: return launch_t<DT, 1, IS>(a, s);
    case 2: return launch_t<DT, 2, IS>(a, s);
    case 4: return launch_t<DT, 4, IS>(a, s);
    default:
      if constexpr (DT != BS_F32) return launch_t<DT, 8, IS>(a, s);
      return cudaErrorInvalidValue;
  }
}

template <int DT>
cudaError_t dispatch_is(const bsk::Geom& g, const SpmvArgs& a, cudaStream_t s) {
  return g.is == 1 ? dispatch_v<DT, 1>(g, a, s) : dispatch_v<DT, 2>(g, a, s);
}

}  // namespace

cudaError_t bsk_launch_spmv(const bsk::Geom& g, const void* packed, const void* x, void* y, cudaStream_t s) {
  SpmvArgs a;
  const uint8_t* base = (const uint8_t*)packed;
  a.VA = base + g.offVA;
  a.VB = base + g.offVB;
  a.IA = base + g.offIA;
  a.IB = base + g.offIB;
  a.x = x;
  a.y = y;
  a.M = g.M; a.NB = g.NB; a.NBf = g.NBf; a.T = g.T; a.B = g.B; a.k = g.k;
  a.NS = 0;
  const bool aligned = ((uintptr_t)x & 15) == 0;
  a.xvec = aligned && (g.es == 2 ? g.B % 8 == 0 : g.B % 4 == 0);
  // chunking of the K dimension by whole panels (depends only on K, B, dtype: deterministic)
  const int64_t group_bytes = (int64_t)g.B * 128;                  // 32 blocks of 32-bit slots
  const int64_t panel_bytes = group_bytes * g.V;
  const int64_t tail_groups = (g.NB + 31) / 32 - g.NBf * g.V;
  if (g.NBf > 0 && g.k > 0) {
    int64_t PC = kXBudget / panel_bytes;
    if (PC < 1) PC = 1;
    if (PC > g.NBf) PC = g.NBf;
    int64_t nchunks = (g.NBf + PC - 1) / PC;
    if (nchunks > kMaxChunks) { nchunks = kMaxChunks; PC = (g.NBf + nchunks - 1) / nchunks; nchunks = (g.NBf + PC - 1) / PC; }
    const int64_t last_np = g.NBf - (nchunks - 1) * PC;
    a.PC = (int)PC;
    a.nchunks = (int)nchunks;
    a.tail_in_last = (last_np * g.V + tail_groups) * group_bytes <= kXBudget;
    int64_t xb = PC * panel_bytes;
    const int64_t need_last = (last_np * g.V + (a.tail_in_last ? tail_groups : 0)) * group_bytes;
    if (need_last > xb) xb = need_last;
    if (!a.tail_in_last && tail_groups * group_bytes > xb) xb = tail_groups * group_bytes;
    a.xbytes = (int)xb;
  } else {  // no full panels (or k == 0): the tail groups only
    a.PC = 1;
    a.nchunks = 0;
    a.tail_in_last = 0;
    a.xbytes = g.k > 0 ? (int)(tail_groups * group_bytes) : 0;
  }
  if (a.xbytes > bsk::dev_props().smem_optin - 16 * 1024) return cudaErrorInvalidConfiguration;
  switch (g.dt) {
    case BS_F32: return dispatch_is<BS_F32>(g, a, s);
    case BS_F16: return dispatch_is<BS_F16>(g, a, s);
    default: return dispatch_is<BS_BF16>(g, a, s);
  }
}
