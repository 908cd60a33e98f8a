// spmv.cu: K3 bs_spmv, y = W_bs · x for a balanced-sparse W in the SPMV (or SPMM) layout.
//
// Paper design (Fig. 3): one thread per block partition; every thread gets the same
// work because every block keeps k entries; x is "rearranged and stored in shared memory to
// avoid bank conflicts". The B200 version:
//   - A warp walks one row. Lane l owns the blocks b ≡ l (mod 32), V of them per panel of 32·V
//     blocks. Each lane streams its V values and V indices of a step with one 16-byte (values) and
//     one 8-byte (u8 indices) L1-bypassing load. The warp's loads are fully coalesced
//     (docs/layout.md).
//   - x is staged once per CTA in a block-interleaved order. Element (b, o) goes to 32-bit word
//     ((b>>5)·ceil(B/2) + (o>>1))·32 + (b&31), half o&1 (16-bit x), or to word
//     ((b>>5)·B + o)·32 + (b&31) (f32 x). Lane l only ever reads words in bank l, whatever the
//     indices are. So every gather is conflict-free by construction.
//   - For f16/bf16 each product is one FHFMA (exact 16x16 product, fp32 accumulate). Lanes keep V
//     independent accumulators. They are summed in a fixed order and reduced with a warp butterfly,
//     so y does not depend on the row range (row-sharding is bit-identical).
//   - The grid is persistent (SMs × CTAs per SM). Each CTA owns a contiguous, balanced row range.
#include "bs_common.cuh"
#include "bs_device.cuh"

namespace {

struct SpmvArgs {
  const uint8_t* VA;
  const uint8_t* VB;
  const uint8_t* IA;
  const uint8_t* IB;
  const void* x;
  void* y;
  int64_t M, NB, NBf, T;
  int B, k;
  int HB;        // words per lane-column of one group: ceil(B/2) for 16-bit x, B for f32
  int GS;        // bytes per group of 32 blocks in smem = HB * 128
  int NG;        // groups = ceil(NB / 32)
  int xvec;      // 1 if x is 16-byte aligned and B allows 16-byte staging loads
};

// Stage x into the block-interleaved smem layout. Warp w fills groups w, w+NW, ...; lane l copies
// block g*32 + l into its own bank column.
template <int ES>
__device__ __forceinline__ void stage_x(const SpmvArgs& a, uint32_t sx) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int g = warp; g < a.NG; g += nw) {
    const int64_t b = (int64_t)g * 32 + lane;
    if (b >= a.NB) continue;
    const uint32_t col = sx + (uint32_t)g * a.GS + lane * 4;  // word (g*HB + i)*32 + lane -> col + i*128
    if (ES == 2) {
      const uint16_t* xs = (const uint16_t*)a.x + b * a.B;
      if (a.xvec) {  // B % 8 == 0 and 16-byte aligned: 8 halves (4 words) per load
        for (int q = 0; q < a.B / 8; ++q) {
          const uint4 v = __ldg((const uint4*)xs + q);
          bsk::sts_u32(col + (4 * q + 0) * 128, v.x);
          bsk::sts_u32(col + (4 * q + 1) * 128, v.y);
          bsk::sts_u32(col + (4 * q + 2) * 128, v.z);
          bsk::sts_u32(col + (4 * q + 3) * 128, v.w);
        }
      } else {
        for (int o = 0; o < a.B; ++o) bsk::sts_u16(col + (o >> 1) * 128 + (o & 1) * 2, __ldg(xs + o));
      }
    } else {
      const uint32_t* xs = (const uint32_t*)a.x + b * a.B;
      if (a.xvec) {  // B % 4 == 0 and aligned
        for (int q = 0; q < a.B / 4; ++q) {
          const uint4 v = __ldg((const uint4*)xs + q);
          bsk::sts_u32(col + (4 * q + 0) * 128, v.x);
          bsk::sts_u32(col + (4 * q + 1) * 128, v.y);
          bsk::sts_u32(col + (4 * q + 2) * 128, v.z);
          bsk::sts_u32(col + (4 * q + 3) * 128, v.w);
        }
      } else {
        for (int o = 0; o < a.B; ++o) bsk::sts_u32(col + o * 128, __ldg(xs + o));
      }
    }
  }
}

// Byte offset of block-local offset o inside a lane's bank column.
template <int ES>
__device__ __forceinline__ uint32_t xofs(uint32_t o) {
  if (ES == 2) return ((o >> 1) << 7) | ((o & 1) << 1);
  return o << 7;
}

template <int DT, int V, int IS>
__global__ void __launch_bounds__(512, 2) spmv_kernel(SpmvArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  using raw_t = typename bsk::DTraits<DT>::raw_t;
  constexpr int ES = bsk::DTraits<DT>::kBytes;
  constexpr int U = V >= 4 ? 4 : 8;  // steps in flight per lane
  constexpr int P = 32 * V;
  const uint32_t sx = (uint32_t)__cvta_generic_to_shared(smem);
  stage_x<ES>(a, sx);
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t rb = (int64_t)blockIdx.x * a.M / gridDim.x;
  const int64_t re = (int64_t)(blockIdx.x + 1) * a.M / gridDim.x;
  const uint32_t sl = sx + lane * 4;
  const int64_t S = a.NBf * a.k;  // full-panel steps per row
  const int Vt = (int)((a.T + 31) / 32);

  for (int64_t r = rb + warp; r < re; r += nw) {
    float acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.f;

    // ---- full panels: S steps of P entries each, contiguous per row
    const int64_t e0 = r * S * P + lane * V;
    const uint8_t* vp = a.VA + e0 * ES;
    const uint8_t* ip = a.IA + e0 * IS;
    uint32_t pb = sl;  // smem base of the current panel: sl + p*V*GS
    int t = 0;
    for (int64_t s0 = 0; s0 < S; s0 += U) {
      bsk::Vec<V * ES> wv[U];
      bsk::Vec<V * IS> iv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (s0 + u < S) {
          wv[u].load(vp + (s0 + u) * (P * ES));
          iv[u].load(ip + (s0 + u) * (P * IS));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (s0 + u < S) {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const uint32_t o = IS == 1 ? bsk::get_u8(iv[u], v) : bsk::get_u16(iv[u], v);
            const uint32_t xa = pb + v * a.GS + xofs<ES>(o);
            const uint32_t xv = ES == 2 ? bsk::lds_u16(xa) : bsk::lds_u32(xa);
            const uint32_t w = ES == 2 ? bsk::get_u16(wv[u], v) : wv[u].w[v];
            bsk::fma_acc<DT>(acc[v], w, xv);
          }
          if (++t == a.k) {
            t = 0;
            pb += V * a.GS;
          }
        }
      }
    }

    // ---- tail: T blocks per row in (t, v, lane) order, one scalar entry per lane and v
    if (a.T > 0) {
      const int64_t f0 = r * a.k * a.T;
      const uint32_t tb = sl + (uint32_t)(a.NBf * V) * a.GS;
      const raw_t* vb = (const raw_t*)a.VB;
      for (int tt = 0; tt < a.k; ++tt) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int bl = v * 32 + lane;
          if (v < Vt && bl < a.T) {
            const int64_t e = f0 + (int64_t)tt * a.T + bl;
            const uint32_t w = vb[e];
            const uint32_t o = IS == 1 ? (uint32_t)a.IB[e] : (uint32_t)((const uint16_t*)a.IB)[e];
            const uint32_t xa = tb + v * a.GS + xofs<ES>(o);
            const uint32_t xv = ES == 2 ? bsk::lds_u16(xa) : bsk::lds_u32(xa);
            bsk::fma_acc<DT>(acc[v], w, xv);
          }
        }
      }
    }

    float sum = acc[0];
#pragma unroll
    for (int v = 1; v < V; ++v) sum += acc[v];
    sum = bsk::warp_sum_f(sum);
    if (lane == 0) ((raw_t*)a.y)[r] = (raw_t)bsk::from_float<DT>(sum);
  }
}

template <int DT, int V, int IS>
cudaError_t launch_t(const SpmvArgs& a, int smem, cudaStream_t s) {
  static bool configured = false;  // per instantiation
  auto kern = spmv_kernel<DT, V, IS>;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bsk::dev_props().smem_optin);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const auto& dp = bsk::dev_props();
  const int threads = 512;
  int ctas = dp.smem_per_sm / (smem + 1024);
  if (ctas > 2) ctas = 2;
  if (ctas < 1) ctas = 1;
  int64_t grid = (int64_t)dp.sms * ctas;
  const int64_t need = (a.M + (threads / 32) - 1) / (threads / 32);
  if (grid > need) grid = need;
  kern<<<(unsigned)grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}

template <int DT, int IS>
cudaError_t dispatch_v(const bsk::Geom& g, const SpmvArgs& a, int smem, cudaStream_t s) {
  switch (g.V) {
    case 1: return launch_t<DT, 1, IS>(a, smem, s);
    case 2: return launch_t<DT, 2, IS>(a, smem, s);
    case 4: return launch_t<DT, 4, IS>(a, smem, s);
    default:
      if constexpr (DT != BS_F32) return launch_t<DT, 8, IS>(a, smem, s);
      return cudaErrorInvalidValue;
  }
}

template <int DT>
cudaError_t dispatch_is(const bsk::Geom& g, const SpmvArgs& a, int smem, cudaStream_t s) {
  return g.is == 1 ? dispatch_v<DT, 1>(g, a, smem, s) : dispatch_v<DT, 2>(g, a, smem, s);
}

}  // namespace

// Bytes of shared memory the SpMV kernel needs for x (0 if it would not fit on one SM).
int64_t bsk_spmv_smem_bytes(const bsk::Geom& g) {
  const int64_t HB = g.es == 2 ? (g.B + 1) / 2 : g.B;
  const int64_t NG = (g.NB + 31) / 32;
  return NG * HB * 128;
}

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
  a.HB = g.es == 2 ? (g.B + 1) / 2 : g.B;
  a.GS = a.HB * 128;
  a.NG = (int)((g.NB + 31) / 32);
  const bool aligned = ((uintptr_t)x & 15) == 0;
  a.xvec = aligned && (g.es == 2 ? g.B % 8 == 0 : g.B % 4 == 0);
  const int64_t smem = bsk_spmv_smem_bytes(g);
  if (smem > bsk::dev_props().smem_optin) return cudaErrorInvalidConfiguration;
  switch (g.dt) {
    case BS_F32: return dispatch_is<BS_F32>(g, a, (int)smem, s);
    case BS_F16: return dispatch_is<BS_F16>(g, a, (int)smem, s);
    default: return dispatch_is<BS_BF16>(g, a, (int)smem, s);
  }
}
