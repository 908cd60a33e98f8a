// spmm.cu: K4 bs_spmm on CUDA cores, Y = W_bs · X for a small batch N (Fig. `benchmark`(b),
// batch 8).
//
// The SPMM layout is the SPMV layout with V = 1 (docs/layout.md): lane l owns block b ≡ l (mod 32)
// of each 32-block panel. X is staged per K-chunk in shared memory as 16-byte "plane slots". A slot
// holds one column c of X for NPL = 16/sizeof(D) consecutive batch columns. Slot (g, o, l), for block
// b = 32g + l and offset o, lives at ((g·B + o)·32 + l)·16 bytes of its plane. So a quarter-warp's
// LDS.128 gathers always cover 8 distinct 16-byte bank groups: conflict-free for any indices (the
// paper's rearranged x, with a batch vector per column).
//
// Per nnz a lane does QP LDS.128 and QP·NPL FMAs (FHFMA for 16-bit). Per-lane partials are reduced
// once per K-chunk with a transposing butterfly (lane l ends with column l>>s). Chunk partials are
// added in chunk order in shared memory. Chunk sizes depend only on (B, dtype), never on N, so
// every column sees the same arithmetic whatever the batch size (batch-sharding is bit-identical).
#include "bs_common.cuh"
#include "bs_device.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kRT = 32;  // rows per CTA tile

struct SpmmArgs {
  const uint8_t* A;   // panel steps: 32 values then 32 indices per step (V = 1)
  const uint8_t* Bt;  // tail values (element r·k·T + t·T + lane)
  const uint8_t* Ct;  // tail indices (same order)
  const void* X;
  void* Y;
  int64_t M, K, NB, NBf, T, N, ldx, ldy;
  int B, k;
  int CP;       // panels per chunk
  int nchunks;  // ceil(NBf / CP) + (T > 0)
  int planes;   // NQ = ceil(N / NPL)
  int xvec;
};

template <int ES>
__device__ __forceinline__ void stage_chunk(const SpmmArgs& a, uint32_t sx, int64_t g0, int ng, int q0, int QP,
                                            int plane_bytes) {
  constexpr int NPL = 16 / ES;
  // slots: (q, gl, l, o) with o fastest so that global reads of X are contiguous in c
  const int64_t nslots = (int64_t)QP * ng * 32 * a.B;
  for (int64_t i = threadIdx.x; i < nslots; i += blockDim.x) {
    const int o = (int)(i % a.B);
    int64_t rest = i / a.B;
    const int l = (int)(rest % 32);
    rest /= 32;
    const int gl = (int)(rest % ng);
    const int q = (int)(rest / ng);
    const int64_t b = (g0 + gl) * 32 + l;
    const int64_t c = b * a.B + o;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    if (b < a.NB) {
#pragma unroll
      for (int j = 0; j < NPL; ++j) {
        const int64_t n = (int64_t)(q0 + q) * NPL + j;
        if (n < a.N) {
          if (ES == 2) {
            const uint32_t h = __ldg((const uint16_t*)a.X + n * a.ldx + c);
            w[j >> 1] |= h << (16 * (j & 1));
          } else {
            w[j] = __ldg((const uint32_t*)a.X + n * a.ldx + c);
          }
        }
      }
    }
    const uint32_t addr = sx + (uint32_t)q * plane_bytes + (uint32_t)(((gl * a.B + o) * 32 + l) * 16);
    bsk::sts_v4(addr, w[0], w[1], w[2], w[3]);
  }
}

// Transposing butterfly over NV per-lane values. Afterwards lane l holds the warp total of value
// (l >> (5 - log2 NV)). The pairing sequence (xor 16, 8, 4, 2, 1) is the same for every value, so
// each value is summed with the same tree whatever NV is.
template <int NV>
__device__ __forceinline__ float transpose_reduce(float (&v)[NV], int lane) {
  int n = NV;
  int off = 16;
#pragma unroll
  for (int step = 0; step < 5; ++step) {
    if (n > 1) {
      const int half = n >> 1;
      const bool sel = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < NV / 2; ++i) {
        if (i < half) {
          const float send = sel ? v[i] : v[i + half];
          const float keep = sel ? v[i + half] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      n = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    }
    off >>= 1;
  }
  return v[0];
}

template <int DT, int QP, int IS>
__global__ void __launch_bounds__(kThreads) spmm_kernel(SpmmArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  using raw_t = typename bsk::DTraits<DT>::raw_t;
  constexpr int ES = bsk::DTraits<DT>::kBytes;
  constexpr int NPL = 16 / ES;
  constexpr int NV = QP * NPL;
  constexpr int LOGNV = NV == 4 ? 2 : NV == 8 ? 3 : NV == 16 ? 4 : 5;
  constexpr int U = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int plane_bytes = a.CP * 32 * a.B * 16;
  float* partial = (float*)(smem + (size_t)QP * plane_bytes);  // [kRT][NV]
  const uint32_t sx = (uint32_t)__cvta_generic_to_shared(smem);
  const int64_t r0 = (int64_t)blockIdx.x * kRT;
  const int64_t S = a.NBf * a.k;

  for (int q0 = 0; q0 < a.planes; q0 += QP) {
    for (int ch = 0; ch < a.nchunks; ++ch) {
      const int64_t p0 = (int64_t)ch * a.CP;
      const bool tail_chunk = p0 >= a.NBf;  // the tail group gets its own chunk
      const int ng = tail_chunk ? 1 : (int)min((int64_t)a.CP, a.NBf - p0);
      __syncthreads();  // previous chunk's smem reads are done
      stage_chunk<ES>(a, sx, tail_chunk ? a.NBf : p0, ng, q0, QP, plane_bytes);
      __syncthreads();
      for (int rl = warp; rl < kRT; rl += nw) {
        const int64_t r = r0 + rl;
        if (r >= a.M) break;
        float acc[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) acc[i] = 0.f;
        const uint32_t sl = sx + lane * 16;
        if (!tail_chunk) {
          const int64_t s_begin = p0 * a.k, s_end = (p0 + ng) * a.k;
          constexpr int STEPB = 32 * (ES + IS);
          const raw_t* vp = (const raw_t*)(a.A + r * S * STEPB) + lane;        // + s·STEPB bytes
          const uint8_t* ip = a.A + r * S * STEPB + 32 * ES + lane * IS;
          for (int64_t s0 = s_begin; s0 < s_end; s0 += U) {
            uint32_t wv[U], iv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (s0 + u < s_end) {
                wv[u] = *(const raw_t*)((const uint8_t*)vp + (s0 + u) * STEPB);
                iv[u] = IS == 1 ? (uint32_t)ip[(s0 + u) * STEPB] : (uint32_t)*(const uint16_t*)(ip + (s0 + u) * STEPB);
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (s0 + u < s_end) {
                const int gl = (int)((s0 + u) / a.k - p0);
                const uint32_t slot = sl + (uint32_t)((gl * a.B + (int)iv[u]) * 32 * 16);
#pragma unroll
                for (int q = 0; q < QP; ++q) {
                  uint32_t x4[4];
                  bsk::lds_v4(slot + q * plane_bytes, x4[0], x4[1], x4[2], x4[3]);
#pragma unroll
                  for (int j = 0; j < NPL; ++j) {
                    const uint32_t xv = ES == 2 ? (x4[j >> 1] >> (16 * (j & 1))) & 0xffffu : x4[j];
                    bsk::fma_acc<DT>(acc[q * NPL + j], wv[u], xv);
                  }
                }
              }
            }
          }
        } else {
          const raw_t* vb = (const raw_t*)a.Bt + r * a.k * a.T;
          const uint8_t* ib = a.Ct + r * a.k * a.T * IS;
          if (lane < a.T) {
            for (int t = 0; t < a.k; ++t) {
              const uint32_t w = vb[t * a.T + lane];
              const uint32_t o = IS == 1 ? (uint32_t)ib[t * a.T + lane] : (uint32_t)((const uint16_t*)ib)[t * a.T + lane];
              const uint32_t slot = sl + (uint32_t)((int)o * 32 * 16);
#pragma unroll
              for (int q = 0; q < QP; ++q) {
                uint32_t x4[4];
                bsk::lds_v4(slot + q * plane_bytes, x4[0], x4[1], x4[2], x4[3]);
#pragma unroll
                for (int j = 0; j < NPL; ++j) {
                  const uint32_t xv = ES == 2 ? (x4[j >> 1] >> (16 * (j & 1))) & 0xffffu : x4[j];
                  bsk::fma_acc<DT>(acc[q * NPL + j], w, xv);
                }
              }
            }
          }
        }
        const float tot = transpose_reduce<NV>(acc, lane);
        if ((lane & ((1 << (5 - LOGNV)) - 1)) == 0) {
          const int col = lane >> (5 - LOGNV);
          float* pp = partial + rl * NV + col;
          *pp = ch == 0 ? tot : *pp + tot;
        }
      }
    }
    __syncthreads();
    // write this pass's columns
    for (int i = threadIdx.x; i < kRT * NV; i += blockDim.x) {
      const int col = i / kRT, rl = i % kRT;
      const int64_t r = r0 + rl;
      const int64_t n = (int64_t)q0 * NPL + col;
      if (r < a.M && n < a.N) ((raw_t*)a.Y)[n * a.ldy + r] = (raw_t)bsk::from_float<DT>(partial[rl * NV + col]);
    }
  }
}

template <int DT, int QP, int IS>
cudaError_t launch_t(const SpmmArgs& a, int smem, cudaStream_t s) {
  static bool configured = false;
  auto kern = spmm_kernel<DT, QP, IS>;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bsk::dev_props().smem_optin);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int64_t grid = (a.M + kRT - 1) / kRT;
  kern<<<(unsigned)grid, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

template <int DT, int IS>
cudaError_t dispatch_qp(int QP, const SpmmArgs& a, int smem, cudaStream_t s) {
  if (QP == 1) return launch_t<DT, 1, IS>(a, smem, s);
  if (QP == 2) return launch_t<DT, 2, IS>(a, smem, s);
  return launch_t<DT, 4, IS>(a, smem, s);
}

}  // namespace

// Returns cudaErrorNotSupported when the shape needs the per-column fallback (caller loops SpMV).
cudaError_t bsk_launch_spmm(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx,
                            void* Y, int64_t ldy, cudaStream_t s) {
  if (g.layout != BS_LAYOUT_SPMM || g.V != 1) return cudaErrorNotSupported;
  const int NPL = 16 / g.es;
  const int64_t cols_per_panel = 32LL * g.B;
  int CP = (int)(2048 / cols_per_panel);
  if (CP < 1) CP = 1;
  const int64_t plane_bytes = (int64_t)CP * cols_per_panel * 16;
  const int planes = (int)((N + NPL - 1) / NPL);
  int QP = planes >= 4 ? 4 : planes >= 2 ? 2 : 1;
  const int64_t budget = 200 * 1024;
  while (QP > 1 && QP * plane_bytes + (int64_t)kRT * QP * NPL * 4 > budget) QP >>= 1;
  const int64_t smem = QP * plane_bytes + (int64_t)kRT * QP * NPL * 4;
  if (smem > bsk::dev_props().smem_optin) return cudaErrorNotSupported;
  SpmmArgs a;
  const uint8_t* base = (const uint8_t*)packed;
  a.A = base + g.offA; a.Bt = base + g.offB; a.Ct = base + g.offC;
  a.X = X; a.Y = Y;
  a.M = g.M; a.K = g.K; a.NB = g.NB; a.NBf = g.NBf; a.T = g.T; a.N = N; a.ldx = ldx; a.ldy = ldy;
  a.B = g.B; a.k = g.k; a.CP = CP;
  a.nchunks = (int)((g.NBf + CP - 1) / CP) + (g.T > 0 ? 1 : 0);
  a.planes = planes;
  a.xvec = 0;
  switch (g.dt) {
    case BS_F32: return g.is == 1 ? dispatch_qp<BS_F32, 1>(QP, a, (int)smem, s) : dispatch_qp<BS_F32, 2>(QP, a, (int)smem, s);
    case BS_F16: return g.is == 1 ? dispatch_qp<BS_F16, 1>(QP, a, (int)smem, s) : dispatch_qp<BS_F16, 2>(QP, a, (int)smem, s);
    default: return g.is == 1 ? dispatch_qp<BS_BF16, 1>(QP, a, (int)smem, s) : dispatch_qp<BS_BF16, 2>(QP, a, (int)smem, s);
  }
}
