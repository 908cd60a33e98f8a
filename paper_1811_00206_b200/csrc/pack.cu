// pack.cu: K2 bs_pack / bs_unpack, pure permutations between canonical and packed layouts.
//
// The layout is written from docs/layout.md. One thread per packed entry computes the canonical
// source (gather), so packed writes are close to coalesced. The paper describes no W layout (SURVEY
// A12); the layout choice is explained in DESIGN.md §4.
#include "bs_common.cuh"

namespace {

struct PackArgs {
  int64_t M, NB, NBf, T, P;
  int V, k, es, is;
  int64_t ri;  // index run bytes per step (160: 5-bit runs, 128: 4-bit runs; both written by pack_idx_runs_kernel)
  int64_t offA, offB, offC;
};

template <typename VT>
__global__ void pack_kernel(const VT* __restrict__ vals, const uint16_t* __restrict__ idx, PackArgs a,
                            uint8_t* __restrict__ base, int64_t nA, int64_t nB, bool unpack,
                            VT* __restrict__ out_vals, uint16_t* __restrict__ out_idx) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t step_bytes = a.P * a.es + a.ri;
  const bool runs = a.ri != a.P * a.is;
  const int64_t kT = (int64_t)a.k * a.T;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nA + nB; e += stride) {
    int64_t src;
    uint8_t* vdst;
    uint8_t* idst;
    if (e < nA) {
      // region A: step s = (r·NBf + p)·k + t holds P values then P indices; position l·V + v
      const int64_t s = e / a.P, pos = e - s * a.P;
      const int t = (int)(s % a.k);
      const int64_t rp = s / a.k;  // r·NBf + p
      const int64_t p = rp % a.NBf, r = rp / a.NBf;
      const int l = (int)(pos / a.V), v = (int)(pos % a.V);
      const int64_t b = p * a.P + (int64_t)v * 32 + l;
      src = (r * a.NB + b) * a.k + t;
      uint8_t* step = base + a.offA + s * step_bytes;
      vdst = step + pos * a.es;
      idst = step + a.P * a.es + pos * a.is;
    } else {
      // regions B / C: tail values / indices; element r·k·T + t·T + (v·32 + l)
      const int64_t f = e - nA;
      const int64_t r = f / kT, q = f - r * kT;
      const int t = (int)(q / a.T);
      const int64_t b = a.NBf * a.P + (q - (int64_t)t * a.T);
      src = (r * a.NB + b) * a.k + t;
      vdst = base + a.offB + f * a.es;
      idst = base + a.offC + f * a.is;
    }
    if (runs && e < nA) {  // 5- or 4-bit runs: indices are packed per lane by pack_idx_runs_kernel
      const int64_t pos = e % a.P;
      const int l = (int)(pos / a.V), v = (int)(pos % a.V);
      if (!unpack) {
        *(VT*)vdst = vals[src];
      } else {
        const uint8_t* run = vdst - pos * a.es + a.P * a.es;
        const int nb = a.ri == 160 ? 5 : 4;
        uint64_t F = (uint64_t)(*(const uint32_t*)(run + 4 * l));
        if (nb == 5) F |= (uint64_t)run[128 + l] << 32;
        out_vals[src] = *(const VT*)vdst;
        out_idx[src] = (uint16_t)((F >> (nb * v)) & ((1u << nb) - 1u));
      }
      continue;
    }
    if (!unpack) {
      *(VT*)vdst = vals[src];
      const uint16_t o = idx[src];
      idst[0] = (uint8_t)(o & 0xff);
      if (a.is == 2) idst[1] = (uint8_t)(o >> 8);
    } else {
      out_vals[src] = *(const VT*)vdst;
      out_idx[src] = a.is == 1 ? (uint16_t)idst[0] : (uint16_t)(idst[0] | (idst[1] << 8));
    }
  }
}

// SPMV layout, one CTA per row (grid-stride): the row's canonical entries (NB·k values and indices,
// contiguous) are copied into shared memory with coalesced loads, then the row's panel steps (one
// contiguous run of region A) and its tail entries (regions B and C) are written in order, so both sides
// of the permutation are coalesced and the index arithmetic is per row, not per entry (the per-entry
// gather of pack_kernel needs six 64-bit divisions per entry). Used whenever a row fits shared memory.
// Index runs of one row (docs/layout.md), NB_ = 5 (B = 32) or 4 (B <= 16) bits per index, V = 8, 16-bit
// values: per (step, lane) the lane's 8 values (one 16-byte store) and its field sum_v idx << NB_·v (a word,
// and a byte for 5-bit runs). The width is a template parameter: with a run-time shift the round-1 5-bit
// pack ran 25 % slower (0.72 -> 0.90 ms at 65536^2).
template <int NB_, typename VT>
__device__ __forceinline__ void pack_runs(const VT* sv, const uint16_t* si, uint8_t* rowA, int64_t steps_row,
                                          int64_t step_bytes, uint32_t P, int k, uint32_t run_off) {
  constexpr uint32_t msk = (1u << NB_) - 1u;
  for (uint32_t e = threadIdx.x; e < (uint32_t)steps_row * 32u; e += blockDim.x) {
    const uint32_t st = e >> 5, l = e & 31u;
    const uint32_t p = st / (uint32_t)k, t = st - p * (uint32_t)k;
    uint64_t F = 0;
    uint32_t vw[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const uint32_t c = (p * P + v * 32u + l) * k + t;
      F |= (uint64_t)(si[c] & msk) << (NB_ * v);
      vw[v >> 1] |= (uint32_t)(uint16_t)sv[c] << (16 * (v & 1));
    }
    *(uint4*)(rowA + (int64_t)st * step_bytes + l * 16u) = make_uint4(vw[0], vw[1], vw[2], vw[3]);
    uint8_t* run = rowA + (int64_t)st * step_bytes + run_off;
    *(uint32_t*)(run + 4 * l) = (uint32_t)F;
    if constexpr (NB_ == 5) run[128 + l] = (uint8_t)(F >> 32);
  }
}

template <typename VT>
__global__ void __launch_bounds__(512) pack_row_kernel(const VT* __restrict__ vals, const uint16_t* __restrict__ idx,
                                                       PackArgs a, uint8_t* __restrict__ base) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int es = sizeof(VT);
  const int64_t nrow = a.NB * a.k;  // canonical entries per row
  VT* sv = (VT*)sm;
  uint16_t* si = (uint16_t*)(sm + bsk::align_up(nrow * es, 16));
  const int64_t step_bytes = a.P * es + a.ri;
  const bool runs = a.ri != a.P * a.is;
  const int k = a.k;
  const int64_t kT = (int64_t)k * a.T;
  const int64_t steps_row = a.NBf * k;
  for (int64_t r = blockIdx.x; r < a.M; r += gridDim.x) {
    // canonical row -> shared memory (16-byte loads when the row start allows it)
    const uint8_t* gv = (const uint8_t*)(vals + r * nrow);
    const uint8_t* gi = (const uint8_t*)(idx + r * nrow);
    auto copy_in = [&](uint8_t* dst, const uint8_t* src, int64_t bytes) {
      int64_t head = 0;
      if (((uintptr_t)src & 15) == 0) {
        const int64_t n16 = bytes / 16;
        for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) ((uint4*)dst)[i] = __ldcs((const uint4*)src + i);
        head = n16 * 16;
      }
      for (int64_t i = head + threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
    };
    copy_in((uint8_t*)sv, gv, nrow * es);
    copy_in((uint8_t*)si, gi, nrow * 2);
    __syncthreads();
    // region A: steps s = (r·NBf + p)·k + t; P values (position l·V + v = block p·P + v·32 + l) then the
    // index run
    uint8_t* rowA = base + a.offA + r * steps_row * step_bytes;
    // 32-bit index arithmetic inside a row (a row holds < 2^31 entries); P = 32·V is a power of two
    const uint32_t P = (uint32_t)a.P, lgP = 31u - __clz(P), V = (uint32_t)a.V, lgV = 31u - __clz(V);
    const uint32_t nvals = runs ? 0u : (uint32_t)(steps_row * a.P);  // 5-bit runs: values written below
    for (uint32_t e = threadIdx.x; e < nvals; e += blockDim.x) {
      const uint32_t st = e >> lgP;
      const uint32_t pos = e & (P - 1u);
      const uint32_t p = st / (uint32_t)k, t = st - p * (uint32_t)k;
      const uint32_t l = pos >> lgV, v = pos & (V - 1u);
      const uint32_t b = p * P + v * 32u + l;
      *(VT*)(rowA + (int64_t)st * step_bytes + pos * es) = sv[b * k + t];
      if (!runs) {
        uint8_t* idst = rowA + st * step_bytes + a.P * es + pos * a.is;
        const uint16_t o = si[b * k + t];
        idst[0] = (uint8_t)(o & 0xff);
        if (a.is == 2) idst[1] = (uint8_t)(o >> 8);
      }
    }
    if (runs) {  // 5-bit runs (B = 32) or 4-bit runs (B <= 16), V = 8, 16-bit values (pack_runs)
      if (a.ri == 160) pack_runs<5>(sv, si, rowA, steps_row, step_bytes, P, k, (uint32_t)(a.P * es));
      else pack_runs<4>(sv, si, rowA, steps_row, step_bytes, P, k, (uint32_t)(a.P * es));
    }
    // regions B / C: the row's tail, element t·T + q (q = v·32 + l) = block NBf·P + q, entry t
    if (kT > 0) {
      VT* tv = (VT*)(base + a.offB) + r * kT;
      uint8_t* ti = base + a.offC + r * kT * a.is;
      const uint32_t T = (uint32_t)a.T, b0 = (uint32_t)(a.NBf * a.P);
      for (uint32_t f = threadIdx.x; f < (uint32_t)kT; f += blockDim.x) {
        const uint32_t t = f / T, q = f - t * T;
        const uint32_t c = (b0 + q) * k + t;
        tv[f] = sv[c];
        const uint16_t o = si[c];
        ti[f * a.is] = (uint8_t)(o & 0xff);
        if (a.is == 2) ti[f * a.is + 1] = (uint8_t)(o >> 8);
      }
    }
    __syncthreads();
  }
}

// SP24 metadata: byte (r, c) holds blocks b = 2c, 2c+1 of row r as nibbles idx0 | idx1 << 2.
// 5-bit / 4-bit index runs (docs/layout.md): one thread per (step, lane) builds the field
// F_l = sum_v idx(l, v) << nb·v of its 8 indices and writes word l of the u32 plane (and, for nb = 5, byte l of
// the byte plane).
__global__ void pack_idx_runs_kernel(const uint16_t* __restrict__ idx, PackArgs a, uint8_t* __restrict__ base, int64_t nsl) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t step_bytes = a.P * a.es + a.ri;
  const int nb = a.ri == 160 ? 5 : 4;
  const uint32_t msk = (1u << nb) - 1u;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nsl; e += stride) {
    const int64_t s = e >> 5;
    const int l = (int)(e & 31);
    const int t = (int)(s % a.k);
    const int64_t rp = s / a.k;
    const int64_t p = rp % a.NBf, r = rp / a.NBf;
    uint64_t F = 0;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int64_t b = p * a.P + (int64_t)v * 32 + l;
      F |= (uint64_t)(idx[(r * a.NB + b) * a.k + t] & msk) << (nb * v);
    }
    uint8_t* run = base + a.offA + s * step_bytes + a.P * a.es;
    *(uint32_t*)(run + 4 * l) = (uint32_t)F;
    if (nb == 5) run[128 + l] = (uint8_t)(F >> 32);
  }
}

__global__ void sp24_meta_kernel(const uint16_t* __restrict__ idx, int64_t nbytes, uint8_t* __restrict__ meta,
                                 bool unpack, uint16_t* __restrict__ out_idx) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nbytes; i += stride) {
    // canonical positions of the two blocks: (2i)*2 and (2i+1)*2 (k = 2)
    if (!unpack) {
      const uint16_t* p = idx + 4 * i;
      meta[i] = (uint8_t)((p[0] | (p[1] << 2)) | ((p[2] | (p[3] << 2)) << 4));
    } else {
      const uint8_t m = meta[i];
      uint16_t* p = out_idx + 4 * i;
      p[0] = m & 3; p[1] = (m >> 2) & 3; p[2] = (m >> 4) & 3; p[3] = (m >> 6) & 3;
    }
  }
}

// SPMM layout (docs/layout.md): one thread per canonical entry src = (r·NB + b)·k + t'; its blob is
// (tile r/128, chunk b/CB), position ((r mod 128)·cb + b mod CB)·k + t'.
template <typename VT>
__global__ void pack_spmm_kernel(const VT* __restrict__ vals, const uint16_t* __restrict__ idx, int64_t M, int64_t NB,
                                 int k, int CB, int is, int64_t tile_stride, uint8_t* __restrict__ base, bool unpack,
                                 VT* __restrict__ out_vals, uint16_t* __restrict__ out_idx) {
  constexpr int es = sizeof(VT);
  const int64_t n = M * NB * k;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t NCh = (NB + CB - 1) / CB;
  for (int64_t src = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; src < n; src += stride) {
    const int tp = (int)(src % k);
    const int64_t rb = src / k;
    const int64_t b = rb % NB, r = rb / NB;
    const int64_t t = r / 128, rl = r - t * 128;
    const int64_t mt = (M - 128 * t) < 128 ? (M - 128 * t) : 128;
    const int64_t c = b / CB, j = b - c * CB;
    const int64_t cb = (NB - CB * c) < CB ? (NB - CB * c) : CB;
    const int64_t blobCB = bsk::align_up(mt * CB * k * es, 16) + bsk::align_up(mt * CB * k * is, 16);
    uint8_t* blob = base + t * tile_stride + c * blobCB;
    const int64_t pos = (rl * cb + j) * k + tp;
    uint8_t* vdst = blob + pos * es;
    uint8_t* idst = blob + bsk::align_up(mt * cb * k * es, 16) + pos * is;
    (void)NCh;
    if (!unpack) {
      *(VT*)vdst = vals[src];
      const uint16_t o = idx[src];
      idst[0] = (uint8_t)(o & 0xff);
      if (is == 2) idst[1] = (uint8_t)(o >> 8);
    } else {
      out_vals[src] = *(const VT*)vdst;
      out_idx[src] = is == 1 ? (uint16_t)idst[0] : (uint16_t)(idst[0] | (idst[1] << 8));
    }
  }
}

cudaError_t zero_gap(uint8_t* base, int64_t from, int64_t to, cudaStream_t s) {
  if (to > from) return cudaMemsetAsync(base + from, 0, (size_t)(to - from), s);
  return cudaSuccess;
}

cudaError_t run(const bsk::Geom& g, const void* vals, const uint16_t* idx, void* packed, bool unpack,
                void* out_vals, uint16_t* out_idx, cudaStream_t s) {
  uint8_t* base = (uint8_t*)packed;
  const int sms = bsk::dev_props().sms;
  cudaError_t err;
  if (g.layout == BS_LAYOUT_SP24) {
    const int64_t nv = g.M * (g.K / 2);
    const int64_t nmeta = g.M * (g.NB / 2);
    if (!unpack) {
      if ((err = cudaMemcpyAsync(base, vals, (size_t)(nv * g.es), cudaMemcpyDeviceToDevice, s))) return err;
      if ((err = zero_gap(base, nv * g.es, g.offB, s))) return err;
      if ((err = zero_gap(base, g.offB + nmeta, g.total, s))) return err;
    } else {
      if ((err = cudaMemcpyAsync(out_vals, base, (size_t)(nv * g.es), cudaMemcpyDeviceToDevice, s))) return err;
    }
    int64_t blocks = (nmeta + 255) / 256;
    if (blocks > (int64_t)sms * 32) blocks = (int64_t)sms * 32;
    if (blocks < 1) blocks = 1;
    sp24_meta_kernel<<<(unsigned)blocks, 256, 0, s>>>(idx, nmeta, base + g.offB, unpack, out_idx);
    return cudaGetLastError();
  }
  if (g.layout == BS_LAYOUT_SPMM) {
    if (!unpack && (err = cudaMemsetAsync(base, 0, (size_t)g.total, s))) return err;  // blob padding
    const int64_t n = g.M * g.NB * g.k;
    if (n == 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sms * 32) blocks = (int64_t)sms * 32;
    if (g.es == 4)
      pack_spmm_kernel<uint32_t><<<(unsigned)blocks, 256, 0, s>>>((const uint32_t*)vals, idx, g.M, g.NB, g.k, g.V, g.is,
                                                                 g.offB, base, unpack, (uint32_t*)out_vals, out_idx);
    else
      pack_spmm_kernel<uint16_t><<<(unsigned)blocks, 256, 0, s>>>((const uint16_t*)vals, idx, g.M, g.NB, g.k, g.V, g.is,
                                                                 g.offB, base, unpack, (uint16_t*)out_vals, out_idx);
    return cudaGetLastError();
  }
  PackArgs a;
  a.M = g.M; a.NB = g.NB; a.NBf = g.NBf; a.T = g.T; a.P = g.P; a.V = g.V; a.k = g.k; a.es = g.es; a.is = g.is;
  a.ri = g.ri;
  a.offA = g.offA; a.offB = g.offB; a.offC = g.offC;
  const int64_t nA = g.M * g.NBf * g.P * g.k, nB = g.M * g.T * g.k;
  if (!unpack) {
    if ((err = zero_gap(base, (nA / (g.P > 0 ? g.P : 1)) * (g.P * g.es + g.ri), g.offB, s))) return err;
    if ((err = zero_gap(base, g.offB + nB * g.es, g.offC, s))) return err;
    if ((err = zero_gap(base, g.offC + nB * g.is, g.total, s))) return err;
  }
  if (nA + nB == 0) return cudaSuccess;
  if (!unpack) {  // one CTA per row when the row's canonical entries fit shared memory
    const int64_t smem = bsk::align_up(g.NB * g.k * g.es, 16) + g.NB * g.k * 2;
    if (smem <= bsk::dev_props().smem_optin - 1024) {
      cudaError_t perr = cudaSuccess;
      const void* fn = g.es == 4 ? (const void*)pack_row_kernel<uint32_t> : (const void*)pack_row_kernel<uint16_t>;
      if (bsk::prepare_func(fn, &perr) < 0) return perr;
      int64_t grid = g.M < (int64_t)sms * 8 ? g.M : (int64_t)sms * 8;
      if (g.es == 4)
        pack_row_kernel<uint32_t><<<(unsigned)grid, 512, (size_t)smem, s>>>((const uint32_t*)vals, idx, a, base);
      else
        pack_row_kernel<uint16_t><<<(unsigned)grid, 512, (size_t)smem, s>>>((const uint16_t*)vals, idx, a, base);
      return cudaGetLastError();
    }
  }
  int64_t blocks = (nA + nB + 255) / 256;
  if (blocks > (int64_t)sms * 32) blocks = (int64_t)sms * 32;
  if (g.es == 4) {
    pack_kernel<uint32_t><<<(unsigned)blocks, 256, 0, s>>>((const uint32_t*)vals, idx, a, base, nA, nB, unpack,
                                                          (uint32_t*)out_vals, out_idx);
  } else {
    pack_kernel<uint16_t><<<(unsigned)blocks, 256, 0, s>>>((const uint16_t*)vals, idx, a, base, nA, nB, unpack,
                                                          (uint16_t*)out_vals, out_idx);
  }
  if (!unpack && nA > 0 && g.ri != g.P * g.is) {
    if ((err = cudaGetLastError())) return err;
    const int64_t nsl = nA / g.P * 32;  // (step, lane) pairs
    int64_t b5 = (nsl + 255) / 256;
    if (b5 > (int64_t)sms * 32) b5 = (int64_t)sms * 32;
    pack_idx_runs_kernel<<<(unsigned)b5, 256, 0, s>>>(idx, a, base, nsl);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t bsk_launch_pack(const void* vals, const uint16_t* idx, const bsk::Geom& g, void* packed,
                            cudaStream_t s) {
  return run(g, vals, idx, packed, false, nullptr, nullptr, s);
}

cudaError_t bsk_launch_unpack(const void* packed, const bsk::Geom& g, void* vals, uint16_t* idx,
                              cudaStream_t s) {
  return run(g, nullptr, nullptr, const_cast<void*>(packed), true, vals, idx, s);
}
