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
  int64_t ri;  // index run bytes per step (160: 5-bit runs, written by pack_idx5_kernel)
  int64_t offA, offB, offC;
};

template <typename VT>
__global__ void pack_kernel(const VT* __restrict__ vals, const uint16_t* __restrict__ idx, PackArgs a,
                            uint8_t* __restrict__ base, int64_t nA, int64_t nB, bool unpack,
                            VT* __restrict__ out_vals, uint16_t* __restrict__ out_idx) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t step_bytes = a.P * a.es + a.ri;
  const bool five = a.ri != a.P * a.is;
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
    if (five && e < nA) {  // 5-bit runs: indices are packed per lane by pack_idx5_kernel
      const int64_t pos = e % a.P;
      const int l = (int)(pos / a.V), v = (int)(pos % a.V);
      if (!unpack) {
        *(VT*)vdst = vals[src];
      } else {
        const uint8_t* run = vdst - pos * a.es + a.P * a.es;
        const uint64_t F = (uint64_t)(*(const uint32_t*)(run + 4 * l)) | ((uint64_t)run[128 + l] << 32);
        out_vals[src] = *(const VT*)vdst;
        out_idx[src] = (uint16_t)((F >> (5 * v)) & 31u);
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

// SP24 metadata: byte (r, c) holds blocks b = 2c, 2c+1 of row r as nibbles idx0 | idx1 << 2.
// 5-bit index runs (docs/layout.md): one thread per (step, lane) builds the 40-bit field
// F_l = sum_v idx(l, v) << 5v of its 8 indices and writes word l of the u32 plane and byte l of the byte plane.
__global__ void pack_idx5_kernel(const uint16_t* __restrict__ idx, PackArgs a, uint8_t* __restrict__ base, int64_t nsl) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t step_bytes = a.P * a.es + a.ri;
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
      F |= (uint64_t)(idx[(r * a.NB + b) * a.k + t] & 31u) << (5 * v);
    }
    uint8_t* run = base + a.offA + s * step_bytes + a.P * a.es;
    *(uint32_t*)(run + 4 * l) = (uint32_t)F;
    run[128 + l] = (uint8_t)(F >> 32);
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
    pack_idx5_kernel<<<(unsigned)b5, 256, 0, s>>>(idx, a, base, nsl);
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
