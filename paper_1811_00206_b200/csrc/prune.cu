// prune.cu: K1 bs_prune, one balance-aware pruning step (Alg. 1 inner loop).
//
// For each (row, block) the kernel keeps the k entries of largest magnitude, ties to the lower
// offset. A NaN ranks above +Inf and all NaNs are equal (docs/layout.md "Canonical form"). Alg. 1
// "sorts elements". Any selection that yields the same top-k set is equivalent,
// so the GPU selects by rank instead of sorting:
//   1. Map every element to an unsigned magnitude key: the abs bit pattern, with every NaN folded
//      onto one key just above Inf. For IEEE formats the unsigned order of these keys is the
//      magnitude order.
//   2. Find T, the k-th largest key, with a bitwise radix select. Each bit costs one warp ballot (or
//      one warp sum for wide blocks): T = max{t : #{key >= t} >= k}.
//   3. Keep every key > T, plus the first (k - #{key > T}) keys equal to T in offset order.
//   4. Compact the kept offsets in ascending order with a warp prefix count.
// Values are copied bit for bit. The result is a pure integer decision, so it matches the oracle
// bit-exactly.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "bs_common.cuh"
#include "bs_keys.cuh"

namespace {

using bsk::KeyOf;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Narrow blocks (B <= 32): a warp holds floor(32/B) blocks, one element per lane. Each segment of B
// lanes runs its own radix select through ballots masked to the segment. Each warp iteration covers
// `nseg` consecutive flattened blocks gid = r*NB + b.
template <int DT>
__global__ void __launch_bounds__(256) prune_narrow(const typename KeyOf<DT>::raw_t* __restrict__ W,
                                                    int64_t M, int64_t NB, int64_t ldw, int B, int k,
                                                    typename KeyOf<DT>::raw_t* __restrict__ vals,
                                                    uint16_t* __restrict__ idx) {
  using raw_t = typename KeyOf<DT>::raw_t;
  const int lane = threadIdx.x & 31;
  const int nseg = 32 / B;
  const int seg = lane / B;
  const int j = lane - seg * B;  // block-local offset held by this lane
  const bool lane_used = seg < nseg;
  const uint32_t segmask = lane_used ? ((B == 32) ? 0xffffffffu : (((1u << B) - 1u) << (seg * B))) : 0u;
  const uint32_t lt = lanemask_lt();
  const int64_t nblocks = M * NB;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int64_t g0 = wid * nseg; g0 < nblocks; g0 += warps * nseg) {
    const int64_t gid = g0 + seg;
    const bool valid = lane_used && gid < nblocks;
    raw_t raw = 0;
    if (valid) {
      const int64_t r = gid / NB, b = gid - r * NB;
      raw = W[r * ldw + b * B + j];
    }
    const uint32_t key = KeyOf<DT>::key((uint32_t)raw);
    uint32_t T = 0;
#pragma unroll
    for (int bit = KeyOf<DT>::kBits - 1; bit >= 0; --bit) {
      const uint32_t cand = T | (1u << bit);
      const uint32_t bal = __ballot_sync(0xffffffffu, valid && key >= cand);
      if (__popc(bal & segmask) >= k) T = cand;
    }
    const bool gt = valid && key > T;
    const bool eq = valid && key == T;
    const int ngt = __popc(__ballot_sync(0xffffffffu, gt) & segmask);
    const uint32_t eqmask = __ballot_sync(0xffffffffu, eq) & segmask;
    const bool keep = gt || (eq && __popc(eqmask & lt) < k - ngt);
    const uint32_t keepmask = __ballot_sync(0xffffffffu, keep) & segmask;
    if (keep) {
      const int pos = __popc(keepmask & lt);
      vals[gid * k + pos] = raw;
      idx[gid * k + pos] = (uint16_t)j;
    }
  }
}

__device__ __forceinline__ int warp_sum(int v) { return __reduce_add_sync(0xffffffffu, v); }

__device__ __forceinline__ int warp_excl_scan(int v, int lane) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x - v;
}

// Wide blocks (B > 32): one warp per block. Lane l owns the contiguous offsets [l*E, min(l*E+E, B))
// with E = ceil(B/32), so lane order is offset order. Counts are warp sums, and the tie rank and
// output slots are exclusive warp scans. Elements are re-read through L1 on every radix step.
template <int DT>
__global__ void __launch_bounds__(256) prune_wide(const typename KeyOf<DT>::raw_t* __restrict__ W,
                                                  int64_t M, int64_t NB, int64_t ldw, int B, int k,
                                                  typename KeyOf<DT>::raw_t* __restrict__ vals,
                                                  uint16_t* __restrict__ idx) {
  using raw_t = typename KeyOf<DT>::raw_t;
  const int lane = threadIdx.x & 31;
  const int E = (B + 31) / 32;
  const int j0 = min(lane * E, B), j1 = min(j0 + E, B);
  const int64_t nblocks = M * NB;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t gid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gid < nblocks; gid += warps) {
    const int64_t r = gid / NB, b = gid - r * NB;
    const raw_t* src = W + r * ldw + b * B;
    uint32_t T = 0;
    for (int bit = KeyOf<DT>::kBits - 1; bit >= 0; --bit) {
      const uint32_t cand = T | (1u << bit);
      int c = 0;
      for (int j = j0; j < j1; ++j) c += KeyOf<DT>::key((uint32_t)__ldg(src + j)) >= cand;
      if (warp_sum(c) >= k) T = cand;
    }
    int cgt = 0, ceq = 0;
    for (int j = j0; j < j1; ++j) {
      const uint32_t key = KeyOf<DT>::key((uint32_t)__ldg(src + j));
      cgt += key > T;
      ceq += key == T;
    }
    const int need = k - warp_sum(cgt);
    int eq_before = warp_excl_scan(ceq, lane);
    // kept count per lane, then output slots
    int ckeep = 0;
    {
      int e = eq_before;
      for (int j = j0; j < j1; ++j) {
        const uint32_t key = KeyOf<DT>::key((uint32_t)__ldg(src + j));
        if (key > T) ++ckeep;
        else if (key == T) { ckeep += e < need; ++e; }
      }
    }
    int pos = warp_excl_scan(ckeep, lane);
    int e = eq_before;
    for (int j = j0; j < j1; ++j) {
      const raw_t raw = __ldg(src + j);
      const uint32_t key = KeyOf<DT>::key((uint32_t)raw);
      bool keep = key > T;
      if (key == T) { keep = e < need; ++e; }
      if (keep) {
        vals[gid * k + pos] = raw;
        idx[gid * k + pos] = (uint16_t)j;
        ++pos;
      }
    }
  }
}

// Thread per block (B in {4, 8, 16, 32}, rows 16-byte aligned): a thread loads its whole block with
// 16-byte loads (a warp reads 32 consecutive blocks: coalesced) and selects in registers, so the
// kernel streams W at HBM speed instead of one 2-byte load per lane per warp step (prune_narrow).
// Selection, with keys as above and ties to the lower offset:
//   - min(k, B - k) <= 6: k passes of "largest untaken key, first in offset order" (or B - k passes
//     of "smallest kept key, last in offset order", removed), over a 32-bit taken mask;
//   - otherwise the radix select of prune_narrow on the thread's B keys (kBits counting passes).
// The kept set is the same as prune_narrow's (the top k under (key desc, offset asc)): bit-exact.
// Sorting network (bitonic), descending, fully unrolled: B·log2(B)·(log2(B)+1)/4 compare-exchanges of
// two IMNMX each (240 for B = 32), no data-dependent control flow.
template <int B>
__device__ __forceinline__ void sort_desc(uint32_t (&c)[B]) {
#pragma unroll
  for (int size = 2; size <= B; size <<= 1)
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1)
#pragma unroll
      for (int i = 0; i < B; ++i) {
        const int j = i ^ stride;
        if (j > i) {
          const uint32_t a = c[i], b = c[j];
          const bool desc = (i & size) == 0;
          c[i] = desc ? max(a, b) : min(a, b);
          c[j] = desc ? min(a, b) : max(a, b);
        }
      }
}

// The K largest of B unique composites, in c[0..K) (insertion into a sorted register list: 2K - 1 IMNMX
// per element).
template <int K, int B>
__device__ __forceinline__ void topk_front(uint32_t (&c)[B]) {
  uint32_t m[K];
#pragma unroll
  for (int i = 0; i < K; ++i) m[i] = 0u;
#pragma unroll
  for (int j = 0; j < B; ++j) {
    uint32_t x = c[j];
#pragma unroll
    for (int i = 0; i < K; ++i) {  // m[i] = max(m[i], x); x = the value pushed down
      const uint32_t hi = max(m[i], x);
      x = min(m[i], x);
      m[i] = hi;
    }
  }
#pragma unroll
  for (int i = 0; i < K; ++i) c[i] = m[i];
}

// Block-wide copy of `bytes` from shared to global memory: 16-byte stores where both sides are 16-byte
// aligned (the destination of a CTA step is, when vals/idx are), then the remaining bytes one by one.
__device__ __forceinline__ void copy_out(uint8_t* dst, const uint8_t* src, int64_t bytes) {
  int64_t head = 0;
  if (((uintptr_t)dst & 15) == 0) {
    const int64_t n16 = bytes / 16;
    for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) ((uint4*)dst)[i] = ((const uint4*)src)[i];
    head = n16 * 16;
  }
  for (int64_t i = head + threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}

// KS: 1..4 = the insertion list of that length (k == KS), 0 = the sorting network (any k); chosen at
// launch so that each instantiation holds one selection path (smaller code: instruction-fetch stalls were
// a quarter of the samples with the choice inside the loop)
template <int DT, int B, int KS = 0>
__global__ void __launch_bounds__(256) prune_thread(const typename KeyOf<DT>::raw_t* __restrict__ W,
                                                    int64_t M, int64_t NB, int64_t ldw, int k,
                                                    typename KeyOf<DT>::raw_t* __restrict__ vals,
                                                    uint16_t* __restrict__ idx) {
  using raw_t = typename KeyOf<DT>::raw_t;
  constexpr int ES = sizeof(raw_t);
  constexpr int NV = B * ES / 16;  // 16-byte loads per block
  // staged outputs: 256·k values, then 256·k indices; 16-bit: then the threads' raw blocks (padded rows)
  extern __shared__ __align__(16) uint8_t sm_out[];
  raw_t* sv = (raw_t*)sm_out;
  uint16_t* si = (uint16_t*)(sm_out + bsk::align_up(256LL * k * ES, 16));
  const uint32_t raw_off = (uint32_t)(bsk::align_up(256LL * k * ES, 16) + bsk::align_up(256LL * k * 2, 16));
  const int64_t nblocks = M * NB;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // the next block's loads are issued before the current block's selection (register double buffer)
  auto load = [&](int64_t g, uint32_t (&w)[B * ES / 4]) {
    const int64_t r = g / NB, b = g - r * NB;
    const uint4* src = (const uint4*)(W + r * ldw + b * B);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const uint4 v = __ldcs(src + q);  // streamed once: do not keep W in L2
      w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
  };
  uint32_t wn[B * ES / 4];
  int64_t base = (int64_t)blockIdx.x * blockDim.x;
  if (base + threadIdx.x < nblocks) load(base + threadIdx.x, wn);
  for (; base < nblocks; base += stride) {  // CTA-uniform: the CTA's 256 blocks are consecutive
    const int64_t gid = base + threadIdx.x;
    const bool valid = gid < nblocks;
    uint32_t w[B * ES / 4];
#pragma unroll
    for (int q = 0; q < B * ES / 4; ++q) w[q] = wn[q];
    if (gid + stride < nblocks) load(gid + stride, wn);
    uint32_t key[ES == 2 ? 1 : B];
    if constexpr (ES != 2) {
#pragma unroll
      for (int j = 0; j < B; ++j) key[j] = KeyOf<DT>::key(w[j]);
    }
    uint32_t taken = 0;
    if constexpr (ES == 2) {
      // 16-bit keys, two per 32-bit word: |w| is one LOP3 and the NaN fold (every NaN onto the key just
      // above Inf) one VIMNMX.U16x2 for both halves; c_j = key_j << 17 | (31 - j) << 12 is unique and
      // orders by magnitude, ties to the lower offset, so the kept set is the k largest composites: an
      // insertion list for k <= 4, else a sorting network, then the first k. The kept values are copied
      // bit for bit from this thread's raw words parked in shared memory (padded rows: conflict-free).
      constexpr uint32_t kNan2 = bsk::KeyOf<DT>::key(0x7fffu) * 0x10001u;  // the folded NaN key, both halves
      uint32_t c[B];
#pragma unroll
      for (int q = 0; q < B / 2; ++q) {
        const uint32_t a2 = __vminu2(w[q] & 0x7fff7fffu, kNan2);
        c[2 * q] = (a2 << 17) | ((31u - 2 * q) << 12);
        c[2 * q + 1] = ((a2 << 1) & 0xfffe0000u) | ((31u - (2 * q + 1)) << 12);
      }
      uint32_t* rawrow = (uint32_t*)(sm_out + raw_off) + threadIdx.x * (B / 2 + 4);
#pragma unroll
      for (int q = 0; q < B / 8; ++q)
        *(uint4*)(rawrow + 4 * q) = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
      if constexpr (KS > 0) topk_front<KS, B>(c);
      else sort_desc<B>(c);
#pragma unroll
      for (int p = 0; p < B; ++p)
        if (p < k) taken |= 1u << (31u - ((c[p] >> 12) & 31u));
      // kept entries in offset order: entry p goes to position popc(taken below its offset)
      if (valid) {
        const int t0 = threadIdx.x * k;
        const uint16_t* raw16 = (const uint16_t*)rawrow;
#pragma unroll
        for (int p = 0; p < B; ++p) {
          if (p < k) {
            const uint32_t j = 31u - ((c[p] >> 12) & 31u);
            const int pos = t0 + __popc(taken & ((1u << j) - 1u));
            sv[pos] = (raw_t)raw16[j];
            si[pos] = (uint16_t)j;
          }
        }
      }
    } else if (k <= 6) {
      for (int p = 0; p < k; ++p) {
        int best = -1, bi = 0;
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (!((taken >> j) & 1u) && (int)key[j] > best) { best = (int)key[j]; bi = j; }
        taken |= 1u << bi;
      }
    } else if (B - k <= 6) {
      uint32_t dropped = 0;
      for (int p = 0; p < B - k; ++p) {
        uint32_t best = 0xffffffffu;
        int bi = 0;
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (!((dropped >> j) & 1u) && key[j] <= best) { best = key[j]; bi = j; }
        dropped |= 1u << bi;
      }
      taken = ~dropped & (B == 32 ? 0xffffffffu : ((1u << B) - 1u));
    } else {
      uint32_t T = 0;
#pragma unroll
      for (int bit = KeyOf<DT>::kBits - 1; bit >= 0; --bit) {
        const uint32_t cand = T | (1u << bit);
        int c[4] = {0, 0, 0, 0};  // four independent counters: the count is not one serial chain
#pragma unroll
        for (int j = 0; j < B; ++j) c[j & 3] += key[j] >= cand;
        if ((c[0] + c[1]) + (c[2] + c[3]) >= k) T = cand;
      }
      int need = k;
#pragma unroll
      for (int j = 0; j < B; ++j) need -= key[j] > T;
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const bool keep = key[j] > T || (key[j] == T && need > 0);
        if (key[j] == T && need > 0) --need;
        taken |= (uint32_t)keep << j;
      }
    }
    // kept entries in offset order into shared memory, then the CTA writes its contiguous output run
    // with 16-byte stores (per-thread stores at stride k would touch a sector per 2-byte element)
    if (ES != 2 && valid) {
      int t = threadIdx.x * k;
#pragma unroll
      for (int j = 0; j < B; ++j) {
        if ((taken >> j) & 1u) {
          sv[t] = (raw_t)(ES == 2 ? (w[j >> 1] >> (16 * (j & 1))) & 0xffffu : w[j]);
          si[t] = (uint16_t)j;
          ++t;
        }
      }
    }
    __syncthreads();
    const int64_t nv = ((nblocks - base) < 256 ? (nblocks - base) : 256) * k;  // entries of this CTA step
    copy_out((uint8_t*)(vals + base * k), (const uint8_t*)sv, nv * ES);
    copy_out((uint8_t*)(idx + base * k), (const uint8_t*)si, nv * 2);
    __syncthreads();
  }
}

// Block ranks (bs_block_rank): thread per block (B <= 32). rank_j = #{i : key_i > key_j} +
// #{i < j : key_i == key_j}, the position of element j in the block's stable descending magnitude
// order; the count is integer-exact, so it equals the oracle's sort bit for bit.
template <int DT, int B>
__global__ void __launch_bounds__(256) block_rank_kernel(const typename KeyOf<DT>::raw_t* __restrict__ W,
                                                         int64_t M, int64_t NB, int64_t ldw,
                                                         uint8_t* __restrict__ rank, bool vec, bool rvec) {
  const int64_t nblocks = M * NB;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t K = NB * B;
  for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < nblocks; gid += stride) {
    const int64_t r = gid / NB, b = gid - r * NB;
    using raw_t = typename KeyOf<DT>::raw_t;
    constexpr int ES = sizeof(raw_t);
    const raw_t* src = W + r * ldw + b * B;
    constexpr bool PACK16 = ES == 2 && B >= 8;  // 16-bit, B >= 8: keys from raw words, two per word
    uint32_t key[PACK16 ? 1 : B];
    uint32_t wraw[PACK16 ? B / 2 : 1];
    if constexpr (PACK16) {
      if (B * ES % 16 == 0 && vec) {  // 16-byte loads (rows 16-byte aligned)
#pragma unroll
        for (int q = 0; q < B * ES / 16; ++q) {
          const uint4 v = __ldcs((const uint4*)src + q);
          wraw[4 * q] = v.x; wraw[4 * q + 1] = v.y; wraw[4 * q + 2] = v.z; wraw[4 * q + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < B / 2; ++q) wraw[q] = (uint32_t)__ldg(src + 2 * q) | ((uint32_t)__ldg(src + 2 * q + 1) << 16);
      }
    } else if constexpr (B * ES % 16 == 0) {
      if (vec) {  // 16-byte loads (rows 16-byte aligned)
        uint32_t w[B * ES / 4];
#pragma unroll
        for (int q = 0; q < B * ES / 16; ++q) {
          const uint4 v = __ldcs((const uint4*)src + q);
          w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int j = 0; j < B; ++j) key[j] = KeyOf<DT>::key(ES == 2 ? (w[j >> 1] >> (16 * (j & 1))) & 0xffffu : w[j]);
      } else {
#pragma unroll
        for (int j = 0; j < B; ++j) key[j] = KeyOf<DT>::key((uint32_t)__ldg(src + j));
      }
    } else {
#pragma unroll
      for (int j = 0; j < B; ++j) key[j] = KeyOf<DT>::key((uint32_t)__ldg(src + j));
    }
    uint8_t* dst = rank + r * K + b * B;
    uint32_t packed[(B + 3) / 4];
#pragma unroll
    for (int q = 0; q < (B + 3) / 4; ++q) packed[q] = 0;
    if constexpr (ES == 2 && B >= 8) {
      // 16-bit keys: sort the unique composites key << 5 | (31 - j) (a sorting network, 2·240 IMNMX for
      // B = 32, instead of B^2 comparisons); the element at sorted position p is j = 31 - (c_p & 31),
      // so rank_j = p, scattered through shared memory (no barrier needed: each thread reads back only its
      // own bytes). Byte j of thread t lives in word (j / 4)·256 + t, i.e. always in bank t mod 32: the
      // data-dependent byte stores and the word loads are conflict-free.
      __shared__ __align__(16) uint32_t srank[(B / 4) * 256];
      uint32_t c[B];
      {  // two keys per word: |w| one LOP3, the NaN fold one VIMNMX.U16x2 (as bs_prune_k)
        constexpr uint32_t kNan2 = KeyOf<DT>::key(0x7fffu) * 0x10001u;
#pragma unroll
        for (int q = 0; q < B / 2; ++q) {
          const uint32_t a2 = __vminu2(wraw[q] & 0x7fff7fffu, kNan2);
          c[2 * q] = (a2 << 17) | ((31u - 2 * q) << 12);
          c[2 * q + 1] = ((a2 << 1) & 0xfffe0000u) | ((31u - (2 * q + 1)) << 12);
        }
      }
      sort_desc<B>(c);
      uint8_t* my = (uint8_t*)(srank + threadIdx.x);
#pragma unroll
      for (int p = 0; p < B; ++p) {
        const uint32_t j = 31u - ((c[p] >> 12) & 31u);
        my[(j >> 2) * 1024u + (j & 3u)] = (uint8_t)p;
      }
#pragma unroll
      for (int q = 0; q < B / 4; ++q) packed[q] = srank[q * 256 + threadIdx.x];
    } else {
#pragma unroll
      for (int j = 0; j < B; ++j) {
        int c = 0;
#pragma unroll
        for (int i = 0; i < B; ++i) c += (key[i] > key[j]) || (i < j && key[i] == key[j]);
        packed[j >> 2] |= (uint32_t)c << (8 * (j & 3));
      }
    }
    bool wide = false;
    if constexpr (B % 4 == 0) wide = rvec;  // 32-bit stores when `rank` is 4-byte aligned (K, B multiples of 4)
    if (wide) {
#pragma unroll
      for (int q = 0; q < (B + 3) / 4; ++q) ((uint32_t*)dst)[q] = packed[q];
    } else {
#pragma unroll
      for (int j = 0; j < B; ++j) dst[j] = (uint8_t)(packed[j >> 2] >> (8 * (j & 3)));
    }
  }
}

template <int DT>
cudaError_t launch_block_rank_t(const void* W, int64_t M, int64_t K, int64_t ldw, int B, uint8_t* rank, cudaStream_t s) {
  using raw_t = typename KeyOf<DT>::raw_t;
  const int64_t NB = K / B;
  int64_t blocks = (M * NB + 255) / 256;
  const int sms = bsk::dev_props().sms;
  blocks = blocks < (int64_t)sms * 8 ? blocks : (int64_t)sms * 8;
  const bool vec = ((uintptr_t)W & 15) == 0 && (ldw * (int64_t)sizeof(raw_t)) % 16 == 0;
  const bool rvec = ((uintptr_t)rank & 3) == 0;  // bs.h does not require an aligned `rank`
  auto run = [&](auto kern) { kern<<<(unsigned)blocks, 256, 0, s>>>((const raw_t*)W, M, NB, ldw, rank, vec, rvec); };
  switch (B) {
    case 32: run(block_rank_kernel<DT, 32>); break;
    case 16: run(block_rank_kernel<DT, 16>); break;
    case 8: run(block_rank_kernel<DT, 8>); break;
    case 4: run(block_rank_kernel<DT, 4>); break;
    case 2: run(block_rank_kernel<DT, 2>); break;
    case 1: run(block_rank_kernel<DT, 1>); break;
    default: return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}

// The prune_thread instantiation for k (16-bit: an insertion list for k <= 4, the sorting network above).
template <int DT, int B, typename R>
void sel_k_impl(int k, R&& run) {
  if constexpr (sizeof(typename KeyOf<DT>::raw_t) == 2) {
    switch (k) {
      case 1: run(prune_thread<DT, B, 1>); return;
      case 2: run(prune_thread<DT, B, 2>); return;
      case 3: run(prune_thread<DT, B, 3>); return;
      case 4: run(prune_thread<DT, B, 4>); return;
      default: run(prune_thread<DT, B, 0>); return;
    }
  } else {
    run(prune_thread<DT, B, 0>);
  }
}

template <int DT>
cudaError_t launch_prune_t(const void* W, int64_t M, int64_t K, int64_t ldw, int B, int k, void* vals,
                           uint16_t* idx, cudaStream_t s) {
  using raw_t = typename KeyOf<DT>::raw_t;
  const int64_t NB = K / B;
  const int threads = 256;
  const int sms = bsk::dev_props().sms;
  const bool aligned16 = ((uintptr_t)W & 15) == 0 && (ldw * (int64_t)sizeof(raw_t)) % 16 == 0;
  if (aligned16 && k > 0 && (B == 32 || B == 16 || B == 8 || (B == 4 && sizeof(raw_t) == 4))) {
    int64_t blocks = (M * NB + 255) / 256;
    blocks = blocks < (int64_t)sms * 8 ? blocks : (int64_t)sms * 8;
    const size_t smem = (size_t)bsk::align_up(256LL * k * sizeof(raw_t), 16) + (size_t)bsk::align_up(256LL * k * 2, 16) +
                        (sizeof(raw_t) == 2 ? 256 * (size_t)(B * 2 + 16) : 0);
    auto run = [&](auto kern) {
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<(unsigned)blocks, 256, smem, s>>>((const raw_t*)W, M, NB, ldw, k, (raw_t*)vals, idx);
    };
    switch (B) {
      case 32: sel_k_impl<DT, 32>(k, run); break;
      case 16: sel_k_impl<DT, 16>(k, run); break;
      case 8: sel_k_impl<DT, 8>(k, run); break;
      default: if constexpr (sizeof(raw_t) == 4) run(prune_thread<DT, 4>); break;
    }
    return cudaGetLastError();
  }
  if (B <= 32) {
    const int nseg = 32 / B;
    const int64_t warps_needed = (M * NB + nseg - 1) / nseg;
    int64_t blocks = (warps_needed + 7) / 8;
    blocks = blocks < (int64_t)sms * 16 ? blocks : (int64_t)sms * 16;
    prune_narrow<DT><<<(unsigned)blocks, threads, 0, s>>>((const raw_t*)W, M, NB, ldw, B, k, (raw_t*)vals, idx);
  } else {
    int64_t blocks = (M * NB + 7) / 8;
    blocks = blocks < (int64_t)sms * 16 ? blocks : (int64_t)sms * 16;
    prune_wide<DT><<<(unsigned)blocks, threads, 0, s>>>((const raw_t*)W, M, NB, ldw, B, k, (raw_t*)vals, idx);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t bsk_launch_prune(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int B, int k,
                             void* vals, uint16_t* idx, cudaStream_t s) {
  switch (dt) {
    case BS_F32: return launch_prune_t<BS_F32>(W, M, K, ldw, B, k, vals, idx, s);
    case BS_F16: return launch_prune_t<BS_F16>(W, M, K, ldw, B, k, vals, idx, s);
    default: return launch_prune_t<BS_BF16>(W, M, K, ldw, B, k, vals, idx, s);
  }
}

cudaError_t bsk_launch_block_rank(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int B, uint8_t* rank,
                                  cudaStream_t s) {
  switch (dt) {
    case BS_F32: return launch_block_rank_t<BS_F32>(W, M, K, ldw, B, rank, s);
    case BS_F16: return launch_block_rank_t<BS_F16>(W, M, K, ldw, B, rank, s);
    default: return launch_block_rank_t<BS_BF16>(W, M, K, ldw, B, rank, s);
  }
}
