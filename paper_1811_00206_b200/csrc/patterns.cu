// patterns.cu: Alg. 1's pruned matrix in dense form and the comparison sparsity patterns of the
// paper's evaluation, as GPU mask generators (the mask schedule without retraining).
//
//   bs_decode       the dense W_bs (= Alg. 1's output M_p) from canonical (vals, idx): with
//                   bs_prune_k it is one pruning iteration of Alg. 1 on a dense matrix; iterating it
//                   along GraduallyIncrease is the gradual schedule.
//   bs_random_mask  random sparsity (Han et al.): magnitude pruning over the whole
//                   matrix, keeping the keep_count(M·K, s) largest |w| (ties to the lower row-major index).
//   bs_block_mask   block sparsity (Narang et al.): bh×bw tiles scored by max or mean |w|,
//                   the keep_count(#tiles, s) best tiles kept whole; vector sparsity (Mao et al.)
//                   is bh = 1, bw = K (rows) or bh = M, bw = 1 (columns).
//
// The global selections are a radix select over unsigned keys (the magnitude key of bs_keys.cuh for
// elements; the tile score's key for tiles), 8 bits per pass from the top: each pass builds a 256-bin
// histogram of the keys that match the digits found so far (integer atomics: the counts, and so the
// result, do not depend on the order of the atomics), and a one-thread kernel picks the next digit. After
// the last pass the threshold key T is exact; every key > T is kept, and of the keys == T the first
// `need` in index order, found with per-CTA counts and an in-CTA ballot scan. Everything is an integer
// decision on keys, so the masks equal the oracle's bit for bit. Nothing synchronises with the host.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "bs_common.cuh"
#include "bs_keys.cuh"

namespace {

constexpr int kSelThreads = 256;
constexpr int kMaxSelCtas = 1024;

struct SelState {
  unsigned long long prefix;  // digits of T found so far
  unsigned long long need;    // keys still to keep among those matching the prefix
  unsigned long long hist[256];
};

// ------------------------------------------------------------------ bs_decode

// One CTA step = one segment of kSeg output elements of one row: zero the segment in shared memory,
// scatter the kept entries of the blocks that overlap it, then store it with 16-byte stores.
constexpr int kSeg = 4096;

template <typename raw_t>
__global__ void __launch_bounds__(256) decode_kernel(const raw_t* __restrict__ vals, const uint16_t* __restrict__ idx,
                                                     int64_t M, int64_t K, int B, int k, raw_t* __restrict__ out,
                                                     int64_t ldo) {
  __shared__ __align__(16) raw_t seg[kSeg];
  const int64_t NB = K / B;
  const int64_t nseg = (K + kSeg - 1) / kSeg;
  for (int64_t job = blockIdx.x; job < M * nseg; job += gridDim.x) {
    const int64_t r = job / nseg, e0 = (job - r * nseg) * kSeg;
    const int64_t E = (K - e0) < kSeg ? (K - e0) : kSeg;
    for (int64_t i = threadIdx.x; i < kSeg * (int64_t)sizeof(raw_t) / 16; i += blockDim.x)
      ((uint4*)seg)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    const int64_t b0 = e0 / B, b1 = (e0 + E - 1) / B;  // blocks overlapping the segment
    const int64_t t0 = (r * NB + b0) * k, t1 = (r * NB + b1 + 1) * k;
    for (int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
      const int64_t b = t / k - r * NB;
      const int64_t pos = b * B + idx[t] - e0;
      if (pos >= 0 && pos < E) seg[pos] = vals[t];
    }
    __syncthreads();
    raw_t* dst = out + r * ldo + e0;
    const int64_t bytes = E * (int64_t)sizeof(raw_t);
    int64_t head = 0;
    if (((uintptr_t)dst & 15) == 0) {
      const int64_t n16 = bytes / 16;
      for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) ((uint4*)dst)[i] = ((const uint4*)seg)[i];
      head = n16 * 16 / (int64_t)sizeof(raw_t);
    }
    for (int64_t i = head + threadIdx.x; i < E; i += blockDim.x) dst[i] = seg[i];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ key sources

// Element keys of W (M×K, leading dimension ldw), index i = r·K + c (row-major).
template <int DT>
struct ElemKeys {
  using raw_t = typename bsk::KeyOf<DT>::raw_t;
  const raw_t* W;
  int64_t K, ldw;
  __device__ __forceinline__ uint64_t operator()(int64_t i) const {
    const int64_t off = ldw == K ? i : (i / K) * ldw + i % K;
    return bsk::KeyOf<DT>::key((uint32_t)W[off]);
  }
};

// Precomputed keys (the tile scores).
struct ArrayKeys {
  const uint64_t* key;
  __device__ __forceinline__ uint64_t operator()(int64_t i) const { return key[i]; }
};

template <int DT>
__device__ __forceinline__ double to_f64(uint32_t raw) {
  if constexpr (DT == BS_F32) return (double)__uint_as_float(raw);
  else if constexpr (DT == BS_F16) return (double)__half2float(__ushort_as_half((unsigned short)raw));
  else return (double)__bfloat162float(__ushort_as_bfloat16((unsigned short)raw));
}

// Tile scores (one thread per tile, tiles row-major): criterion 0 = max |w| as the element key (NaN
// above Inf); criterion 1 = the fp64 sum of |w| in row-major order inside the tile (the mean times the
// tile size), keyed by its bit pattern (non-negative doubles order as their bits), any NaN -> the top key.
template <int DT>
__global__ void __launch_bounds__(256) tile_score_kernel(const typename bsk::KeyOf<DT>::raw_t* __restrict__ W,
                                                         int64_t ldw, int64_t TR, int64_t TC, int64_t bh,
                                                         int64_t bw, int criterion, uint64_t* __restrict__ key) {
  const int64_t n = TR * TC;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tr = t / TC, tc = t - tr * TC;
    const auto* base = W + tr * bh * ldw + tc * bw;
    uint64_t out;
    if (criterion == 0) {
      uint32_t mx = 0;
      for (int64_t i = 0; i < bh; ++i)
        for (int64_t j = 0; j < bw; ++j) {
          const uint32_t kk = bsk::KeyOf<DT>::key((uint32_t)base[i * ldw + j]);
          mx = kk > mx ? kk : mx;
        }
      out = mx;
    } else {
      double sum = 0.0;
      bool nan = false;
      for (int64_t i = 0; i < bh; ++i)
        for (int64_t j = 0; j < bw; ++j) {
          const double v = to_f64<DT>((uint32_t)base[i * ldw + j]);
          if (v != v) nan = true;
          else sum += fabs(v);
        }
      out = nan ? ~0ULL : (uint64_t)__double_as_longlong(sum);
    }
    key[t] = out;
  }
}

// ------------------------------------------------------------------ radix select

__global__ void sel_init_kernel(SelState* st, unsigned long long need) {
  const int i = threadIdx.x;
  if (i < 256) st->hist[i] = 0;
  if (i == 0) {
    st->prefix = 0;
    st->need = need;
  }
}

template <class Src>
__global__ void __launch_bounds__(kSelThreads) hist_kernel(Src src, int64_t n, SelState* st, int shift) {
  __shared__ unsigned int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned long long prefix = st->prefix;
  const unsigned long long hi = shift >= 56 ? 0ULL : (~0ULL << (shift + 8));  // digits already fixed
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = src(i);
    if (((key ^ prefix) & hi) == 0) atomicAdd(&h[(key >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&st->hist[i], (unsigned long long)h[i]);
}

// Picks the digit at `shift`: the highest bin d with #{keys above d} < need <= #{keys >= d}.
__global__ void sel_digit_kernel(SelState* st, int shift) {
  if (threadIdx.x != 0) return;
  unsigned long long above = 0, need = st->need;
  int d = 255;
  if (need > 0) {
    for (; d > 0; --d) {
      if (above + st->hist[d] >= need) break;
      above += st->hist[d];
    }
    st->prefix |= (unsigned long long)d << shift;
    st->need = need - above;
  }
  for (int i = 0; i < 256; ++i) st->hist[i] = 0;
}

// Per-CTA count of keys equal to T over the CTA's contiguous index range.
template <class Src>
__global__ void __launch_bounds__(kSelThreads) count_eq_kernel(Src src, int64_t n, const SelState* st, int64_t chunk,
                                                              unsigned long long* cnt) {
  __shared__ unsigned long long part[kSelThreads / 32];
  const uint64_t T = st->prefix;
  const int64_t i0 = (int64_t)blockIdx.x * chunk, i1 = (i0 + chunk) < n ? (i0 + chunk) : n;
  unsigned long long c = 0;
  if (st->need > 0)
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) c += src(i) == T;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) s += part[w];
    cnt[blockIdx.x] = s;
  }
}

// keep[i] = key > T, or key == T and fewer than `need` keys equal to T precede it in index order.
template <class Src>
__global__ void __launch_bounds__(kSelThreads) mark_kernel(Src src, int64_t n, const SelState* st, int64_t chunk,
                                                          const unsigned long long* cnt, uint8_t* __restrict__ keep) {
  __shared__ unsigned long long before_s;
  __shared__ unsigned int wsum[kSelThreads / 32];
  const uint64_t T = st->prefix;
  const unsigned long long need = st->need;
  if (threadIdx.x == 0) {
    unsigned long long b = 0;
    for (unsigned int c = 0; c < blockIdx.x; ++c) b += cnt[c];
    before_s = b;
  }
  __syncthreads();
  unsigned long long before = before_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * chunk, i1 = (i0 + chunk) < n ? (i0 + chunk) : n;
  for (int64_t base = i0; base < i1; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    uint64_t key = 0;
    bool eq = false;
    if (i < i1) {
      key = src(i);
      eq = need > 0 && key == T;
    }
    const unsigned int bal = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    unsigned int pre = __popc(bal & ((1u << lane) - 1u));
    unsigned int tot = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) {
      pre += w < warp ? wsum[w] : 0u;
      tot += wsum[w];
    }
    if (i < i1) keep[i] = (need > 0 && key > T) || (eq && before + pre < need);
    before += tot;
    __syncthreads();
  }
}

// Tile decision -> element mask.
__global__ void expand_tiles_kernel(const uint8_t* __restrict__ tk, int64_t M, int64_t K, int64_t bh, int64_t bw,
                                    uint8_t* __restrict__ mask) {
  const int64_t TC = K / bw;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * K; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / K, c = i - r * K;
    mask[i] = tk[(r / bh) * TC + c / bw];
  }
}

struct Workspace {
  SelState* st;
  unsigned long long* cnt;
  uint64_t* tkey;
  uint8_t* tkeep;
};

int64_t ws_layout(int64_t ntiles, Workspace* w, uint8_t* base) {
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    const int64_t o = off;
    off = bsk::align_up(off + bytes, 256);
    return base ? base + o : nullptr;
  };
  uint8_t* p0 = take(sizeof(SelState));
  uint8_t* p1 = take(8LL * kMaxSelCtas);
  uint8_t* p2 = take(8LL * ntiles);
  uint8_t* p3 = take(ntiles);
  if (w) *w = Workspace{(SelState*)p0, (unsigned long long*)p1, (uint64_t*)p2, p3};
  return off;
}

// keep[0..n) for the `need` best keys of src (key bits: the number of significant key bits).
template <class Src>
cudaError_t select_top(const Src& src, int64_t n, unsigned long long need, int key_bits, const Workspace& w,
                       uint8_t* keep, cudaStream_t s) {
  const int sms = bsk::dev_props().sms;
  int64_t grid = (n + kSelThreads - 1) / kSelThreads;
  if (grid > (int64_t)sms * 8) grid = (int64_t)sms * 8;
  sel_init_kernel<<<1, 256, 0, s>>>(w.st, need);
  const int passes = (key_bits + 7) / 8;
  for (int p = passes - 1; p >= 0; --p) {
    hist_kernel<<<(unsigned)grid, kSelThreads, 0, s>>>(src, n, w.st, 8 * p);
    sel_digit_kernel<<<1, 32, 0, s>>>(w.st, 8 * p);
  }
  int64_t ctas = (int64_t)sms * 4 < kMaxSelCtas ? (int64_t)sms * 4 : kMaxSelCtas;
  int64_t chunk = (n + ctas - 1) / ctas;
  chunk = (chunk + kSelThreads - 1) / kSelThreads * kSelThreads;
  ctas = (n + chunk - 1) / chunk;
  count_eq_kernel<<<(unsigned)ctas, kSelThreads, 0, s>>>(src, n, w.st, chunk, w.cnt);
  mark_kernel<<<(unsigned)ctas, kSelThreads, 0, s>>>(src, n, w.st, chunk, w.cnt, keep);
  return cudaGetLastError();
}

unsigned long long keep_count(int64_t n, double sparsity) {
  return (unsigned long long)llround((1.0 - sparsity) * (double)n);
}

template <int DT>
cudaError_t random_mask_t(const void* W, int64_t M, int64_t K, int64_t ldw, double sparsity, uint8_t* mask,
                          const Workspace& w, cudaStream_t s) {
  ElemKeys<DT> src{(const typename bsk::KeyOf<DT>::raw_t*)W, K, ldw};
  return select_top(src, M * K, keep_count(M * K, sparsity), bsk::KeyOf<DT>::kBits, w, mask, s);
}

template <int DT>
cudaError_t block_mask_t(const void* W, int64_t M, int64_t K, int64_t ldw, int64_t bh, int64_t bw, double sparsity,
                         int criterion, uint8_t* mask, const Workspace& w, cudaStream_t s) {
  const int64_t TR = M / bh, TC = K / bw, n = TR * TC;
  const int sms = bsk::dev_props().sms;
  int64_t grid = (n + 255) / 256;
  if (grid > (int64_t)sms * 8) grid = (int64_t)sms * 8;
  tile_score_kernel<DT><<<(unsigned)grid, 256, 0, s>>>((const typename bsk::KeyOf<DT>::raw_t*)W, ldw, TR, TC, bh, bw,
                                                       criterion, w.tkey);
  ArrayKeys src{w.tkey};
  cudaError_t e = select_top(src, n, keep_count(n, sparsity), criterion == 0 ? bsk::KeyOf<DT>::kBits : 64, w,
                             w.tkeep, s);
  if (e != cudaSuccess) return e;
  int64_t g2 = (M * K + 255) / 256;
  if (g2 > (int64_t)sms * 16) g2 = (int64_t)sms * 16;
  expand_tiles_kernel<<<(unsigned)g2, 256, 0, s>>>(w.tkeep, M, K, bh, bw, mask);
  return cudaGetLastError();
}

}  // namespace

cudaError_t bsk_launch_decode(const void* vals, const uint16_t* idx, int64_t M, int64_t K, int B, int k, int dt,
                              void* W, int64_t ldw, cudaStream_t s) {
  const int64_t nseg = (K + kSeg - 1) / kSeg;
  int64_t grid = M * nseg;
  const int64_t cap = (int64_t)bsk::dev_props().sms * 8;
  if (grid > cap) grid = cap;
  if (dt == BS_F32)
    decode_kernel<uint32_t><<<(unsigned)grid, 256, 0, s>>>((const uint32_t*)vals, idx, M, K, B, k, (uint32_t*)W, ldw);
  else
    decode_kernel<uint16_t><<<(unsigned)grid, 256, 0, s>>>((const uint16_t*)vals, idx, M, K, B, k, (uint16_t*)W, ldw);
  return cudaGetLastError();
}

size_t bsk_pattern_workspace_bytes(int64_t M, int64_t K, int64_t bh, int64_t bw) {
  const int64_t ntiles = (bh > 0 && bw > 0) ? (M / bh) * (K / bw) : 0;
  return (size_t)ws_layout(ntiles, nullptr, nullptr);
}

cudaError_t bsk_launch_random_mask(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, double sparsity,
                                   uint8_t* mask, void* ws, cudaStream_t s) {
  Workspace w;
  ws_layout(0, &w, (uint8_t*)ws);
  switch (dt) {
    case BS_F32: return random_mask_t<BS_F32>(W, M, K, ldw, sparsity, mask, w, s);
    case BS_F16: return random_mask_t<BS_F16>(W, M, K, ldw, sparsity, mask, w, s);
    default: return random_mask_t<BS_BF16>(W, M, K, ldw, sparsity, mask, w, s);
  }
}

cudaError_t bsk_launch_block_mask(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int64_t bh, int64_t bw,
                                  double sparsity, int criterion, uint8_t* mask, void* ws, cudaStream_t s) {
  Workspace w;
  ws_layout((M / bh) * (K / bw), &w, (uint8_t*)ws);
  switch (dt) {
    case BS_F32: return block_mask_t<BS_F32>(W, M, K, ldw, bh, bw, sparsity, criterion, mask, w, s);
    case BS_F16: return block_mask_t<BS_F16>(W, M, K, ldw, bh, bw, sparsity, criterion, mask, w, s);
    default: return block_mask_t<BS_BF16>(W, M, K, ldw, bh, bw, sparsity, criterion, mask, w, s);
  }
}
