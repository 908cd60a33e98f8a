// spmv_impl.cuh (instantiated per dtype by spmv_f16.cu / spmv_bf16.cu / spmv_f32.cu): K3 bs_spmv, y = W_bs · x for a balanced-sparse W in the SPMV (or SPMM) layout.
//
// Paper design (Fig. 3): one thread per block partition; every thread gets the same
// work because every block keeps k entries; x is "rearranged and stored in shared memory to
// avoid bank conflicts". The B200 version:
//   - A warp walks a contiguous range of rows. Lane l owns the blocks b ≡ l (mod 32), V of them per
//     panel of 32·V blocks (docs/layout.md). A row's panel steps are contiguous in HBM, each step
//     being 32·V values followed by their 32·V indices.
//   - Steps reach shared memory through the TMA bulk-copy engine (cp.async.bulk, SASS UBLKCP): each
//     warp owns a ring of NS stages of up to Q steps, one bulk copy per stage. Lane 0 refills a stage
//     as soon as the warp has consumed it, and mbarriers with transaction counts signal arrival. So
//     the bytes in flight do not depend on register pressure or on the compute phase
//     (tools/membench.cu: >= 6.9 TB/s at 64 KB in flight per SM).
//   - x is staged per CTA in a block-interleaved order of slots (halfwords for f16/bf16, words for
//     f32; NV·2 bytes holding NV batch columns for the batched variant): element (b, o) of a chunk
//     goes to slot (gl·B + o)·32 + (b & 31), with gl = (b>>5) - first group of the chunk. Lane l
//     only ever touches its own bank (16-bit: lanes 2m, 2m+1 share a word, which is a broadcast,
//     not a conflict), whatever the indices are, so every gather is conflict-free by construction.
//     The slot address is one IMAD of the index byte (extracted by one PRMT): about 4 instructions
//     per nonzero including the FHFMA. Staging is lane-per-block too, so its stores are
//     conflict-free; all of a lane's loads are issued before its stores.
//   - K is processed in chunks of whole panels when x does not fit in 128 KB of shared memory (16-bit
//     x fits up to 65536 columns; f32 x and the batched variant chunk). Each (row, chunk) partial is reduced by the warp and added
//     in chunk order. The tail blocks (T < 32·V per row) follow through the same ring.
//   - f16/bf16 products are one FHFMA (exact 16x16 product, fp32 accumulate). Each lane keeps V
//     independent accumulators. They are summed in a fixed order and reduced with a warp butterfly.
//     Chunking depends only on (K, B, dtype), never on the row range, so row-sharded results are
//     bit-identical to unsharded ones.
//   - The grid is persistent, one CTA per SM. Each CTA owns a contiguous, balanced row range.
#pragma once
#include "bs_common.cuh"
#include "bs_device.cuh"

#include <stdlib.h>

#if defined(BS_TRACE) && defined(BS_TRACE_TU)
// Debug timeline (tools/trace_probe.py): %globaltimer at phase boundaries, per (CTA, warp).
__device__ unsigned long long g_bs_trace[1024 * 16 * 16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define BS_MARK(i)                                                                                       \
  do {                                                                                                   \
    if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < 16)                                              \
      g_bs_trace[(blockIdx.x * 16 + (threadIdx.x >> 5)) * 16 + (i)] = gtime();                           \
  } while (0)
extern "C" int bs_trace_read(void* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_bs_trace, (size_t)n * 8);
}
#else
#define BS_MARK(i) \
  do {             \
  } while (0)
#endif

namespace bsk_spmv {

constexpr int kXBudget = 128 * 1024;  // bytes of x slots per chunk
constexpr int kMaxChunks = 8;

// IS (index encoding of the panel steps): 1 or 2 index bytes, 5 = 5-bit index runs (B = 32, V = 8), 4 = 4-bit
// index runs (B <= 16, V = 8); docs/layout.md. Runs: lane l's indices of a step in one u32 word (+ one byte
// plane for 5-bit). Tail indices (regions B/C) are one byte for the runs.
template <int V, int IS>
constexpr uint32_t run_bytes() { return IS == 5 ? 160u : IS == 4 ? 128u : 32u * V * IS; }
template <int IS>
constexpr int tail_is() { return (IS == 5 || IS == 4) ? 1 : IS; }

struct SpmvArgs {
  const uint8_t* A;   // panel steps (region A)
  const uint8_t* Bt;  // tail values (region B): element r·k·T + t·T + v·32 + l
  const uint8_t* Ct;  // tail indices (region C), same order
  const void* x;
  void* y;
  int64_t M, NB, NBf, T;
  int B, k;
  int NS;            // ring stages per warp
  int xbytes;        // smem bytes reserved for x slots (max over chunks)
  int nchunks;       // panel chunks
  int PC;            // panels per chunk (the last may be shorter)
  int tail_in_last;  // tail groups are staged with the last panel chunk
  int tail_rows;     // rows per ring-streamed tail stage (0: direct loads)
  int xvec;          // x is 16-byte aligned and B allows 16-byte staging loads
  int64_t ldx, ldy;  // batch-column strides of X and Y (NV > 1)
  int ncols;         // valid batch columns in this pass (NV > 1)
  int w_early;       // PDL: W may be streamed before griddepcontrol.wait (BS_SPMV_W_STATIC)
  int pdl;           // host: launch with programmatic stream serialization (BS_SPMV_PDL)
  int direct;        // host: short rows take spmv_rows_kernel (NV = 1, one x chunk; see below)
  const void* bias;  // NV = 1: optional per-row bias (M elements of D), Eq. 1's +B
  int act;           // NV = 1: bs_act applied after the bias (BS_ACT_NONE = 0)
  uint32_t bias_off; // shared-memory byte offset of the CTA's bias rows (fp32)
  // LSTM cell epilogue (bs_lstm_step; NV = 1): rows are gate rows interleaved 4j + g (i, f, g, o of
  // unit j). The CTA's row range is a whole number of units; each row's z = W·x + pre + bias is parked
  // in shared memory (in place of its bias) and, once the CTA's rows are done, one thread per unit
  // applies the cell: c = sigmoid(z_f)·c_prev + sigmoid(z_i)·tanh(z_g), h = sigmoid(z_o)·tanh(c).
  int lstm;
  const void* pre;     // a second per-row addend of D (W_ih·x_t computed ahead), or NULL
  const float* c_prev; // M/4 fp32
  float* c_out;        // M/4 fp32
  void* h_out;         // M/4 of D
  // Fused all-gather epilogue (bs_spmv_allgather; NV = 1): this launch computes one rank's row shard;
  // its rows are parked in shared memory and each CTA stores its contiguous run to every rank's full y
  // (peer-mapped pointers over NVLink), then the last CTA raises this rank's flag on every rank.
  int ag_n;             // ranks (0: off)
  int ag_rank;
  int64_t ag_row0;      // global row of the shard's first row
  void* ag_y[8];        // every rank's full y (M_total elements of D)
  uint32_t* ag_flag[8]; // every rank's arrival flags (ag_n words)
  uint32_t* ag_cnt;     // this rank's CTA completion counter (monotonic)
  uint32_t ag_epoch;    // call number, >= 1
  uint32_t ag_off;      // shared-memory byte offset of the parked y rows
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Layer epilogue y = act(W·x + b) in fp32 before the single rounding to D (bs_spmv_fused).
__device__ __forceinline__ float apply_act(float v, int act) {
  switch (act) {
    case BS_ACT_RELU: return fmaxf(v, 0.f);
    case BS_ACT_SIGMOID: return 1.f / (1.f + expf(-v));
    case BS_ACT_TANH: return tanhf(v);
    default: return v;
  }
}

// Programmatic dependent launch (PDL). launch_dependents lets the next kernel on the stream be
// scheduled while this one runs; wait blocks until the previous kernel has completed and its writes
// are visible. Both are no-ops when the kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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
                 : "=r"(done)
                 : "r"(bar), "r"(parity)
                 : "memory");
  }
}
// W is streamed exactly once per call: its bulk copies carry an L2 evict_first policy so that they
// do not push the activations (x, y) out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
// Byte i (compile-time after unrolling) of w, zero-extended: one PRMT.
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int i) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "r"(0x4440 | i));
  return r;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint16_t b8;
  asm volatile("ld.shared.u8 %0, [%1];" : "=h"(b8) : "r"(a));
  return b8;
}

// Byte offset, from the start of a chunk's x slots, of element (block 32·(g0 + gl) + lane, offset o) of
// the rearranged x (the paper's conflict-free x): ES-byte slots (NV = 1), paired 16-bit
// groups (PAIR), or 2·NV-byte batch slots (NV > 1). stage_x / stage_xn store through it; the gathers read
// the same slots (the unit-vector and integer-exact parity tests prove it), and bs_x_slot_offset exports
// it to the host bank-conflict model (tests/test_bank_model.py).
__host__ __device__ __forceinline__ uint32_t x_slot(uint32_t gl, uint32_t o, uint32_t lane, uint32_t B, uint32_t ES,
                                                    uint32_t NV, bool pair) {
  if (NV > 1) return (gl * B + o) * (32u * 2u * NV) + lane * 2u * NV;
  if (pair) return ((gl >> 1) * B + o) * 128u + lane * 4u + (gl & 1u) * 2u;
  return (gl * B + o) * (32u * ES) + lane * ES;
}

// NV = 16: a slot is 32 bytes (two 16-byte halves, columns 0-7 and 8-15), read by two LDS.128. A 16-byte
// request is served 8 lanes per wavefront; with the halves in column order, lanes l and l + 4 of a phase
// would hit the same banks (slot stride 32 B: 2-way conflicts, found by the T2 model). So lane l keeps
// columns 0-7 in half ((l >> 2) & 1) and columns 8-15 in the other: byte offset of part p in the slot.
__host__ __device__ __forceinline__ uint32_t x_part_off(uint32_t lane, uint32_t NV, uint32_t part) {
  return NV == 16 ? 16u * (((lane >> 2) & 1u) ^ part) : 0u;
}

// Stage the x columns of groups [g0, g1) into slots of ES bytes (halfwords for f16/bf16, words
// for f32): element (b, o), b = 32·g + l, goes to slot (gl·B + o)·32 + l, gl = g - g0. Lane l always
// copies block 32·g + l. So for f32 every slot of lane l is in bank l, and for 16-bit x the lanes
// 2m and 2m+1 share a word. Work items are (group, 16-byte piece of a block); each lane issues up to
// 8 piece loads before storing them. `after_loads()` runs once, right after the first batch of
// loads is in flight, so that the caller can queue the W bulk copies behind them.
// PAIR (16-bit x, any V; a single group is paired with an empty one): groups 2j and 2j+1 share slot words. Element (b, o), b = 32·g + l, goes to
// byte ((g>>1)·B + o)·128 + 4·l + 2·(g&1): lane l's slots are all in bank l, for any offsets (with
// halfword slots per group, lanes 2m and 2m+1 would share a bank with different offsets: 2-way
// conflicts). The consumer's group index is compile-time, so the address is still one IMAD.
template <int ES, int BT, bool PAIR, typename F>
__device__ __forceinline__ void stage_x(const SpmvArgs& a, uint32_t sx, int64_t g0, int64_t g1, F after_loads) {
  constexpr int PE = 16 / ES;        // elements per 16-byte piece
  constexpr uint32_t ROWB = PAIR ? 128 : 32 * ES;  // bytes per slot row (one offset o of 32 blocks, or of 64 when paired)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int B = BT > 0 ? BT : a.B;
  bool hooked = false;
  if (a.xvec) {  // 16-byte aligned x and B % PE == 0
    const uint32_t ppb = (uint32_t)(B / PE);  // pieces per block (x slots fit in shared memory: 32-bit)
    const uint32_t items = (uint32_t)(g1 - g0) * ppb;
    for (uint32_t j0 = warp; j0 < items || !hooked; j0 += 8u * nw) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t j = j0 + (uint32_t)u * nw;
        if (j < items) {
          const uint32_t gl = j / ppb;
          const uint32_t q = j - gl * ppb;
          const int64_t b = (g0 + gl) * 32 + lane;
          if (b < a.NB) v[u] = __ldg((const uint4*)((const uint8_t*)a.x + (b * B + q * PE) * ES));
        }
      }
      if (!hooked) {
        after_loads();
        hooked = true;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t j = j0 + (uint32_t)u * nw;
        if (j < items) {
          const uint32_t gl = j / ppb;
          const uint32_t q = j - gl * ppb;
          const int64_t b = (g0 + gl) * 32 + lane;
          if (b < a.NB) {
            const uint32_t col = sx + x_slot(gl, q * PE, lane, B, ES, 1, PAIR);
            const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int e = 0; e < PE; ++e) {
              if (ES == 2) bsk::sts_u16(col + e * ROWB, (uint16_t)(w[e >> 1] >> (16 * (e & 1))));
              else bsk::sts_u32(col + e * ROWB, w[e]);
            }
          }
        }
      }
    }
  } else {
    after_loads();
    for (int64_t g = g0 + warp; g < g1; g += nw) {
      const int64_t b = g * 32 + lane;
      if (b >= a.NB) continue;
      const uint32_t gl = (uint32_t)(g - g0);
      const uint32_t col = sx + x_slot(gl, 0, lane, B, ES, 1, PAIR);
      for (int o = 0; o < B; ++o) {
        if (ES == 2) bsk::sts_u16(col + o * ROWB, __ldg((const uint16_t*)a.x + b * B + o));
        else bsk::sts_u32(col + o * ROWB, __ldg((const uint32_t*)a.x + b * B + o));
      }
    }
  }
}

// NV > 1 (16-bit x only): a slot holds X[0..NV)[c] for one column c, so one 2·NV-byte shared load
// gathers the column's batch vector. Slot (gl·B + o)·32 + l of NV halves; rows n >= ncols are zero.
// Lane l copies block 32·g + l: per 8-column piece it loads NV 16-byte row pieces, transposes them in
// registers and writes 8 slots.
template <int NV, int BT, typename F>
__device__ __forceinline__ void stage_xn(const SpmvArgs& a, uint32_t sx, int64_t g0, int64_t g1, F after_loads) {
  constexpr uint32_t SLB = 2 * NV, ROWB = 32 * SLB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int B = BT > 0 ? BT : a.B;
  bool hooked = false;
  if (a.xvec) {  // rows 16-byte aligned, B % 8 == 0
    const uint32_t ppb = (uint32_t)(B / 8);
    const uint32_t items = (uint32_t)(g1 - g0) * ppb;
    for (uint32_t j = warp; j < items || !hooked; j += nw) {
      uint4 v[NV];
      const uint32_t gl = j < items ? j / ppb : 0;
      const uint32_t q = j < items ? j - gl * ppb : 0;
      const int64_t b = (g0 + gl) * 32 + lane;
      const bool ok = j < items && b < a.NB;
#pragma unroll
      for (int n = 0; n < NV; ++n) {
        v[n] = make_uint4(0u, 0u, 0u, 0u);
        if (ok && n < a.ncols) v[n] = __ldg((const uint4*)((const uint16_t*)a.x + n * a.ldx + b * B + q * 8));
      }
      if (!hooked) {
        after_loads();
        hooked = true;
      }
      if (ok) {
        const uint32_t col = sx + x_slot(gl, q * 8, lane, B, 2, NV, false);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          uint32_t h[NV];
#pragma unroll
          for (int n = 0; n < NV; ++n) {
            const uint32_t w = e < 2 ? (e == 0 ? v[n].x : v[n].x) : e < 4 ? v[n].y : e < 6 ? v[n].z : v[n].w;
            h[n] = (w >> (16 * (e & 1))) & 0xffffu;
          }
          if constexpr (NV == 16) {
            bsk::sts_v4(col + e * ROWB + x_part_off(lane, 16, 0), h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
            bsk::sts_v4(col + e * ROWB + x_part_off(lane, 16, 1), h[8] | (h[9] << 16), h[10] | (h[11] << 16), h[12] | (h[13] << 16), h[14] | (h[15] << 16));
          } else if constexpr (NV == 8) bsk::sts_v4(col + e * ROWB, h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
          else if constexpr (NV == 4) asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(col + e * ROWB), "r"(h[0] | (h[1] << 16)), "r"(h[2] | (h[3] << 16)));
          else bsk::sts_u32(col + e * ROWB, h[0] | (h[1] << 16));
        }
      }
      if (j >= items) break;
    }
  } else {
    after_loads();
    for (int64_t g = g0 + warp; g < g1; g += nw) {
      const int64_t b = g * 32 + lane;
      if (b >= a.NB) continue;
      const uint32_t col = sx + x_slot((uint32_t)(g - g0), 0, lane, B, 2, NV, false);
      for (int o = 0; o < B; ++o) {
        uint32_t h[NV];
#pragma unroll
        for (int n = 0; n < NV; ++n) h[n] = n < a.ncols ? (uint32_t)__ldg((const uint16_t*)a.x + n * a.ldx + b * B + o) : 0u;
        if constexpr (NV == 16) {
          bsk::sts_v4(col + o * ROWB + x_part_off(lane, 16, 0), h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
          bsk::sts_v4(col + o * ROWB + x_part_off(lane, 16, 1), h[8] | (h[9] << 16), h[10] | (h[11] << 16), h[12] | (h[13] << 16), h[14] | (h[15] << 16));
        } else if constexpr (NV == 8) bsk::sts_v4(col + o * ROWB, h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
        else if constexpr (NV == 4) asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(col + o * ROWB), "r"(h[0] | (h[1] << 16)), "r"(h[2] | (h[3] << 16)));
        else bsk::sts_u32(col + o * ROWB, h[0] | (h[1] << 16));
      }
    }
  }
}

// Transposing butterfly over NV per-lane values: afterwards lane l holds the warp total of value
// l >> (5 - log2 NV). Every value is summed over the lanes with the same pairing sequence
// (xor 16, 8, 4, 2, 1), so its result does not depend on NV.
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
      for (int i = 0; i < (NV > 1 ? NV / 2 : 1); ++i) {
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

// One CTA per SM, NT/32 warps. Warp rows [wr0, wr0 + nrows). For panel chunk c (panels
// [c·PC, c·PC + np)), each row contributes a segment of L = np·k consecutive steps. The ring streams
// the segments of all chunks in order (a stage never crosses a segment), then the tails (R rows
// per stage).
template <int DT, int V, int IS, int Q, int BT, bool MULTI, int NT, int NV>
__global__ void __launch_bounds__(NT, 1) spmv_kernel(SpmvArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[NT / 32][4];
  using raw_t = typename bsk::DTraits<DT>::raw_t;
  constexpr int ES = bsk::DTraits<DT>::kBytes;
  constexpr int P = 32 * V;
  // IS: index bytes (1 or 2), or 5 = 5-bit index runs (B = 32, V = 8; docs/layout.md): per step a
  // plane of 32 u32 words and a plane of 32 bytes, lane l's 40-bit field sum_v idx(l, v) << 5v
  static_assert(IS != 5 || (V == 8 && BT == 32), "5-bit runs need V = 8 and B = 32");
  static_assert(IS != 4 || V == 8, "4-bit runs need V = 8");
  constexpr int ISt = tail_is<IS>();                   // tail index bytes (regions B/C)
  constexpr uint32_t RI = run_bytes<V, IS>();          // index run bytes per step
  constexpr uint32_t STEPB = P * ES + RI;              // bytes per step (values then indices)
  constexpr uint32_t SB = Q * STEPB;         // bytes per ring stage
  const int B = BT > 0 ? BT : a.B;
  constexpr uint32_t SLB = ES * NV;       // bytes per x slot (NV batch columns of one x column)
  constexpr uint32_t ROWB = 32 * SLB;     // bytes per slot row of x (one offset o of 32 blocks)
  constexpr bool PAIR = ES == 2 && NV == 1;  // paired groups (stage_x): lane l stays in bank l (tests/test_bank_model.py)
  constexpr uint32_t XROW = PAIR ? 128u : ROWB;         // slot-row stride seen by the gathers
  constexpr uint32_t LSLB = PAIR ? 4u : SLB;            // lane stride of the slots
  constexpr int NA = NV == 1 ? V : NV;    // accumulators: V chains (SpMV) or one per batch column
  const uint32_t GSW = (uint32_t)B * ROWB;  // bytes per group of 32 blocks
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = NT / 32;
  // balanced row ranges (32-bit arithmetic: M·(grid + 1) < 2^32 is checked on the host); the LSTM
  // epilogue needs whole units (4 gate rows) per CTA
  const uint32_t RU = (NV == 1 && a.lstm) ? 4u : 1u;
  const int64_t rb = RU * (blockIdx.x * ((uint32_t)a.M / RU) / gridDim.x);
  const int64_t re = RU * ((blockIdx.x + 1) * ((uint32_t)a.M / RU) / gridDim.x);
  const uint32_t nr = (uint32_t)(re - rb);
  const int64_t wr0 = rb + warp * nr / nw;
  const int64_t nrows = rb + (warp + 1) * nr / nw - wr0;
  const int64_t S = a.NBf * a.k;  // full-panel steps per row
  const int NS = a.NS;
  // XALIGN (5-bit runs): the x slots start on a 4 KB boundary, so a gather address is
  // panel_base | (o << 7) (the panel base has bits 7..11 clear) plus an immediate: one LOP3 instead of
  // LOP3 + IADD per nonzero. The host reserves the 4 KB of slack.
  constexpr bool XALIGN = IS == 5 && NV == 1;
  const uint32_t sx0 = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t xoff = XALIGN ? ((sx0 + 4095u) & ~4095u) - sx0 : 0u;
  const uint32_t sx = sx0 + xoff;
  const uint32_t ring = sx + a.xbytes + (uint32_t)(warp * NS) * SB;
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[warp][0]);
  BS_MARK(0);
  float* part = (float*)(smem + xoff + a.xbytes + (size_t)nw * NS * SB) - rb * NV;  // fp32 partials [row][NV] (MULTI)
  const int64_t kT = (int64_t)a.k * a.T;  // entries of one row's tail
  // A tail stage holds R rows: the value run (from the 16-byte-aligned address at or below it, offset
  // dv), then, at the next 16-byte boundary, the index run (offset di).
  auto tail_geom = [&](int64_t t0, int64_t R, uint32_t& dv, uint32_t& bv, uint32_t& di, uint32_t& bi) {
    const int64_t ov = (wr0 + t0) * kT * ES, oi = (wr0 + t0) * kT * ISt;
    dv = (uint32_t)(ov & 15);
    di = (uint32_t)(oi & 15);
    bv = (uint32_t)((dv + R * kT * ES + 15) & ~15LL);
    bi = (uint32_t)((di + R * kT * ISt + 15) & ~15LL);
  };

  // ---- producer cursor (lane 0). Phase 1: (chunk pc, row pr, step ps) of the next panel stage.
  // Phase 2 (pc == nchunks): tail stages of R rows each starting at row tr.
  int pc = 0;
  int64_t pr = 0, ps = 0, tr = 0;
  auto seg_len = [&](int c) -> int64_t {
    const int64_t p0 = (int64_t)c * a.PC;
    const int64_t np = (a.NBf - p0) < a.PC ? (a.NBf - p0) : a.PC;
    return np * a.k;
  };
  int64_t pL = seg_len(0);
  const bool have_panels = S > 0 && nrows > 0;
  if (!have_panels) pc = a.nchunks;
  const bool ring_tail = a.T > 0 && a.k > 0 && a.tail_rows > 0 && nrows > 0;
  auto more = [&]() { return pc < a.nchunks || (ring_tail && tr < nrows); };
  const uint64_t pol = policy_evict_first();
  auto issue = [&](uint32_t st) {  // load the next stage into ring slot st: one bulk copy
    const uint32_t bar = bar0 + st * 8;
    if (pc < a.nchunks) {
      const int64_t n = (pL - ps) < Q ? (pL - ps) : Q;
      const int64_t step0 = (wr0 + pr) * S + (int64_t)pc * a.PC * a.k + ps;
      const uint32_t bytes = (uint32_t)n * STEPB;
      mbar_expect_tx(bar, bytes);
      bulk_g2s(ring + st * SB, a.A + step0 * STEPB, bytes, bar, pol);
      ps += n;
      if (ps == pL) {
        ps = 0;
        if (++pr == nrows) {
          pr = 0;
          ++pc;
          if (pc < a.nchunks) pL = seg_len(pc);
        }
      }
    } else {
      // rows [tr, tr + R) of the tail region; bulk copies need 16-byte aligned sources and sizes, so
      // copy from the aligned-down address (the consumer re-derives the same offset)
      const int64_t R = (nrows - tr) < a.tail_rows ? (nrows - tr) : a.tail_rows;
      uint32_t dv, bv, di, bi;
      tail_geom(tr, R, dv, bv, di, bi);
      mbar_expect_tx(bar, bv + bi);
      bulk_g2s(ring + st * SB, a.Bt + (wr0 + tr) * kT * ES - dv, bv, bar, pol);
      bulk_g2s(ring + st * SB + bv, a.Ct + (wr0 + tr) * kT * ISt - di, bi, bar, pol);
      tr += R;
    }
  };
  if (lane == 0) {
    for (int st = 0; st < NS; ++st) mbar_init(bar0 + st * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    BS_MARK(5);
  }
  __syncwarp();
  // the first x loads go out before the ring is armed, so that they do not queue behind W
  auto arm_ring = [&]() {
    if (lane == 0) {
      for (int st = 0; st < NS && more(); ++st) {
        issue((uint32_t)st);
        if (st == 0) BS_MARK(7);
      }
    }
  };
  bool armed = false;
  auto arm_once = [&]() {
    if (!armed) {
      arm_ring();
      armed = true;
    }
  };
  pdl_launch_dependents();
  // Everything above touched only shared memory. With w_early (static weights) the W ring fills while
  // the previous kernel finishes; x (its output) and y (which it may still read) wait for it.
  if (a.w_early) arm_once();
  pdl_wait();

  float acc[NA];
#pragma unroll
  for (int v = 0; v < NA; ++v) acc[v] = 0.f;
  // gather x slot(s) of offset o for owned block v and accumulate w·x
  auto gather_fma = [&](uint32_t base, uint32_t o, int v, uint32_t w) {
    if constexpr (NV == 1) {
      const uint32_t ad = PAIR ? base + o * XROW + (uint32_t)(v >> 1) * 2u * GSW + (uint32_t)(v & 1) * 2u
                               : base + o * ROWB + v * GSW;
      bsk::fma_acc<DT>(acc[v], w, lds_x<DT>(ad));
    } else {
      uint32_t xw[NV / 2 > 4 ? NV / 2 : 4];
      const uint32_t ad = base + o * ROWB + v * GSW;
      if constexpr (NV == 16) {
        bsk::lds_v4(ad + x_part_off(lane, 16, 0), xw[0], xw[1], xw[2], xw[3]);
        bsk::lds_v4(ad + x_part_off(lane, 16, 1), xw[4], xw[5], xw[6], xw[7]);
      } else if constexpr (NV == 8) bsk::lds_v4(ad, xw[0], xw[1], xw[2], xw[3]);
      else if constexpr (NV == 4) asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(xw[0]), "=r"(xw[1]) : "r"(ad));
      else xw[0] = bsk::lds_u32(ad);
#pragma unroll
      for (int n = 0; n < NV; ++n) bsk::fma_acc<DT>(acc[n], w, (xw[n >> 1] >> (16 * (n & 1))) & 0xffffu);
    }
  };
  // row total: SpMV -> one value (lane 0 holds it); NV > 1 -> lane l holds column l >> (5 - log2 NV)
  constexpr int LOGNV = NV == 16 ? 4 : NV == 8 ? 3 : NV == 4 ? 2 : NV == 2 ? 1 : 0;
  auto row_total = [&](float& tot, int& col) -> bool {
    if constexpr (NV == 1) {
      tot = warp_total<V>(acc);
      col = 0;
      return lane == 0;
    } else {
      tot = transpose_reduce<NV>(acc, lane);
#pragma unroll
      for (int n = 0; n < NV; ++n) acc[n] = 0.f;
      col = lane >> (5 - LOGNV);
      return (lane & ((32 >> LOGNV) - 1)) == 0;
    }
  };
  // the CTA's bias rows are staged into shared memory with the first x staging (their loads go out
  // before the x loads and land while x is staged), so the epilogue adds no global round trip
  const bool lstm = NV == 1 && a.lstm;
  const bool ag = NV == 1 && a.ag_n > 0;
  const bool has_bias = NV == 1 && (a.bias != nullptr || a.pre != nullptr || lstm);
  float* sbias = (float*)(smem + xoff + a.bias_off);
  // each thread prefetches up to 4 bias rows into registers before the x loads; stored after them
  float bp0 = 0.f, bp1 = 0.f, bp2 = 0.f, bp3 = 0.f;
  bool bias_done = false;
  auto bias_ld = [&](uint32_t i) {
    float b = a.bias ? bsk::to_float<DT>(__ldg((const raw_t*)a.bias + rb + i)) : 0.f;
    if (a.pre) b += bsk::to_float<DT>(__ldg((const raw_t*)a.pre + rb + i));
    return b;
  };
  auto bias_issue = [&]() {
    if (has_bias && !bias_done) {
      const uint32_t i = threadIdx.x;
      if (i < nr) bp0 = bias_ld(i);
      if (i + NT < nr) bp1 = bias_ld(i + NT);
      if (i + 2 * NT < nr) bp2 = bias_ld(i + 2 * NT);
      if (i + 3 * NT < nr) bp3 = bias_ld(i + 3 * NT);
    }
  };
  auto bias_store = [&]() {
    if (has_bias && !bias_done) {
      const uint32_t i = threadIdx.x;
      if (i < nr) sbias[i] = bp0;
      if (i + NT < nr) sbias[i + NT] = bp1;
      if (i + 2 * NT < nr) sbias[i + 2 * NT] = bp2;
      if (i + 3 * NT < nr) sbias[i + 3 * NT] = bp3;
      for (uint32_t j = i + 4 * NT; j < nr; j += NT) sbias[j] = bias_ld(j);
    }
    bias_done = true;
  };
  auto store_y = [&](int64_t r, int col, float y) {
    if (NV == 1) {
      if (has_bias) y += sbias[r - rb];
      if (lstm) {  // the gate pre-activation z waits in shared memory for the cell epilogue
        sbias[r - rb] = y;
        return;
      }
      if (a.act) y = apply_act(y, a.act);
      if (ag) {  // parked for the fused all-gather epilogue
        ((raw_t*)(smem + xoff + a.ag_off))[r - rb] = (raw_t)bsk::from_float<DT>(y);
        return;
      }
      ((raw_t*)a.y)[r] = (raw_t)bsk::from_float<DT>(y);
    }
    else if (col < a.ncols) ((raw_t*)a.y)[col * a.ldy + r] = (raw_t)bsk::from_float<DT>(y);
  };

  BS_MARK(1);
  // ---- consumer
  // ring position of the next stage to consume: slot cst, mbarrier phase cph (no divisions)
  uint32_t cst = 0, cph = 0;
  bool first_stage = true;
  auto advance = [&]() {
    if (++cst == (uint32_t)NS) {
      cst = 0;
      cph ^= 1u;
    }
  };
  for (int c = 0; c < a.nchunks; ++c) {
    const int64_t g0 = (int64_t)c * a.PC * V;
    const bool last = c == a.nchunks - 1;
    const int64_t npc = (a.NBf - (int64_t)c * a.PC) < a.PC ? (a.NBf - (int64_t)c * a.PC) : a.PC;
    const int64_t g1 = last && a.tail_in_last ? (a.NB + 31) / 32 : g0 + npc * V;
    if (c > 0) __syncthreads();  // all warps are done with the previous chunk's x
    if (c == 0) bias_issue();
    if constexpr (NV == 1) stage_x<ES, BT, PAIR>(a, sx, g0, g1, arm_once);
    else stage_xn<NV, BT>(a, sx, g0, g1, arm_once);
    if (c == 0) bias_store();
    if (c == 0) BS_MARK(6);
    __syncthreads();
    if (c == 0) BS_MARK(2);
    if (!have_panels) continue;
    const int64_t L = seg_len(c);
    const uint32_t pstep = V * GSW;
    const int k = a.k;
    for (int64_t i = 0; i < nrows; ++i) {
      uint32_t pb = sx + lane * LSLB;  // slot base of the current panel within the chunk
      int t = 0;
      for (int64_t s0 = 0; s0 < L; s0 += Q) {
        const uint32_t st = cst;
        mbar_wait(bar0 + st * 8, cph);
        if (first_stage) BS_MARK(3);
        first_stage = false;
        const uint32_t sbase = ring + st * SB;
        const int nq = (L - s0) < Q ? (int)(L - s0) : Q;
        auto step = [&](int q) {
          uint32_t wv[(V * ES + 3) / 4], iv[(V * ISt + 3) / 4 > 2 ? (V * ISt + 3) / 4 : 2];
          const uint32_t av = sbase + q * STEPB + lane * (V * ES);
          const uint32_t ai = sbase + q * STEPB + P * ES + lane * ((IS == 5 || IS == 4) ? 4 : V * IS);
          if constexpr (V * ES == 16) bsk::lds_v4(av, wv[0], wv[1], wv[2], wv[3]);
          else if constexpr (V * ES == 8) asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(wv[0]), "=r"(wv[1]) : "r"(av));
          else if constexpr (V * ES == 4) wv[0] = bsk::lds_u32(av);
          else wv[0] = bsk::lds_u16(av);
          if constexpr (IS == 5) {
            iv[0] = bsk::lds_u32(ai);
            iv[1] = lds_u8(sbase + q * STEPB + P * ES + 128 + lane);
          } else if constexpr (IS == 4) {
            iv[0] = bsk::lds_u32(ai);
          } else if constexpr (V * IS == 16) bsk::lds_v4(ai, iv[0], iv[1], iv[2], iv[3]);
          else if constexpr (V * IS == 8) asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(iv[0]), "=r"(iv[1]) : "r"(ai));
          else if constexpr (V * IS == 4) iv[0] = bsk::lds_u32(ai);
          else if constexpr (V * IS == 2) iv[0] = bsk::lds_u16(ai);
          else iv[0] = lds_u8(ai);
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const uint32_t w = ES == 2 ? (wv[v >> 1] >> (16 * (v & 1))) & 0xffffu : wv[v];
            if constexpr (XALIGN) {
              // o << 7 straight out of the 40-bit field (o = bits 5v..5v+4), OR-ed into the panel base
              uint32_t o7;
              if (v == 0) o7 = iv[0] << 7;
              else if (v == 1) o7 = iv[0] << 2;
              else if (v == 7) o7 = iv[1] << 4;
              else o7 = __funnelshift_r(iv[0], iv[1], 5 * v - 7);
              const uint32_t ad = (pb | (o7 & 0xF80u)) + (uint32_t)(v >> 1) * 2u * GSW + (uint32_t)(v & 1) * 2u;
              bsk::fma_acc<DT>(acc[v], w, lds_x<DT>(ad));
            } else {
              uint32_t o;
              if constexpr (IS == 5) o = (v < 7 ? __funnelshift_r(iv[0], iv[1], 5 * v) : iv[1] >> 3) & 31u;
              else if constexpr (IS == 4) o = (iv[0] >> (4 * v)) & 15u;
              else if constexpr (IS == 1) o = byte_of(iv[v >> 2], v & 3);
              else o = (iv[v >> 1] >> (16 * (v & 1))) & 0xffffu;
              gather_fma(pb, o, v, w);
            }
          }
          if (++t == k) {
            t = 0;
            pb += pstep;
          }
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
        advance();
        if (lane == 0 && more()) issue(st);
      }
      const int64_t r = wr0 + i;
      float tot;
      int col;
      if (row_total(tot, col)) {
        if (MULTI) part[r * NV + col] = c == 0 ? tot : part[r * NV + col] + tot;
        else store_y(r, col, tot);
      }
    }
  }

  BS_MARK(4);
  // ---- tail blocks (region B: per row k·T values then k·T indices, (t, v, lane) order)
  if (a.T > 0 && a.k > 0) {
    const int64_t gt0 = a.NBf * V, gt1 = (a.NB + 31) / 32;
    uint32_t tbase;
    // paired x slots: the tail starts at a pair boundary plus tpar groups (tpar = 1 only for V = 1 with an
    // odd number of groups before the tail in the staged chunk)
    uint32_t tpar = 0;
    if (a.tail_in_last) {
      const uint32_t tg0 = (uint32_t)(gt0 - (int64_t)(a.nchunks - 1) * a.PC * V);
      tpar = PAIR ? (tg0 & 1u) : 0u;
      tbase = sx + (tg0 - tpar) * GSW;
    } else {
      __syncthreads();
      bias_issue();
      if constexpr (NV == 1) stage_x<ES, BT, PAIR>(a, sx, gt0, gt1, arm_once);
      else stage_xn<NV, BT>(a, sx, gt0, gt1, arm_once);
      bias_store();
      __syncthreads();
      tbase = sx;
    }
    const int Vt = (int)((a.T + 31) / 32);
    auto finish_row = [&](int64_t r) {
      float tot;
      int col;
      if (row_total(tot, col)) store_y(r, col, S > 0 ? part[r * NV + col] + tot : tot);
    };
    // one row's tail; ldv/ldi load entry e (position t·T + v·32 + l) of the value / index runs
    auto tail_row = [&](auto ldv, auto ldi) {
      int tt = 0;
      if constexpr (NV == 1) {
        // four entries per block at a time: their loads and gathers are issued before the FMAs (the
        // shared-memory loads are volatile, so they are issued in program order); the FMAs into acc[v]
        // stay in tt order, so the sum is the same as one entry at a time
        for (; tt + 4 <= a.k; tt += 4) {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const int bl = v * 32 + lane;
            if (v < Vt && bl < a.T) {
              uint32_t w[4], o[4], xv[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                w[u] = ldv((uint32_t)(tt + u) * (uint32_t)a.T + bl);
                o[u] = ldi((uint32_t)(tt + u) * (uint32_t)a.T + bl);
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const uint32_t base = tbase + lane * LSLB;
                const uint32_t ad = PAIR ? base + o[u] * XROW + ((uint32_t)v + tpar) / 2u * 2u * GSW + (((uint32_t)v + tpar) & 1u) * 2u
                                         : base + o[u] * ROWB + v * GSW;
                xv[u] = lds_x<DT>(ad);
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) bsk::fma_acc<DT>(acc[v], w[u], xv[u]);
            }
          }
        }
      }
      for (; tt < a.k; ++tt) {
        const uint32_t e0 = (uint32_t)tt * (uint32_t)a.T;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int bl = v * 32 + lane;
          if (v < Vt && bl < a.T) {
            const uint32_t w = ldv(e0 + bl);
            const uint32_t o = ldi(e0 + bl);
            if constexpr (PAIR) {
              const uint32_t g = (uint32_t)v + tpar;
              bsk::fma_acc<DT>(acc[v], w, lds_x<DT>(tbase + lane * LSLB + o * XROW + g / 2u * 2u * GSW + (g & 1u) * 2u));
            } else {
              gather_fma(tbase + lane * LSLB, o, v, w);
            }
          }
        }
      }
    };
    if (ring_tail) {  // tails arrive through the ring, R rows per stage
      for (int64_t t0 = 0; t0 < nrows; t0 += a.tail_rows) {
        const int64_t R = (nrows - t0) < a.tail_rows ? (nrows - t0) : a.tail_rows;
        const uint32_t st = cst;
        mbar_wait(bar0 + st * 8, cph);
        uint32_t dv, bv, di, bi;
        tail_geom(t0, R, dv, bv, di, bi);
        for (int64_t rr = 0; rr < R; ++rr) {
          const uint32_t rv = ring + st * SB + dv + (uint32_t)(rr * kT * ES);
          const uint32_t ri = ring + st * SB + bv + di + (uint32_t)(rr * kT * ISt);
          tail_row([&](uint32_t e) { return ES == 2 ? bsk::lds_u16(rv + e * 2) : bsk::lds_u32(rv + e * 4); },
                   [&](uint32_t e) { return ISt == 1 ? lds_u8(ri + e) : bsk::lds_u16(ri + e * 2); });
          finish_row(wr0 + t0 + rr);
        }
        __syncwarp();
        advance();
        if (lane == 0 && more()) issue(st);
      }
    } else {  // direct loads (a row's tail does not fit a ring stage)
      for (int64_t i = 0; i < nrows; ++i) {
        const uint8_t* rv = a.Bt + (wr0 + i) * kT * ES;
        const uint8_t* ri = a.Ct + (wr0 + i) * kT * ISt;
        tail_row([&](uint32_t e) { return ES == 2 ? (uint32_t)__ldg((const uint16_t*)rv + e) : __ldg((const uint32_t*)rv + e); },
                 [&](uint32_t e) { return ISt == 1 ? (uint32_t)__ldg(ri + e) : (uint32_t)__ldg((const uint16_t*)ri + e); });
        finish_row(wr0 + i);
      }
    }
  } else if (S == 0) {  // k == 0: y = act(0 + b)
    if (has_bias) {
      bias_issue();
      bias_store();
      __syncthreads();
    }
    for (int64_t i = lane; i < nrows * NV; i += 32) store_y(wr0 + i / NV, (int)(i % NV), 0.f);
  } else if (MULTI) {
    __syncwarp();
    for (int64_t i = lane; i < nrows * NV; i += 32) store_y(wr0 + i / NV, (int)(i % NV), part[(wr0 + i / NV) * NV + i % NV]);
  }
  if (lstm) {  // LSTM cell over the CTA's units, from the gate pre-activations in shared memory
    __syncthreads();
    for (uint32_t u = threadIdx.x; u < nr / 4; u += NT) {
      const float zi = sbias[4 * u], zf = sbias[4 * u + 1], zg = sbias[4 * u + 2], zo = sbias[4 * u + 3];
      const int64_t j = rb / 4 + u;
      const float c = apply_act(zf, BS_ACT_SIGMOID) * a.c_prev[j] + apply_act(zi, BS_ACT_SIGMOID) * apply_act(zg, BS_ACT_TANH);
      a.c_out[j] = c;
      ((raw_t*)a.h_out)[j] = (raw_t)bsk::from_float<DT>(apply_act(zo, BS_ACT_SIGMOID) * apply_act(c, BS_ACT_TANH));
    }
  }
  if (ag) {  // fused all-gather: the CTA's rows to every rank's y, then the completion protocol
    __syncthreads();
    const raw_t* sy = (const raw_t*)(smem + xoff + a.ag_off);
    for (int p = 0; p < a.ag_n; ++p) {
      raw_t* dst = (raw_t*)a.ag_y[p] + a.ag_row0 + rb;
      for (uint32_t i = threadIdx.x; i < nr; i += NT) dst[i] = sy[i];
    }
    __syncthreads();  // every thread's peer stores precede thread 0's fence (cumulativity)
    if (threadIdx.x == 0) {
      __threadfence_system();
      const uint32_t prev = atomicAdd(a.ag_cnt, 1u);
      if (prev == a.ag_epoch * gridDim.x - 1u) {  // the last CTA: every CTA's stores are fenced
        __threadfence_system();
        for (int p = 0; p < a.ag_n; ++p) st_release_sys(a.ag_flag[p] + a.ag_rank, a.ag_epoch);
      }
    }
  }
  BS_MARK(8);
}

// Short rows (the latency-regime layers: PTB, fc7, CTC): a warp per row reads the row's packed bytes
// straight from global memory (a group of up to 4 steps issued before any is used; with W_STATIC before
// the PDL wait) and gathers x from the L1 cache: no x staging, ring or CTA barrier, so a row costs
// tens of instructions per lane instead of the ring kernel's per-row stage bookkeeping (74 lane
// instructions per nonzero on PTB in round 1's ncu). Its arithmetic is exactly the ring kernel's: acc[v]
// over the panel steps in order; with a tail, the panel total and the tail total (tail entries in t
// order) are reduced separately and added; the same FHFMA. So both kernels give bit-identical rows, and
// the choice (host: per-row bytes, never M) keeps row sharding bit-identical.
// HW (half-warp rows): 16 lanes per row, so that twice as many rows are resident in one wave (PTB: 6000
// rows, one wave of warps holds 4736). Lane h plays the ring kernel's lanes h and h + 16 (separate
// accumulators, acc[j][v] for lane h + 16j); their lane totals are added first, which is exactly the
// butterfly's xor-16 step, and xor 8, 4, 2, 1 follow within the half: the same sums in the same order.
template <int V, int NJ>
__device__ __forceinline__ float row_total(float (&acc)[NJ][V]) {
  float sj[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    float s = acc[j][0];
#pragma unroll
    for (int v = 1; v < V; ++v) s += acc[j][v];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[j][v] = 0.f;
    sj[j] = s;
  }
  float t = sj[0];
  if constexpr (NJ == 2) t = sj[0] + sj[1];
#pragma unroll
  for (int o = 16 / NJ; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// LS (the LSTM step, NJ = 2): a CTA's 8 warps take 16 consecutive gate rows = 4 units per round (the loop
// is CTA-uniform); each row's z = W·x + (bias + pre) goes to shared memory and, after a CTA barrier, one
// thread per unit applies the cell with the ring kernel's expressions (bit-identical, test_gpu_lstm.py).
template <int DT, int V, int IS, bool TP, int NJ, bool LS = false>
__global__ void __launch_bounds__(256, (V <= 4 ? (NJ == 2 ? 3 : 4) : 2)) spmv_rows_kernel(SpmvArgs a) {
  constexpr bool HW = NJ > 1;
  static_assert(!LS || NJ == 2, "the LSTM step takes half-warp rows");
  using raw_t = typename bsk::DTraits<DT>::raw_t;
  constexpr int ES = bsk::DTraits<DT>::kBytes;
  constexpr int P = 32 * V;
  constexpr int ISt = tail_is<IS>();
  constexpr uint32_t RI = run_bytes<V, IS>();
  constexpr uint32_t STEPB = (uint32_t)P * ES + RI;
  constexpr int G = HW ? 3 : 4;                          // steps per load group (HW: registers for two lanes)
  constexpr int WW = (V * ES + 3) / 4;                   // value words per lane and step
  constexpr int IW = IS == 5 ? 2 : IS == 4 ? 1 : (V * IS + 3) / 4;  // index words per lane and step
  const int lane = threadIdx.x & 31;
  constexpr int LPR = 32 / NJ;                           // lanes per row; lane hl plays ring lanes hl + LPR·j
  const int sub = lane / LPR;                            // which row of the warp's NJ rows
  const int hl = lane % LPR;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  pdl_launch_dependents();
  bool waited = !a.w_early;
  if (waited) pdl_wait();
  const raw_t* __restrict__ x = (const raw_t*)a.x;
  const int64_t B = a.B;
  const int k = a.k;
  const int64_t S = a.NBf * k;
  const int64_t kT = (int64_t)k * a.T;
  const int Vt = (int)((a.T + 31) / 32);
  // TP (chosen at launch: a tail with k·V <= 8): the row's tail entries are held in registers, issued with
  // the panel loads (one memory round trip per row); a separate instantiation keeps the registers of the
  // layers without a tail. 16-bit values: value | index << 16 in one register per entry.
  constexpr int TM = TP ? 8 : 1;
  constexpr int TO = ES == 2 ? 1 : TM;
  __shared__ float zs[LS ? 16 : 1];
  const int64_t first = LS ? (int64_t)blockIdx.x * 8 * NJ : ((((int64_t)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5)) * NJ;
  for (int64_t base = first; base < a.M; base += nwarps * NJ) {
    const int64_t r0 = LS ? base + (threadIdx.x >> 5) * NJ : base;
    const int64_t r = r0 + sub;
    const bool live = !HW || r < a.M;  // NJ > 1: the warp's last rows may not exist (the shuffles still need the lanes)
    float bz = 0.f, cp = 0.f;
    if constexpr (LS) {  // the row's bias + pre and the unit's c_prev, loaded before the W stream
      if (hl == 0 && live) {
        bz = a.bias ? bsk::to_float<DT>(__ldg((const raw_t*)a.bias + r)) : 0.f;
        if (a.pre) bz += bsk::to_float<DT>(__ldg((const raw_t*)a.pre + r));
      }
      if (threadIdx.x < 4 && base + 4 * threadIdx.x < a.M) cp = __ldg(a.c_prev + (base / 4 + threadIdx.x));
    }
    float acc[NJ][V];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[j][v] = 0.f;
    const uint8_t* rowA = a.A + r * S * STEPB;
    if (!HW && r + nwarps < a.M) {  // this warp's next row (rows beyond one wave): its lines into L2 now
      const int64_t rn = r + nwarps;
      const int64_t pb = S * STEPB, vb = kT * ES, ib = kT * ISt;
      const uint8_t* line = nullptr;
      if (lane < 16) {
        if ((int64_t)lane * 128 < pb) line = a.A + rn * pb + lane * 128;
      } else if (lane < 24) {
        if ((int64_t)(lane - 16) * 128 < vb) line = a.Bt + rn * vb + (lane - 16) * 128;
      } else if ((int64_t)(lane - 24) * 128 < ib) {
        line = a.Ct + rn * ib + (lane - 24) * 128;
      }
      if (line) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(line));
    }
    uint32_t tw[NJ][TM], to[NJ][TO];
    if constexpr (TP) {
      const raw_t* tv = (const raw_t*)a.Bt + r * kT;
      const uint8_t* ti = a.Ct + r * kT * ISt;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int q = 0; q < TM; ++q) {
          const int tt = q / V, v = q - (q / V) * V;  // entry q = (tt, v)
          const int bl = v * 32 + hl + LPR * j;
          tw[j][q] = 0u;
          if constexpr (ES != 2) to[j][q] = 0u;
          if (live && tt < k && v < Vt && bl < a.T) {
            const int64_t e = (int64_t)tt * a.T + bl;
            const uint32_t o = ISt == 1 ? (uint32_t)__ldg(ti + e) : (uint32_t)__ldg((const uint16_t*)ti + e);
            if constexpr (ES == 2) tw[j][q] = (uint32_t)__ldg(tv + e) | (o << 16);
            else {
              tw[j][q] = (uint32_t)__ldg(tv + e);
              to[j][q] = o;
            }
          }
        }
    }
    // 32-bit index math (x has K < 2^31 elements): the gather column of entry (p, v) of ring lane L is
    // (p·P + 32·v + L)·B + o = p·PB + v·B32 + L·B + o; the panel of step s0 + g follows from one division
    // per group (round 1's 64-bit division per step made ALU the busiest pipe: ncu, PTB).
    const uint32_t Bu = (uint32_t)B, B32 = 32u * Bu, PB = (uint32_t)P * Bu;
    for (int s0 = 0; s0 < (int)S; s0 += G) {
      uint32_t wv[G][NJ][WW], iv[G][NJ][IW];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (live && s0 + g < (int)S) {
          const uint8_t* st = rowA + (int64_t)(s0 + g) * STEPB;
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const int L = hl + LPR * j;
            bsk::Vec<V * ES> vv;
            vv.load(st + L * (V * ES));
#pragma unroll
            for (int q = 0; q < WW; ++q) wv[g][j][q] = vv.w[q];
            if constexpr (IS == 5) {
              bsk::Vec<4> i0;
              bsk::Vec<1> i1;
              i0.load(st + P * ES + 4 * L);
              i1.load(st + P * ES + 128 + L);
              iv[g][j][0] = i0.w[0];
              iv[g][j][1] = i1.w[0];
            } else if constexpr (IS == 4) {
              bsk::Vec<4> i0;
              i0.load(st + P * ES + 4 * L);
              iv[g][j][0] = i0.w[0];
            } else {
              bsk::Vec<V * IS> ii;
              ii.load(st + P * ES + L * (V * IS));
#pragma unroll
              for (int q = 0; q < IW; ++q) iv[g][j][q] = ii.w[q];
            }
          }
        }
      }
      if (!waited) {  // W was static: its loads went out before the dependency wait, x waits for it
        pdl_wait();
        waited = true;
      }
      uint32_t p = (uint32_t)s0 / (uint32_t)k, t = (uint32_t)s0 - p * (uint32_t)k;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (live && s0 + g < (int)S) {
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const uint32_t cb = p * PB + (uint32_t)(hl + LPR * j) * Bu;
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const uint32_t w = ES == 2 ? (wv[g][j][v >> 1] >> (16 * (v & 1))) & 0xffffu : wv[g][j][v];
              uint32_t o;
              if constexpr (IS == 5) o = (v < 7 ? __funnelshift_r(iv[g][j][0], iv[g][j][1], 5 * v) : iv[g][j][1] >> 3) & 31u;
              else if constexpr (IS == 4) o = (iv[g][j][0] >> (4 * v)) & 15u;
              else if constexpr (IS == 1) o = byte_of(iv[g][j][v >> 2], v & 3);
              else o = (iv[g][j][v >> 1] >> (16 * (v & 1))) & 0xffffu;
              bsk::fma_acc<DT>(acc[j][v], w, (uint32_t)__ldg(x + (cb + (uint32_t)v * B32 + o)));
            }
          }
        }
        if (++t == (uint32_t)k) {
          t = 0;
          ++p;
        }
      }
    }
    if (!waited) {
      pdl_wait();
      waited = true;
    }
    float y;
    if (a.T > 0 && k > 0) {
      const float panel = S > 0 ? row_total<V, NJ>(acc) : 0.f;  // (zeroes acc)
      const raw_t* tv = (const raw_t*)a.Bt + r * kT;
      const uint8_t* ti = a.Ct + r * kT * ISt;
      if constexpr (TP) {  // the same (tt, v) order as the loop below
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int q = 0; q < TM; ++q) {
            const int tt = q / V, v = q - (q / V) * V;
            const int bl = v * 32 + hl + LPR * j;
            if (live && tt < k && v < Vt && bl < a.T) {
              const uint32_t cb = ((uint32_t)a.NBf * (uint32_t)P + (uint32_t)bl) * (uint32_t)B;
              const uint32_t w = ES == 2 ? (tw[j][q] & 0xffffu) : tw[j][q];
              const uint32_t o = ES == 2 ? (tw[j][q] >> 16) : to[j][q < TO ? q : 0];
              bsk::fma_acc<DT>(acc[j][v], w, (uint32_t)__ldg(x + (cb + o)));
            }
          }
      }
      for (int tt = TP ? k : 0; tt < k; ++tt) {
        const int64_t e0 = (int64_t)tt * a.T;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const int bl = v * 32 + hl + LPR * j;
            if (live && v < Vt && bl < a.T) {
              const uint32_t w = (uint32_t)__ldg(tv + e0 + bl);
              const uint32_t o = ISt == 1 ? (uint32_t)__ldg(ti + e0 + bl) : (uint32_t)__ldg((const uint16_t*)ti + e0 + bl);
              const uint32_t cb = ((uint32_t)a.NBf * (uint32_t)P + (uint32_t)bl) * (uint32_t)B;
              bsk::fma_acc<DT>(acc[j][v], w, (uint32_t)__ldg(x + (cb + o)));
            }
          }
      }
      const float tail = row_total<V, NJ>(acc);
      y = S > 0 ? panel + tail : tail;
    } else {
      y = row_total<V, NJ>(acc);  // k == 0: 0
    }
    if constexpr (LS) {
      if (hl == 0 && live) zs[(threadIdx.x >> 5) * NJ + sub] = y + bz;
      __syncthreads();
      if (threadIdx.x < 4 && base + 4 * threadIdx.x < a.M) {
        const int u = threadIdx.x;
        const float zi = zs[4 * u], zf = zs[4 * u + 1], zg = zs[4 * u + 2], zo = zs[4 * u + 3];
        const int64_t j = base / 4 + u;
        const float c = apply_act(zf, BS_ACT_SIGMOID) * cp + apply_act(zi, BS_ACT_SIGMOID) * apply_act(zg, BS_ACT_TANH);
        a.c_out[j] = c;
        ((raw_t*)a.h_out)[j] = (raw_t)bsk::from_float<DT>(apply_act(zo, BS_ACT_SIGMOID) * apply_act(c, BS_ACT_TANH));
      }
      __syncthreads();
      continue;
    }
    if (hl == 0 && live) {
      if (a.bias) y += bsk::to_float<DT>(__ldg((const raw_t*)a.bias + r));
      if (a.act) y = apply_act(y, a.act);
      ((raw_t*)a.y)[r] = (raw_t)bsk::from_float<DT>(y);
    }
  }
  if (!waited) pdl_wait();
}

template <int DT, int V, int IS, int NJ, bool LS = false>
const void* rows_fn(const SpmvArgs& a) {
  if (a.T > 0 && a.k > 0 && a.k * V <= 8) return (const void*)spmv_rows_kernel<DT, V, IS, true, NJ, LS>;
  return (const void*)spmv_rows_kernel<DT, V, IS, false, NJ, LS>;
}

template <int DT, int V, int IS, int NJ, bool LS = false>
cudaError_t launch_rows(const SpmvArgs& a0, cudaStream_t s) {
  SpmvArgs a = a0;
  if (!a.pdl) a.w_early = 0;
  const auto& dp = bsk::dev_props();
  // one resident wave of warps (occupancy query): a warp with a second row keeps running (no CTA launch
  // in between) and finds that row's lines already in L2
  const int per_sm = bsk::resident_ctas(rows_fn<DT, V, IS, NJ, LS>(a), 256);
  const int64_t cap = (int64_t)(per_sm > 0 ? per_sm : 1) * dp.sms * 8;
  const int64_t need = (a.M + NJ - 1) / NJ;
  const int64_t warps = need < cap ? need : cap;
  const int64_t grid = (warps + 7) / 8;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  if (a.T > 0 && a.k > 0 && a.k * V <= 8) return cudaLaunchKernelEx(&cfg, spmv_rows_kernel<DT, V, IS, true, NJ, LS>, a);
  return cudaLaunchKernelEx(&cfg, spmv_rows_kernel<DT, V, IS, false, NJ, LS>, a);
}

// The direct kernel pays off while every row gets its own resident warp (one wave): a second wave adds
// a whole row latency (PTB, 6000 rows: 7.0 us direct vs 6.8 us ring; fc7 and CTC, 4096 rows: 1.15-1.35x
// faster direct). Rows beyond one wave of warps take half-warp rows (V <= 4) while those fit one wave,
// else (BS_DIRECT_WAVES, default 2) a warp takes a second row. All give bit-identical rows, so the choice
// may depend on M. Returns 0 (ring kernel), 1 (warp rows) or 2 (half-warp rows).
template <int DT, int V, int IS>
int rows_mode(const SpmvArgs& a) {
  const int per_sm = bsk::resident_ctas(rows_fn<DT, V, IS, 1>(a), 256);
  const int64_t wave = (int64_t)per_sm * bsk::dev_props().sms * 8;
  if (per_sm > 0 && a.M <= wave) return 1;
  static const int half = [] {  // BS_DIRECT_HALF=0: no half-warp rows (A/B)
    const char* e = getenv("BS_DIRECT_HALF");
    return e && e[0] ? atoi(e) : 1;
  }();
  if constexpr (V <= 4) {
    if (half) {
      const int ph = bsk::resident_ctas(rows_fn<DT, V, IS, 2>(a), 256);
      if (ph > 0 && a.M <= (int64_t)ph * bsk::dev_props().sms * 16) return 2;
    }
  }
  static const int waves = [] {  // BS_DIRECT_WAVES: rows per resident warp allowed (a warp's next row is
    const char* e = getenv("BS_DIRECT_WAVES");  // prefetched into L2 while it computes the current one)
    return e && e[0] ? atoi(e) : 2;  // PTB (6000 rows, 1.3 waves): 6.78 us ring -> 6.26 us direct
  }();
  return per_sm > 0 && a.M <= wave * waves ? 1 : 0;
}

template <int DT, int V, int IS>
bool try_rows(const SpmvArgs& a, cudaStream_t s, cudaError_t* e) {
  if (a.lstm) {  // the LSTM step: half-warp rows, 16-bit values, u8 indices, V <= 4; else the ring kernel
    if constexpr (DT != BS_F32 && IS == 1 && V <= 4) {
      *e = launch_rows<DT, V, IS, 2, true>(a, s);
      return true;
    }
    return false;
  }
  const int m = rows_mode<DT, V, IS>(a);
  if (m == 0) return false;
  if constexpr (V <= 4) {
    if (m == 2) {
      *e = launch_rows<DT, V, IS, 2>(a, s);
      return true;
    }
  }
  *e = launch_rows<DT, V, IS, 1>(a, s);
  return true;
}

template <int V, int ES>
struct StageSteps {
  // Q, steps per ring stage: at most 4. The stage loop is unrolled (twice: full and partial stages), so
  // a small Q keeps the kernel's code small; the latency-regime layers are instruction-fetch bound
  // (ncu: no_instructions the top stall on PTB). A/B on one box, against ~2 KB of values per stage:
  // CTC W_hh 4.87 -> 3.27 us, W_ih 4.16 -> 3.35, fc7 90% 3.87 -> 3.68, PTB 90% 7.25 -> 6.61.
  static constexpr int raw = 2048 / (32 * V * ES) < 1 ? 1 : 2048 / (32 * V * ES);
  static constexpr int value = raw > 4 ? 4 : raw;
  static constexpr int big = raw / value;  // stage multiplier of the variant whose stage holds a row's tail
};

template <int DT, int V, int IS, int BT, bool MULTI, int NT, int QM, int NV>
cudaError_t launch_cfg(const SpmvArgs& a0, cudaStream_t s) {
  constexpr int ES = bsk::DTraits<DT>::kBytes;
  constexpr int Q = StageSteps<V, ES>::value * QM;
  constexpr int SB = Q * (32 * V * ES + (int)run_bytes<V, IS>());
  auto kern = spmv_kernel<DT, V, IS, Q, BT, MULTI, NT, NV>;
  const auto& dp = bsk::dev_props();
  cudaError_t perr = cudaSuccess;
  const int static_smem = bsk::prepare_func((const void*)kern, &perr);
  if (static_smem < 0) return perr;
  SpmvArgs a = a0;
  a.tail_rows = 0;
  if (a.T > 0 && a.k > 0) {  // whole rows of tail per ring stage (32 bytes of alignment slack)
    const int64_t per = (int64_t)a.k * a.T * (ES + tail_is<IS>());
    const int64_t R = (SB - 64) / per;
    a.tail_rows = R >= 1 ? (int)(R < 64 ? R : 64) : 0;
  }
  int64_t grid = dp.sms;
  const int64_t need = (a.M + (NT / 32) - 1) / (NT / 32);
  if (grid > need) grid = need;
  // most rows a CTA owns: ceil(M / grid), plus 4 when the LSTM epilogue rounds row ranges to whole units
  const int64_t rows_max = (a.M + grid - 1) / grid + (a.lstm ? 4 : 1);
  const int64_t scratch = MULTI ? rows_max * 4 * NV : 0;
  const int64_t bias_bytes = (a.bias || a.pre || a.lstm) ? rows_max * 4 : 0;
  const int64_t ag_bytes = a.ag_n > 0 ? bsk::align_up(rows_max * ES, 16) : 0;
  const int64_t xslack = (IS == 5 && NV == 1) ? 4096 : 0;  // XALIGN in the kernel
  const int64_t avail =
      dp.smem_optin - static_smem - a.xbytes - scratch - bias_bytes - ag_bytes - xslack - (a.ag_n > 0 ? 16 : 0);
  int NS = (int)(avail / ((NT / 32) * (int64_t)SB));
  if (NS > 4) NS = 4;
  if (NS < (NV == 16 ? 2 : 1)) return cudaErrorInvalidConfiguration;  // NV = 16: the caller falls back to passes of 8
  a.NS = NS;
  a.bias_off = (uint32_t)(a.xbytes + (int64_t)(NT / 32) * NS * SB + scratch);
  a.ag_off = (uint32_t)bsk::align_up(a.bias_off + bias_bytes, 16);
  const int64_t smem_all = xslack + a.ag_off + ag_bytes;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = (size_t)smem_all;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  if (!a.pdl) a.w_early = 0;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

// One 16-warp CTA per SM. (8-warp CTAs in half an SM, so that the next PDL kernel's CTA could be
// resident and prefetch its W, measured 1.1-1.4x slower on every latency-regime layer: DESIGN.md §4.)
template <int DT, int V, int IS, int BT, bool MULTI, int NV>
cudaError_t launch_nt(const SpmvArgs& a, cudaStream_t s) {
  constexpr int ES = bsk::DTraits<DT>::kBytes;
  constexpr int BIG = StageSteps<V, ES>::big;
  if constexpr (BIG > 1 && MULTI) {  // rows with tails always run the MULTI variant
    // tails stream through the ring a whole row per stage; a row's tail that does not fit a small stage
    // would fall back to per-entry global loads (PTB at 50%: 1.6x slower), so take the big-stage variant
    constexpr int64_t SBs = (int64_t)StageSteps<V, ES>::value * (32 * V * ES + (int)run_bytes<V, IS>());
    const int64_t per = (int64_t)a.k * a.T * (ES + tail_is<IS>());
    if (a.T > 0 && a.k > 0 && per > SBs - 64) return launch_cfg<DT, V, IS, BT, MULTI, 512, BIG, NV>(a, s);
  }
  return launch_cfg<DT, V, IS, BT, MULTI, 512, 1, NV>(a, s);
}

template <int DT, int V, int IS, int NV>
cudaError_t launch_t(const SpmvArgs& a, cudaStream_t s) {
  const bool multi = a.nchunks > 1 || a.T > 0;
  if constexpr (IS == 5) {  // B = 32, V = 8 only
    return multi ? launch_nt<DT, V, IS, 32, true, NV>(a, s) : launch_nt<DT, V, IS, 32, false, NV>(a, s);
  } else if constexpr (IS == 4) {  // B <= 16, V = 8: B at run time
    return multi ? launch_nt<DT, V, IS, 0, true, NV>(a, s) : launch_nt<DT, V, IS, 0, false, NV>(a, s);
  } else {
    // B = 32 with V = 8 (16-bit) always uses 5-bit runs, so the B = 32 specialisation is for V < 8
    if constexpr (IS == 1 && V < 8)
      if (a.B == 32) return multi ? launch_nt<DT, V, IS, 32, true, NV>(a, s) : launch_nt<DT, V, IS, 32, false, NV>(a, s);
    return multi ? launch_nt<DT, V, IS, 0, true, NV>(a, s) : launch_nt<DT, V, IS, 0, false, NV>(a, s);
  }
}

template <int DT, int IS, int NV>
cudaError_t dispatch_v(const bsk::Geom& g, const SpmvArgs& a, cudaStream_t s) {
  if constexpr (NV == 1) {
    if (a.direct) {
      cudaError_t e = cudaSuccess;
      switch (g.V) {
        case 1: if (try_rows<DT, 1, IS>(a, s, &e)) return e; break;
        case 2: if (try_rows<DT, 2, IS>(a, s, &e)) return e; break;
        case 4: if (try_rows<DT, 4, IS>(a, s, &e)) return e; break;
        default:
          if constexpr (DT != BS_F32)
            if (try_rows<DT, 8, IS>(a, s, &e)) return e;
      }
    }
  }
  switch (g.V) {
    case 1: return launch_t<DT, 1, IS, NV>(a, s);
    case 2: return launch_t<DT, 2, IS, NV>(a, s);
    case 4: return launch_t<DT, 4, IS, NV>(a, s);
    default:
      if constexpr (DT != BS_F32) return launch_t<DT, 8, IS, NV>(a, s);
      return cudaErrorInvalidValue;
  }
}

template <int DT, int NV>
cudaError_t dispatch_is(const bsk::Geom& g, const SpmvArgs& a, cudaStream_t s) {
  if constexpr (DT != BS_F32)
    if (g.ri == 160) {  // 5-bit index runs
      if constexpr (NV == 1)
        if (a.direct) {
          cudaError_t e = cudaSuccess;
          if (try_rows<DT, 8, 5>(a, s, &e)) return e;
        }
      return launch_t<DT, 8, 5, NV>(a, s);
    } else if (g.ri != g.P * g.is) {  // 4-bit index runs
      if constexpr (NV == 1)
        if (a.direct) {
          cudaError_t e = cudaSuccess;
          if (try_rows<DT, 8, 4>(a, s, &e)) return e;
        }
      return launch_t<DT, 8, 4, NV>(a, s);
    }
  return g.is == 1 ? dispatch_v<DT, 1, NV>(g, a, s) : dispatch_v<DT, 2, NV>(g, a, s);
}

}  // namespace bsk_spmv
