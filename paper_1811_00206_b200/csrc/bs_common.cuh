// bs_common.cuh: shared device/host definitions of the CUDA path (not shared with oracle/).
//
// Geometry of the packed layouts, written from docs/layout.md. The oracle re-derives the same
// geometry independently from the same text; the tests compare bytes.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "bs.h"

namespace bsk {

constexpr int kAlign = 256;

__host__ __device__ inline int64_t align_up(int64_t n, int64_t a) { return (n + a - 1) / a * a; }

inline int dtype_bytes(int dt) { return dt == BS_F32 ? 4 : 2; }

// docs/layout.md "SPMV layout" / "SPMM layout".
struct Geom {
  int64_t M, K, NB;
  int B, k, dt, layout;
  int es;       // value bytes
  int is;       // index bytes (1 if B <= 256 else 2)
  int V;        // lanes own V blocks per panel
  int64_t P;    // 32*V blocks per panel
  int64_t NBf;  // full panels per row
  int64_t T;    // tail blocks per row
  int64_t ri;   // SPMV: bytes of a step's index run (160 = 5-bit runs for B = 32, V = 8; 128 = 4-bit runs for B <= 16, V = 8; else P·is)
  int64_t offA, offB, offC, total;  // SPMV/SPMM: panel steps, tail values, tail indices. SP24: values, metadata.
};

// Returns false on invalid arguments.
inline bool make_geom(int64_t M, int64_t K, int B, int k, int dt, int layout, Geom* g) {
  if (M < 1 || K < 1 || B < 1 || B > 65536 || K % B != 0 || k < 0 || k > B) return false;
  if (dt != BS_F32 && dt != BS_F16 && dt != BS_BF16) return false;
  g->M = M; g->K = K; g->NB = K / B; g->B = B; g->k = k; g->dt = dt; g->layout = layout;
  g->es = dtype_bytes(dt);
  g->is = B <= 256 ? 1 : 2;
  if (layout == BS_LAYOUT_SPMM) {
    // docs/layout.md SPMM: 128-row tiles x CB-block chunks; V holds CB, P the row tiles, NBf the
    // chunks, offB the byte stride of a full row tile.
    const int64_t CB = B <= 64 ? (64 + B - 1) / B : 1;
    g->V = (int)CB;
    g->P = (M + 127) / 128;
    g->NBf = (g->NB + CB - 1) / CB;
    g->T = 0;
    g->ri = 0;
    const int64_t mt_last = M - 128 * (g->P - 1), cb_last = g->NB - CB * (g->NBf - 1);
    auto blob = [&](int64_t mt, int64_t cb) {
      return align_up(mt * cb * k * g->es, 16) + align_up(mt * cb * k * g->is, 16);
    };
    const int64_t tb_full = (g->NBf - 1) * blob(128, CB) + blob(128, cb_last);
    const int64_t tb_last = (g->NBf - 1) * blob(mt_last, CB) + blob(mt_last, cb_last);
    g->offA = 0;
    g->offB = tb_full;
    g->offC = 0;
    g->total = align_up((g->P - 1) * tb_full + tb_last, kAlign);
    return true;
  }
  if (layout == BS_LAYOUT_SPMV) {
    int vmax = 16 / g->es;
    int V = 1;
    while (V * 2 <= vmax && 32LL * V * 2 <= g->NB) V *= 2;
    g->V = V;
    g->P = 32LL * V;
    g->NBf = g->NB / g->P;
    g->T = g->NB - g->NBf * g->P;
    // docs/layout.md: 5-bit index runs (a u32 plane and a byte plane of 40-bit lane fields) when
    // B = 32 and V = 8; 4-bit index runs (one u32 lane word) when B <= 16 and V = 8; otherwise P indices
    // of `is` bytes
    g->ri = (B == 32 && V == 8) ? 160 : (B <= 16 && V == 8) ? 128 : g->P * g->is;
    // region A: M·NBf·k steps of P·es + ri bytes; B / C: tail values / indices (M·k·T each)
    g->offA = 0;
    g->offB = align_up(M * g->NBf * k * (g->P * g->es + g->ri), kAlign);
    g->offC = g->offB + align_up(M * k * g->T * g->es, kAlign);
    g->total = g->offC + align_up(M * k * g->T * g->is, kAlign);
    return true;
  }
  if (layout == BS_LAYOUT_SP24) {
    if (B != 4 || k != 2 || K % 8 != 0) return false;
    g->V = 0; g->P = 0; g->NBf = 0; g->T = 0; g->ri = 0;
    g->offA = 0;
    g->offB = align_up(M * (K / 2) * g->es, kAlign);
    g->offC = 0;
    g->total = g->offB + align_up(M * (g->NB / 2), kAlign);
    return true;
  }
  return false;
}

// Per-device properties cached once per device (the library's only state).
struct DevProps {
  int sms;
  int smem_optin;   // max dynamic smem per block (opt-in)
  int smem_per_sm;
  int l2_bytes;
};
const DevProps& dev_props();

// Opts kernel `func` into the current device's largest dynamic shared memory allocation and returns
// its static shared memory bytes. Done once per (function, device) under the library mutex: the
// attribute belongs to the device context, so a process that drives several GPUs sets it on each.
// Returns a negative value (and leaves *err set) on failure.
int prepare_func(const void* func, cudaError_t* err);

// Resident CTAs per SM of `func` at `threads` threads and no dynamic shared memory (occupancy query,
// cached per function and device). 0 on error.
int resident_ctas(const void* func, int threads);

// Split-K of the tensor-core SpMM kernels: at least this many K chunks per CTA (measured defaults:
// K6 3, K5 6; BS_SPLITK_MIN_CHUNKS overrides both for tuning). It depends on nothing but the
// environment, so the split (and the summation order) stays a function of M and K only.
inline int splitk_min_chunks(int dflt) {
  static const int v = [] {
    const char* e = getenv("BS_SPLITK_MIN_CHUNKS");
    return e && e[0] ? atoi(e) : 0;
  }();
  return v >= 1 ? v : dflt;
}

// Tensor-core SpMM grid order (K5, K6): 1 (default) launches a row tile's column tiles next to each other
// (grid x = column tile · S + split rank, y = row tile), so that they stream the tile's W from HBM once and
// share it through L2; 0 (BS_TC_ORDER=0) is round 1's order (x = row tile · S + rank, y = column tile),
// which streams all of W once per column tile when W exceeds L2.
inline int tc_cols_fast() {
  static const int v = [] {
    const char* e = getenv("BS_TC_ORDER");
    return e && e[0] ? atoi(e) : 1;
  }();
  return v;
}

// Tensor-core SpMM column-tile width: when the grid (row tiles × split × column tiles) would occupy at
// most 1/busy_div of the SMs, narrower column tiles put more CTAs to work. BN only partitions the batch
// columns, so every column's sum is unchanged. BS_TC_FILL=0 turns it off (A/B).
inline int64_t fill_bn(int64_t N, int64_t BN, int64_t ctas_per_coltile, int64_t quantum, int64_t busy_div) {
  static const int on = [] {
    const char* e = getenv("BS_TC_FILL");
    return e && e[0] ? atoi(e) : 1;
  }();
  const int64_t sms = dev_props().sms;
  if (!on || ctas_per_coltile <= 0 || ctas_per_coltile * ((N + BN - 1) / BN) * busy_div > sms) return BN;
  const int64_t want = sms / ctas_per_coltile;  // column tiles that still fit one wave
  int64_t bn = ((N + want - 1) / want + quantum - 1) / quantum * quantum;
  if (bn < quantum) bn = quantum;
  return bn < BN ? bn : BN;
}

}  // namespace bsk

// Launchers implemented in the kernel translation units. All return cudaError_t of the launch.
cudaError_t bsk_launch_prune(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int B, int k,
                             void* vals, uint16_t* idx, cudaStream_t s);
cudaError_t bsk_launch_block_rank(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int B, uint8_t* rank,
                                  cudaStream_t s);
cudaError_t bsk_launch_pack(const void* vals, const uint16_t* idx, const bsk::Geom& g, void* packed,
                            cudaStream_t s);
cudaError_t bsk_launch_decode(const void* vals, const uint16_t* idx, int64_t M, int64_t K, int B, int k, int dt,
                              void* W, int64_t ldw, cudaStream_t s);
size_t bsk_pattern_workspace_bytes(int64_t M, int64_t K, int64_t bh, int64_t bw);
cudaError_t bsk_launch_random_mask(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, double sparsity,
                                   uint8_t* mask, void* ws, cudaStream_t s);
cudaError_t bsk_launch_block_mask(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int64_t bh, int64_t bw,
                                  double sparsity, int criterion, uint8_t* mask, void* ws, cudaStream_t s);
cudaError_t bsk_launch_im2col(const void* in, int dt, int64_t Nimg, int64_t H, int64_t W, int64_t C, int kh, int kw,
                              int pad, int stride, void* X, int64_t ldx, cudaStream_t s);
cudaError_t bsk_launch_unpack(const void* packed, const bsk::Geom& g, void* vals, uint16_t* idx,
                              cudaStream_t s);
cudaError_t bsk_launch_spmv(const bsk::Geom& g, const void* packed, const void* x, void* y, unsigned flags,
                            cudaStream_t s, const void* bias = nullptr, int act = 0);
namespace bsk {
// Operands of the fused LSTM step (bs_lstm_step).
struct LstmIO {
  const void* pre;      // M elements of D or NULL
  const float* c_prev;  // M/4
  float* c_out;         // M/4
  void* h_out;          // M/4 of D
};
}  // namespace bsk
cudaError_t bsk_launch_spmv_allgather(const bsk::Geom& g, const void* packed, const void* x, const bs_allgather& ag,
                                      unsigned flags, cudaStream_t s, const void* bias, int act);
cudaError_t bsk_launch_allgather_wait(const bs_allgather& ag, cudaStream_t s);
cudaError_t bsk_launch_lstm(const bsk::Geom& g, const void* packed, const void* x, const void* bias,
                            const bsk::LstmIO& io, unsigned flags, cudaStream_t s);
cudaError_t bsk_launch_spmv_batch(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx,
                                  void* Y, int64_t ldy, cudaStream_t s);
// spmv: the batch-1 product of bs_spmv (CUDA cores, HBM-bound). Otherwise the batched product of bs_spmm,
// whose per-column summation order does not depend on N (tensor cores whenever the operands allow).
cudaError_t bsk_launch_sp24(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx, void* Y,
                            int64_t ldy, cudaStream_t s, bool spmv);
cudaError_t bsk_launch_spmm(const bsk::Geom& g, const void* packed, const void* X, int64_t N,
                            int64_t ldx, void* Y, int64_t ldy, cudaStream_t s);
cudaError_t bsk_launch_conv24(const bsk::Geom& g, const void* packed, const void* in, int64_t Nimg, int64_t H, int64_t W,
                              int64_t C, int kh, int kw, int pad, const void* bias, int act, void* Y, cudaStream_t s);
cudaError_t bsk_launch_sp24_fused(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx, void* Y,
                                  int64_t ldy, const void* bias, int act, cudaStream_t s);
cudaError_t bsk_launch_spmm_fused(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx,
                                  void* Y, int64_t ldy, const void* bias, int act, cudaStream_t s);
cudaError_t bsk_launch_conv(const bsk::Geom& g, const void* packed, const void* in, int64_t Nimg, int64_t H, int64_t W,
                            int64_t C, int kh, int kw, int pad, const void* bias, int act, void* Y, cudaStream_t s);
