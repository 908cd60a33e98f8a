// spmv.cu: host side of K3 bs_spmv and of the batched (8 columns per pass) variant: argument set-up,
// K-chunking and dispatch to the per-dtype instantiations (spmv_f16.cu, spmv_bf16.cu, spmv_f32.cu).
// The kernel and its design notes are in spmv_impl.cuh.
#include "spmv_impl.cuh"

using bsk_spmv::SpmvArgs;
using bsk_spmv::kXBudget;
using bsk_spmv::kMaxChunks;

cudaError_t bsk_spmv_dispatch_f16(const bsk::Geom& g, const SpmvArgs& a, int nv, cudaStream_t s);
cudaError_t bsk_spmv_dispatch_bf16(const bsk::Geom& g, const SpmvArgs& a, int nv, cudaStream_t s);
cudaError_t bsk_spmv_dispatch_f32(const bsk::Geom& g, const SpmvArgs& a, cudaStream_t s);

// nv = 1: SpMV (y = W·x). nv = 8: one pass over W for up to 8 batch columns (16-bit dtypes): column
// n of X at x + n·ldx, column n of Y at y + n·ldy, n < ncols.
// chunk_nv: the slot width that fixes the K-chunking (the panels summed per partial). Batch passes of
// every width use chunk_nv = 8, so a column's fp32 summation order does not depend on the pass width
// (NV = 2, 4, 8 accumulate each column in the same order), i.e. on N.
static cudaError_t launch_spmv_nv(const bsk::Geom& g, const void* packed, const void* x, int64_t ldx, void* y,
                                  int64_t ldy, int ncols, int nv, int chunk_nv, unsigned flags, cudaStream_t s,
                                  const void* bias = nullptr, int act = 0, const bsk::LstmIO* lstm = nullptr,
                                  const bs_allgather* ag = nullptr) {
  SpmvArgs a;
  a.ag_n = 0;
  a.ag_rank = 0;
  a.ag_row0 = 0;
  a.ag_cnt = nullptr;
  a.ag_epoch = 0;
  a.ag_off = 0;
  for (int p = 0; p < 8; ++p) {
    a.ag_y[p] = nullptr;
    a.ag_flag[p] = nullptr;
  }
  if (ag && nv == 1) {
    a.ag_n = ag->nranks;
    a.ag_rank = ag->rank;
    a.ag_row0 = ag->row0;
    a.ag_cnt = ag->counter;
    a.ag_epoch = ag->epoch;
    for (int p = 0; p < ag->nranks; ++p) {
      a.ag_y[p] = ag->y[p];
      a.ag_flag[p] = ag->flags[p];
    }
  }
  a.bias = nv == 1 ? bias : nullptr;
  a.act = nv == 1 ? act : 0;
  a.bias_off = 0;
  a.lstm = nv == 1 && lstm != nullptr;
  a.pre = a.lstm ? lstm->pre : nullptr;
  a.c_prev = a.lstm ? lstm->c_prev : nullptr;
  a.c_out = a.lstm ? lstm->c_out : nullptr;
  a.h_out = a.lstm ? lstm->h_out : nullptr;
  a.pdl = (flags & BS_SPMV_PDL) != 0;
  a.w_early = a.pdl && (flags & BS_SPMV_W_STATIC) != 0;
  const uint8_t* base = (const uint8_t*)packed;
  a.A = base + g.offA;
  a.Bt = base + g.offB;
  a.Ct = base + g.offC;
  a.x = x;
  a.y = y;
  a.M = g.M;
  a.NB = g.NB;
  a.NBf = g.NBf;
  a.T = g.T;
  a.B = g.B;
  a.k = g.k;
  a.NS = 0;
  a.tail_rows = 0;
  a.ldx = ldx;
  a.ldy = ldy;
  a.ncols = ncols;
  const bool aligned = ((uintptr_t)x & 15) == 0 && (nv == 1 || ldx % 8 == 0);
  a.xvec = aligned && (g.es == 2 ? g.B % 8 == 0 : g.B % 4 == 0);
  // chunking of the K dimension by whole panels (depends only on K, B, dtype: deterministic)
  const int64_t group_bytes = (int64_t)g.B * 32 * g.es * nv;  // 32 blocks of x slots
  const int64_t chunk_group = (int64_t)g.B * 32 * g.es * chunk_nv;
  const int64_t tail_groups = (g.NB + 31) / 32 - g.NBf * g.V;
  // 16-bit SpMV stores x in group pairs (spmv_impl.cuh stage_x PAIR): round staged groups up to even. With V = 1
  // unpaired halfword slots put lanes 2m, 2m+1 in one bank with different offsets (2-way conflicts, T2 model)
  const bool pair = g.es == 2 && nv == 1;
  auto ev = [&](int64_t n) { return pair ? (n + 1) / 2 * 2 : n; };
  if (g.NBf > 0 && g.k > 0) {
    int64_t PC = kXBudget / (chunk_group * g.V);
    if (PC < 1) PC = 1;
    if (PC > g.NBf) PC = g.NBf;
    int64_t nchunks = (g.NBf + PC - 1) / PC;
    if (nchunks > kMaxChunks) {
      nchunks = kMaxChunks;
      PC = (g.NBf + nchunks - 1) / nchunks;
      nchunks = (g.NBf + PC - 1) / PC;
    }
    const int64_t last_np = g.NBf - (nchunks - 1) * PC;
    a.PC = (int)PC;
    a.nchunks = (int)nchunks;
    a.tail_in_last = (last_np * g.V + tail_groups) * chunk_group <= kXBudget;
    int64_t xb = PC * g.V * group_bytes;
    const int64_t need_last = ev(last_np * g.V + (a.tail_in_last ? tail_groups : 0)) * group_bytes;
    if (need_last > xb) xb = need_last;
    if (!a.tail_in_last && ev(tail_groups) * group_bytes > xb) xb = ev(tail_groups) * group_bytes;
    a.xbytes = (int)xb;
  } else {  // no full panels (or k == 0): the tail groups only
    a.PC = 1;
    a.nchunks = 0;
    a.tail_in_last = 0;
    a.xbytes = g.k > 0 ? (int)(ev(tail_groups) * group_bytes) : 0;
  }
  // Short rows take the direct kernel (spmv_impl.cuh spmv_rows_kernel): plain SpMV / fused bias+act / the
  // LSTM step (half-warp rows, 4 units per CTA round), one x chunk, at most kDirectRowBytes of packed bytes per row (BS_DIRECT_ROW_BYTES overrides; 0 = off).
  // The choice depends on (K, B, k, dtype) only, never on M, and both kernels sum in the same order.
  {
    static const int64_t thr = [] {
      const char* e = getenv("BS_DIRECT_ROW_BYTES");
      return e && e[0] ? (int64_t)atoll(e) : (int64_t)2304;  // 2304: fc6 at 97 % (2064 B) 7.1 -> 6.4 us
    }();
    const int ist = g.ri == g.P * g.is ? g.is : 1;
    const int64_t row_bytes = g.NBf * g.k * (g.P * g.es + g.ri) + (int64_t)g.k * g.T * (g.es + ist);
    a.direct = nv == 1 && ag == nullptr && a.nchunks <= 1 && row_bytes <= thr &&
               (flags & BS_SPMV_RING) == 0;
  }
  if (a.xbytes > bsk::dev_props().smem_optin - 16 * 1024) return cudaErrorInvalidConfiguration;
  if ((uint64_t)g.M * (uint64_t)(bsk::dev_props().sms + 1) >= (1ULL << 32)) return cudaErrorInvalidConfiguration;
  switch (g.dt) {
    case BS_F32: return nv == 1 ? bsk_spmv_dispatch_f32(g, a, s) : cudaErrorNotSupported;
    case BS_F16: return bsk_spmv_dispatch_f16(g, a, nv, s);
    default: return bsk_spmv_dispatch_bf16(g, a, nv, s);
  }
}

cudaError_t bsk_launch_spmv(const bsk::Geom& g, const void* packed, const void* x, void* y, unsigned flags,
                            cudaStream_t s, const void* bias, int act) {
  return launch_spmv_nv(g, packed, x, 0, y, 0, 1, 1, 1, flags, s, bias, act);
}

// The row shard's SpMV with the all-gather of y fused into its epilogue (spmv_impl.cuh).
cudaError_t bsk_launch_spmv_allgather(const bsk::Geom& g, const void* packed, const void* x, const bs_allgather& ag,
                                      unsigned flags, cudaStream_t s, const void* bias, int act) {
  return launch_spmv_nv(g, packed, x, 0, ag.y[ag.rank], 0, 1, 1, 1, flags, s, bias, act, nullptr, &ag);
}

namespace {
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Waits until every rank's flag on this rank has reached `epoch` (wrap-safe compare: a faster rank may
// already have raised the next epoch).
__global__ void ag_wait_kernel(const uint32_t* flags, int n, uint32_t epoch) {
  const int i = threadIdx.x;
  if (i < n)
    while ((int32_t)(ld_acquire_sys_u32(flags + i) - epoch) < 0) __nanosleep(64);
  __syncwarp();
}
}  // namespace

cudaError_t bsk_launch_allgather_wait(const bs_allgather& ag, cudaStream_t s) {
  ag_wait_kernel<<<1, 32, 0, s>>>(ag.flags[ag.rank], ag.nranks, ag.epoch);
  return cudaGetLastError();
}

// One LSTM step: the gate rows' SpMV with the cell applied in the kernel's epilogue (spmv_impl.cuh).
cudaError_t bsk_launch_lstm(const bsk::Geom& g, const void* packed, const void* x, const void* bias,
                            const bsk::LstmIO& io, unsigned flags, cudaStream_t s) {
  return launch_spmv_nv(g, packed, x, 0, io.h_out, 0, 1, 1, 1, flags, s, bias, 0, &io);
}

// Batched product on the SPMV layout (16-bit): passes of up to 8 batch columns, each one stream of W;
// a pass of w columns uses x slots of NV = 2, 4 or 8 columns (the smallest >= w). When 9..16 columns
// remain and 32-byte slots fit in shared memory (K up to about 3000 columns: the CTC layers), one pass
// of NV = 16 streams W once for all of them. Every pass uses the K-chunking of NV = 8, so column n's
// summation order does not depend on N.
cudaError_t bsk_launch_spmv_batch(const bsk::Geom& g, const void* packed, const void* X, int64_t N, int64_t ldx,
                                  void* Y, int64_t ldy, cudaStream_t s) {
  if (g.es != 2) return cudaErrorNotSupported;
  for (int64_t n0 = 0; n0 < N;) {
    if (N - n0 > 8) {
      const int nc = (int)((N - n0) < 16 ? (N - n0) : 16);
      cudaError_t e = launch_spmv_nv(g, packed, (const uint16_t*)X + n0 * ldx, ldx, (uint16_t*)Y + n0 * ldy, ldy, nc,
                                     16, 8, BS_SPMV_PDL, s);
      if (e == cudaSuccess) {
        n0 += nc;
        continue;
      }
      if (e != cudaErrorInvalidConfiguration) return e;  // 32-byte slots do not fit: passes of 8
    }
    const int nc = (int)((N - n0) < 8 ? (N - n0) : 8);
    const int nv = nc <= 2 ? 2 : nc <= 4 ? 4 : 8;
    cudaError_t e =
        launch_spmv_nv(g, packed, (const uint16_t*)X + n0 * ldx, ldx, (uint16_t*)Y + n0 * ldy, ldy, nc, nv, 8, BS_SPMV_PDL, s);
    if (e != cudaSuccess) return e;
    n0 += nc;
  }
  return cudaSuccess;
}
