// bs_api.cu: the C ABI of libbs.so (include/bs.h). It validates arguments and dispatches to the
// kernels. It never allocates device memory and never synchronises.
#include <cuda.h>
#include <math.h>
#include <string.h>
#include <map>
#include <mutex>
#include <utility>

#include "bs_common.cuh"
#include "spmv_impl.cuh"

int64_t bsk_spmv_smem_bytes(const bsk::Geom& g);

namespace bsk {

const DevProps& dev_props() {
  static DevProps props[64];
  static bool have[64] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> lock(mu);
  if (!have[dev]) {
    DevProps p{};
    cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&p.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&p.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&p.l2_bytes, cudaDevAttrL2CacheSize, dev);
    if (p.sms <= 0) p.sms = 148;
    props[dev] = p;
    have[dev] = true;
  }
  return props[dev];
}

int prepare_func(const void* func, cudaError_t* err) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const int optin = dev_props().smem_optin;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({func, dev});
  if (it != done.end()) return it->second;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, func);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  if (e != cudaSuccess) {
    *err = e;
    return -1;
  }
  done[{func, dev}] = (int)fa.sharedSizeBytes;
  return (int)fa.sharedSizeBytes;
}

int resident_ctas(const void* func, int threads) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({func, dev});
  if (it != done.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, func, threads, 0) != cudaSuccess) n = 0;
  done[{func, dev}] = n;
  return n;
}

}  // namespace bsk

namespace {

int from_cuda(cudaError_t e) {
  if (e == cudaSuccess) return BS_OK;
  if (e == cudaErrorNotSupported || e == cudaErrorInvalidConfiguration) return BS_ERR_UNSUPPORTED;
  return BS_ERR_CUDA;
}

bool valid_dt(int dt) { return dt == BS_F32 || dt == BS_F16 || dt == BS_BF16; }

int check_shape(int64_t M, int64_t K, int B, int k) {
  if (M < 1 || K < 1 || B < 1) return BS_ERR_SHAPE;
  if (B > 65536) return BS_ERR_UNSUPPORTED;
  if (K % B != 0) return BS_ERR_SHAPE;
  if (k < 0 || k > B) return BS_ERR_ARG;
  return BS_OK;
}

int matrix_geom(const bs_matrix* A, bsk::Geom* g) {
  if (!A) return BS_ERR_ARG;
  if (!valid_dt(A->dt)) return BS_ERR_DTYPE;
  int st = check_shape(A->M, A->K, A->block, A->k);
  if (st) return st;
  if (A->layout != BS_LAYOUT_SPMV && A->layout != BS_LAYOUT_SPMM && A->layout != BS_LAYOUT_SP24)
    return BS_ERR_ARG;
  if (!bsk::make_geom(A->M, A->K, A->block, A->k, A->dt, A->layout, g)) return BS_ERR_UNSUPPORTED;
  if (!A->packed && g->total > 0) return BS_ERR_ARG;  /* k == 0 packs to zero bytes */
  return BS_OK;
}

}  // namespace

extern "C" {

int bs_k_from_sparsity(int block, double sparsity) {
  if (block < 1 || !(sparsity >= 0.0) || !(sparsity < 1.0)) return -1;
  return (int)lround((1.0 - sparsity) * (double)block);
}

size_t bs_packed_bytes(int64_t M, int64_t K, int block, int k, int dt, int layout) {
  bsk::Geom g;
  if (!bsk::make_geom(M, K, block, k, dt, layout, &g)) return 0;
  return (size_t)g.total;
}

int bs_choose_layout(int64_t M, int64_t K, int block, int k, int dt, int64_t N) {
  if (!valid_dt(dt) || check_shape(M, K, block, k) || N < 1) return -1;
  const bool half = dt != BS_F32;
  if (block == 4 && k == 2 && half && K % 128 == 0) return BS_LAYOUT_SP24;
  // one 16-column pass streams W once when 32-byte x slots fit (CTC: 7.7 us vs 8.7 us on tensor cores)
  const bool sixteen = N <= 16 && K <= 3072;
  if (N > 8 && !sixteen && half && 64 % block == 0) return BS_LAYOUT_SPMM;
  return BS_LAYOUT_SPMV;
}

const char* bs_status_str(int status) {
  switch (status) {
    case BS_OK: return "BS_OK";
    case BS_ERR_ARG: return "BS_ERR_ARG";
    case BS_ERR_SHAPE: return "BS_ERR_SHAPE";
    case BS_ERR_DTYPE: return "BS_ERR_DTYPE";
    case BS_ERR_UNSUPPORTED: return "BS_ERR_UNSUPPORTED";
    case BS_ERR_CUDA: return "BS_ERR_CUDA";
    default: return "BS_UNKNOWN";
  }
}

const char* bs_version(void) { return "libbs 0.1 sm_100a (balanced sparsity, arXiv 1811.00206)"; }

int bs_prune_k(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int block, int k, void* vals,
               uint16_t* idx, void* stream) {
  if (!valid_dt(dt)) return BS_ERR_DTYPE;
  int st = check_shape(M, K, block, k);
  if (st) return st;
  if (!W || ldw < K) return BS_ERR_ARG;
  if (k == 0) return BS_OK;
  if (!vals || !idx) return BS_ERR_ARG;
  return from_cuda(bsk_launch_prune(W, dt, M, K, ldw, block, k, vals, idx, (cudaStream_t)stream));
}

int bs_block_rank(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int block, uint8_t* rank,
                  void* stream) {
  if (!valid_dt(dt)) return BS_ERR_DTYPE;
  int st = check_shape(M, K, block, 0);
  if (st) return st;
  if (!W || !rank || ldw < K) return BS_ERR_ARG;
  if (block > 32 || (block & (block - 1)) != 0) return BS_ERR_UNSUPPORTED;
  return from_cuda(bsk_launch_block_rank(W, dt, M, K, ldw, block, rank, (cudaStream_t)stream));
}

int bs_prune(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int block, double sparsity, int* k_out,
             void* vals, uint16_t* idx, void* stream) {
  if (!(sparsity >= 0.0) || !(sparsity < 1.0)) return BS_ERR_ARG;
  if (block < 1) return BS_ERR_SHAPE;
  const int k = bs_k_from_sparsity(block, sparsity);
  if (k_out) *k_out = k;
  return bs_prune_k(W, dt, M, K, ldw, block, k, vals, idx, stream);
}

int bs_pack(const void* vals, const uint16_t* idx, int64_t M, int64_t K, int block, int k, int dt, int layout,
            void* packed, void* stream) {
  if (!valid_dt(dt)) return BS_ERR_DTYPE;
  int st = check_shape(M, K, block, k);
  if (st) return st;
  if (layout != BS_LAYOUT_SPMV && layout != BS_LAYOUT_SPMM && layout != BS_LAYOUT_SP24) return BS_ERR_ARG;
  bsk::Geom g;
  if (!bsk::make_geom(M, K, block, k, dt, layout, &g)) return BS_ERR_UNSUPPORTED;
  if ((!packed && g.total > 0) || (k > 0 && (!vals || !idx))) return BS_ERR_ARG;
  if (g.total == 0) return BS_OK;
  return from_cuda(bsk_launch_pack(vals, idx, g, packed, (cudaStream_t)stream));
}

int bs_unpack(const void* packed, int64_t M, int64_t K, int block, int k, int dt, int layout, void* vals,
              uint16_t* idx, void* stream) {
  if (!valid_dt(dt)) return BS_ERR_DTYPE;
  int st = check_shape(M, K, block, k);
  if (st) return st;
  if (layout != BS_LAYOUT_SPMV && layout != BS_LAYOUT_SPMM && layout != BS_LAYOUT_SP24) return BS_ERR_ARG;
  bsk::Geom g;
  if (!bsk::make_geom(M, K, block, k, dt, layout, &g)) return BS_ERR_UNSUPPORTED;
  if ((!packed && g.total > 0) || (k > 0 && (!vals || !idx))) return BS_ERR_ARG;
  if (k == 0) return BS_OK;
  return from_cuda(bsk_launch_unpack(packed, g, vals, idx, (cudaStream_t)stream));
}

double bs_schedule_sparsity(double target, int n, int i) {
  if (n < 1 || i < 0 || i > n || !(target >= 0.0) || !(target < 1.0)) return -1.0;
  const double u = 1.0 - (double)i / (double)n;
  return target * (1.0 - u * u * u);
}

int64_t bs_keep_count(int64_t n, double sparsity) {
  if (n < 0 || !(sparsity >= 0.0) || !(sparsity < 1.0)) return -1;
  return (int64_t)llround((1.0 - sparsity) * (double)n);
}

int bs_decode(const void* vals, const uint16_t* idx, int64_t M, int64_t K, int block, int k, int dt, void* W,
              int64_t ldw, void* stream) {
  if (!valid_dt(dt)) return BS_ERR_DTYPE;
  int st = check_shape(M, K, block, k);
  if (st) return st;
  if (!W || ldw < K || (k > 0 && (!vals || !idx))) return BS_ERR_ARG;
  return from_cuda(bsk_launch_decode(vals, idx, M, K, block, k, dt, W, ldw, (cudaStream_t)stream));
}

size_t bs_pattern_workspace_bytes(int64_t M, int64_t K, int64_t bh, int64_t bw) {
  if (M < 1 || K < 1 || bh < 0 || bw < 0 || (bh > 0 && M % bh) || (bw > 0 && K % bw)) return 0;
  return bsk_pattern_workspace_bytes(M, K, bh, bw);
}

int bs_random_mask(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, double sparsity, uint8_t* mask,
                   void* workspace, size_t workspace_bytes, void* stream) {
  if (!valid_dt(dt)) return BS_ERR_DTYPE;
  if (M < 1 || K < 1) return BS_ERR_SHAPE;
  if (!W || !mask || !workspace || ldw < K || !(sparsity >= 0.0) || !(sparsity < 1.0)) return BS_ERR_ARG;
  if (workspace_bytes < bsk_pattern_workspace_bytes(M, K, 0, 0)) return BS_ERR_ARG;
  return from_cuda(bsk_launch_random_mask(W, dt, M, K, ldw, sparsity, mask, workspace, (cudaStream_t)stream));
}

int bs_block_mask(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int64_t bh, int64_t bw, double sparsity,
                  int criterion, uint8_t* mask, void* workspace, size_t workspace_bytes, void* stream) {
  if (!valid_dt(dt)) return BS_ERR_DTYPE;
  if (M < 1 || K < 1 || bh < 1 || bw < 1 || M % bh || K % bw) return BS_ERR_SHAPE;
  if (!W || !mask || !workspace || ldw < K || !(sparsity >= 0.0) || !(sparsity < 1.0)) return BS_ERR_ARG;
  if (criterion != 0 && criterion != 1) return BS_ERR_ARG;
  if (workspace_bytes < bsk_pattern_workspace_bytes(M, K, bh, bw)) return BS_ERR_ARG;
  return from_cuda(
      bsk_launch_block_mask(W, dt, M, K, ldw, bh, bw, sparsity, criterion, mask, workspace, (cudaStream_t)stream));
}

int bs_im2col(const void* in, int dt, int64_t Nimg, int64_t H, int64_t W, int64_t C, int kh, int kw, int pad,
              int stride, void* X, int64_t ldx, void* stream) {
  if (!valid_dt(dt)) return BS_ERR_DTYPE;
  if (Nimg < 1 || H < 1 || W < 1 || C < 1 || kh < 1 || kw < 1 || pad < 0 || stride < 1) return BS_ERR_SHAPE;
  const int64_t OH = (H + 2 * pad - kh) / stride + 1, OW = (W + 2 * pad - kw) / stride + 1;
  if (H + 2 * pad < kh || W + 2 * pad < kw || OH < 1 || OW < 1) return BS_ERR_SHAPE;
  if (!in || !X || ldx < (int64_t)kh * kw * C) return BS_ERR_ARG;
  return from_cuda(bsk_launch_im2col(in, dt, Nimg, H, W, C, kh, kw, pad, stride, X, ldx, (cudaStream_t)stream));
}

int bs_spmm_fused(const bs_matrix* A, const void* X, int64_t N, int64_t ldx, const void* bias, int act, void* Y,
                  int64_t ldy, void* stream) {
  bsk::Geom g;
  int st = matrix_geom(A, &g);
  if (st) return st;
  if (!X || !Y || N < 1 || ldx < g.K || ldy < g.M) return BS_ERR_ARG;
  if (act < BS_ACT_NONE || act > BS_ACT_TANH) return BS_ERR_ARG;
  const cudaError_t e = g.layout == BS_LAYOUT_SP24
                            ? bsk_launch_sp24_fused(g, A->packed, X, N, ldx, Y, ldy, bias, act, (cudaStream_t)stream)
                            : bsk_launch_spmm_fused(g, A->packed, X, N, ldx, Y, ldy, bias, act, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported) return BS_ERR_UNSUPPORTED;
  return from_cuda(e);
}

int bs_conv2d(const bs_matrix* A, const void* in, int64_t Nimg, int64_t H, int64_t W, int64_t C, int kh, int kw,
              int pad, int stride, const void* bias, int act, void* Y, void* stream) {
  bsk::Geom g;
  int st = matrix_geom(A, &g);
  if (st) return st;
  if (Nimg < 1 || H < 1 || W < 1 || C < 1 || kh < 1 || kw < 1 || pad < 0 || stride < 1) return BS_ERR_SHAPE;
  if (g.K != (int64_t)kh * kw * C) return BS_ERR_SHAPE;
  if (H + 2 * pad < kh || W + 2 * pad < kw) return BS_ERR_SHAPE;
  if (!in || !Y) return BS_ERR_ARG;
  if (act < BS_ACT_NONE || act > BS_ACT_TANH) return BS_ERR_ARG;
  if (stride != 1) return BS_ERR_UNSUPPORTED;
  const cudaError_t e =
      g.layout == BS_LAYOUT_SP24
          ? bsk_launch_conv24(g, A->packed, in, Nimg, H, W, C, kh, kw, pad, bias, act, Y, (cudaStream_t)stream)
          : bsk_launch_conv(g, A->packed, in, Nimg, H, W, C, kh, kw, pad, bias, act, Y, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported) return BS_ERR_UNSUPPORTED;
  return from_cuda(e);
}

int64_t bs_x_slot_offset(int64_t K, int block, int dt, int nv, int64_t b, int o, int part) {
  bsk::Geom g;
  if (!bsk::make_geom(1, K, block, 1, dt, BS_LAYOUT_SPMV, &g)) return -1;
  if (b < 0 || b >= g.NB || o < 0 || o >= block || part < 0 || part > (nv == 16 ? 1 : 0)) return -1;
  if (!(nv == 1 || ((nv == 2 || nv == 4 || nv == 8 || nv == 16) && g.es == 2))) return -1;
  const bool pair = g.es == 2 && nv == 1;  // as launch_spmv_nv / the kernel's PAIR
  return (int64_t)bsk_spmv::x_slot((uint32_t)(b >> 5), (uint32_t)o, (uint32_t)(b & 31), (uint32_t)block,
                                   (uint32_t)g.es, (uint32_t)nv, pair) +
         (int64_t)bsk_spmv::x_part_off((uint32_t)(b & 31), (uint32_t)nv, (uint32_t)part);
}

int bs_spmv_ex(const bs_matrix* A, const void* x, void* y, unsigned flags, void* stream) {
  bsk::Geom g;
  int st = matrix_geom(A, &g);
  if (st) return st;
  if (!x || !y) return BS_ERR_ARG;
  if (flags & ~(BS_SPMV_PDL | BS_SPMV_W_STATIC | BS_SPMV_RING)) return BS_ERR_ARG;
  if (g.layout == BS_LAYOUT_SP24)  // 2:4: CUDA-core path with 2-bit metadata
    return from_cuda(bsk_launch_sp24(g, A->packed, x, 1, g.K, y, g.M, (cudaStream_t)stream, true));
  if (g.layout != BS_LAYOUT_SPMV) return BS_ERR_UNSUPPORTED;  // SPMM tiles feed bs_spmm
  return from_cuda(bsk_launch_spmv(g, A->packed, x, y, flags, (cudaStream_t)stream));
}

int bs_spmv_fused(const bs_matrix* A, const void* x, const void* bias, int act, void* y, unsigned flags,
                  void* stream) {
  if (!bias && act == BS_ACT_NONE) return bs_spmv_ex(A, x, y, flags, stream);
  bsk::Geom g;
  int st = matrix_geom(A, &g);
  if (st) return st;
  if (!x || !y) return BS_ERR_ARG;
  if (flags & ~(BS_SPMV_PDL | BS_SPMV_W_STATIC | BS_SPMV_RING)) return BS_ERR_ARG;
  if (act < BS_ACT_NONE || act > BS_ACT_TANH) return BS_ERR_ARG;
  if (g.layout != BS_LAYOUT_SPMV) return BS_ERR_UNSUPPORTED;
  return from_cuda(bsk_launch_spmv(g, A->packed, x, y, flags, (cudaStream_t)stream, bias, act));
}

int bs_lstm_step(const bs_matrix* A, const void* x, const void* pre, const void* bias, const float* c_prev,
                 void* h_out, float* c_out, unsigned flags, void* stream) {
  bsk::Geom g;
  int st = matrix_geom(A, &g);
  if (st) return st;
  if (!x || !c_prev || !h_out || !c_out) return BS_ERR_ARG;
  if (flags & ~(BS_SPMV_PDL | BS_SPMV_W_STATIC | BS_SPMV_RING)) return BS_ERR_ARG;
  if (g.M % 4 != 0) return BS_ERR_SHAPE;
  if (g.layout != BS_LAYOUT_SPMV) return BS_ERR_UNSUPPORTED;
  const bsk::LstmIO io{pre, c_prev, c_out, h_out};
  return from_cuda(bsk_launch_lstm(g, A->packed, x, bias, io, flags, (cudaStream_t)stream));
}

static bool valid_ag(const bs_allgather* ag) {
  if (!ag || ag->nranks < 1 || ag->nranks > 8 || ag->rank < 0 || ag->rank >= ag->nranks || ag->row0 < 0) return false;
  if (!ag->counter || ag->epoch == 0) return false;
  for (int p = 0; p < ag->nranks; ++p)
    if (!ag->y[p] || !ag->flags[p]) return false;
  return true;
}

int bs_spmv_allgather(const bs_matrix* A, const void* x, const void* bias, int act, const bs_allgather* ag,
                      unsigned flags, void* stream) {
  bsk::Geom g;
  int st = matrix_geom(A, &g);
  if (st) return st;
  if (!x || !valid_ag(ag)) return BS_ERR_ARG;
  if (flags & ~(BS_SPMV_PDL | BS_SPMV_W_STATIC | BS_SPMV_RING)) return BS_ERR_ARG;
  if (act < BS_ACT_NONE || act > BS_ACT_TANH) return BS_ERR_ARG;
  if (g.layout != BS_LAYOUT_SPMV) return BS_ERR_UNSUPPORTED;
  return from_cuda(bsk_launch_spmv_allgather(g, A->packed, x, *ag, flags, (cudaStream_t)stream, bias, act));
}

int bs_allgather_wait(const bs_allgather* ag, void* stream) {
  if (!valid_ag(ag)) return BS_ERR_ARG;
  return from_cuda(bsk_launch_allgather_wait(*ag, (cudaStream_t)stream));
}

using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

int bs_peer_export(const void* ptr, void* handle, int64_t* offset) {
  if (!ptr || !handle || !offset) return BS_ERR_ARG;
  static AddrRangeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return BS_ERR_CUDA;
    fn = (AddrRangeFn)p;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return BS_ERR_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, (void*)base) != cudaSuccess) return BS_ERR_CUDA;
  memcpy(handle, &h, sizeof(h));
  *offset = (int64_t)((CUdeviceptr)ptr - base);
  return BS_OK;
}

int bs_peer_import(const void* handle, int64_t offset, void** ptr) {
  if (!handle || !ptr || offset < 0) return BS_ERR_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return BS_ERR_CUDA;
  *ptr = (char*)base + offset;
  return BS_OK;
}

int bs_peer_close(void* ptr, int64_t offset) {
  if (!ptr || offset < 0) return BS_ERR_ARG;
  return cudaIpcCloseMemHandle((char*)ptr - offset) == cudaSuccess ? BS_OK : BS_ERR_CUDA;
}

int bs_spmv(const bs_matrix* A, const void* x, void* y, void* stream) {
  return bs_spmv_ex(A, x, y, BS_SPMV_PDL, stream);
}

int bs_spmv_host(const bs_matrix* A, const void* x_host, void* y_host, void* x_dev, void* y_dev, void* stream) {
  bsk::Geom g;
  int st = matrix_geom(A, &g);
  if (st) return st;
  if (!x_host || !y_host || !x_dev || !y_dev) return BS_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(x_dev, x_host, (size_t)(g.K * g.es), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return BS_ERR_CUDA;
  st = bs_spmv(A, x_dev, y_dev, stream);
  if (st) return st;
  if (cudaMemcpyAsync(y_host, y_dev, (size_t)(g.M * g.es), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return BS_ERR_CUDA;
  return BS_OK;
}

int bs_spmm(const bs_matrix* A, const void* X, int64_t N, int64_t ldx, void* Y, int64_t ldy, void* stream) {
  bsk::Geom g;
  int st = matrix_geom(A, &g);
  if (st) return st;
  if (!X || !Y || N < 1 || ldx < g.K || ldy < g.M) return BS_ERR_ARG;
  if (g.layout == BS_LAYOUT_SP24)  // 2:4: sparse tensor cores (tcgen05.mma.sp) or CUDA cores
    return from_cuda(bsk_launch_sp24(g, A->packed, X, N, ldx, Y, ldy, (cudaStream_t)stream, false));
  cudaError_t e = bsk_launch_spmm(g, A->packed, X, N, ldx, Y, ldy, (cudaStream_t)stream);
  if (e != cudaErrorNotSupported) return from_cuda(e);
  // SPMV layout: passes of 8 batch columns through the SpMV kernel (16-bit), or one SpMV per column
  e = bsk_launch_spmv_batch(g, A->packed, X, N, ldx, Y, ldy, (cudaStream_t)stream);
  if (e != cudaErrorNotSupported) return from_cuda(e);
  const size_t es = (size_t)g.es;
  for (int64_t n = 0; n < N; ++n) {
    e = bsk_launch_spmv(g, A->packed, (const char*)X + (size_t)(n * ldx) * es, (char*)Y + (size_t)(n * ldy) * es,
                        BS_SPMV_PDL, (cudaStream_t)stream);
    if (e != cudaSuccess) return from_cuda(e);
  }
  return BS_OK;
}

}  // extern "C"
