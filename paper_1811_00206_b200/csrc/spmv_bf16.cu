// spmv_bf16.cu: bf16 instantiations of the SpMV kernel (spmv_impl.cuh).
#define BS_TRACE_TU_BF16

#include "spmv_impl.cuh"

cudaError_t bsk_spmv_dispatch_bf16_batch(const bsk::Geom& g, const bsk_spmv::SpmvArgs& a, int nv, cudaStream_t s);

cudaError_t bsk_spmv_dispatch_bf16(const bsk::Geom& g, const bsk_spmv::SpmvArgs& a, int nv, cudaStream_t s) {
  if (nv > 1) return bsk_spmv_dispatch_bf16_batch(g, a, nv, s);
  return bsk_spmv::dispatch_is<BS_BF16, 1>(g, a, s);
}
