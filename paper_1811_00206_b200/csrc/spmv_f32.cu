// spmv_f32.cu: f32 instantiations of the SpMV kernel (spmv_impl.cuh).
#include "spmv_impl.cuh"

cudaError_t bsk_spmv_dispatch_f32(const bsk::Geom& g, const bsk_spmv::SpmvArgs& a, cudaStream_t s) {
  return bsk_spmv::dispatch_is<BS_F32, 1>(g, a, s);
}
