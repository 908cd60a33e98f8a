// spmv_bf16_batch.cu: bf16 instantiations of the batched SpMV kernel (spmv_impl.cuh): NV = 2, 4, 8, 16
// batch columns per x slot.
#include "spmv_impl.cuh"

cudaError_t bsk_spmv_dispatch_bf16_batch(const bsk::Geom& g, const bsk_spmv::SpmvArgs& a, int nv, cudaStream_t s) {
  switch (nv) {
    case 2: return bsk_spmv::dispatch_is<BS_BF16, 2>(g, a, s);
    case 4: return bsk_spmv::dispatch_is<BS_BF16, 4>(g, a, s);
    case 16: return bsk_spmv::dispatch_is<BS_BF16, 16>(g, a, s);
    default: return bsk_spmv::dispatch_is<BS_BF16, 8>(g, a, s);
  }
}
