// conv.cu: im2col for convolution layers run as balanced-sparse SpMM.
//
// The paper runs VGG-16's convolutions "using im2col that converts convolution operation to
// matrix-matrix multiplication", with "the weights of all kernels in one convolution layer ...
// considered as one weight matrix". Here activations are NHWC (channels last) and the weight
// matrix is Cout × (kh·kw·C) with columns in (dy, dx, c) order (reading A23), so the product
// Y = W_bs · X^T of bs_spmm with X = im2col(in) is the NHWC output [pixels][Cout] directly and the next
// layer's im2col reads it without a transpose.
//
// bs_im2col writes X [Nimg·OH·OW][kh·kw·C]: row p = output pixel, kh·kw runs of C channels, each run a
// contiguous copy of one input pixel (or zeros past the border). One thread moves one 16-byte vector
// (8 channels of 16-bit data, 4 of fp32) when C allows it, so reads and writes are coalesced runs.
#include "bs_common.cuh"

namespace {

template <typename T>
__global__ void __launch_bounds__(256) im2col_kernel(const T* __restrict__ in, int64_t H, int64_t W, int64_t C,
                                                     int kh, int kw, int pad, int stride, int64_t OH, int64_t OW,
                                                     int64_t npix, T* __restrict__ X, int64_t ldx) {
  // T is the unit moved per thread: uint4 (16 bytes) or one element; C counts units here
  const int64_t taps = (int64_t)kh * kw;
  const int64_t per_pix = taps * C;
  const int64_t n = npix * per_pix;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / per_pix, rem = i - p * per_pix;
    const int64_t tap = rem / C, c = rem - tap * C;
    const int64_t img = p / (OH * OW), pix = p - img * (OH * OW);
    const int64_t oy = pix / OW, ox = pix - oy * OW;
    const int64_t dy = tap / kw, dx = tap - dy * kw;
    const int64_t iy = oy * stride + dy - pad, ix = ox * stride + dx - pad;
    T v;
    if (iy < 0 || iy >= H || ix < 0 || ix >= W) {
      memset(&v, 0, sizeof(T));
    } else {
      v = __ldg(in + ((img * H + iy) * W + ix) * C + c);
    }
    X[p * ldx + tap * C + c] = v;
  }
}

}  // namespace

cudaError_t bsk_launch_im2col(const void* in, int dt, int64_t Nimg, int64_t H, int64_t W, int64_t C, int kh, int kw,
                              int pad, int stride, void* X, int64_t ldx, cudaStream_t s) {
  const int64_t OH = (H + 2 * pad - kh) / stride + 1, OW = (W + 2 * pad - kw) / stride + 1;
  const int64_t npix = Nimg * OH * OW;
  const int es = bsk::dtype_bytes(dt);
  const int64_t per = 16 / es;  // elements per 16-byte unit
  const bool vec = C % per == 0 && ldx % per == 0 && ((uintptr_t)in & 15) == 0 && ((uintptr_t)X & 15) == 0;
  const int64_t units = vec ? npix * kh * kw * (C / per) : npix * kh * kw * C;
  int64_t grid = (units + 255) / 256;
  const int64_t cap = (int64_t)bsk::dev_props().sms * 16;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  if (vec) {
    im2col_kernel<uint4><<<(unsigned)grid, 256, 0, s>>>((const uint4*)in, H, W, C / per, kh, kw, pad, stride, OH, OW,
                                                        npix, (uint4*)X, ldx / per);
  } else if (es == 2) {
    im2col_kernel<uint16_t><<<(unsigned)grid, 256, 0, s>>>((const uint16_t*)in, H, W, C, kh, kw, pad, stride, OH, OW,
                                                           npix, (uint16_t*)X, ldx);
  } else {
    im2col_kernel<uint32_t><<<(unsigned)grid, 256, 0, s>>>((const uint32_t*)in, H, W, C, kh, kw, pad, stride, OH, OW,
                                                           npix, (uint32_t*)X, ldx);
  }
  return cudaGetLastError();
}
