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

// A warp per (output pixel, tap): the pixel/tap decomposition (32-bit divisions) once per warp, then the
// lanes copy the tap's C-run of units (16-byte vectors or elements) with coalesced loads and stores. Round 1's
// kernel above did six 64-bit divisions per 16-byte unit and was ALU-bound (conv3_3: 10.5 us for 14.5 MB).
template <typename T>
__global__ void __launch_bounds__(256) im2col_warp_kernel(const T* __restrict__ in, uint32_t H, uint32_t W, uint32_t Cu,
                                                          uint32_t kh, uint32_t kw, int pad, int stride, uint32_t OH,
                                                          uint32_t OW, uint32_t npairs, T* __restrict__ X, int64_t ldx) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t taps = kh * kw, ohw = OH * OW;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < npairs; q += nw) {
    const uint32_t p = q / taps, tap = q - p * taps;
    const uint32_t img = p / ohw, pix = p - img * ohw;
    const uint32_t oy = pix / OW, ox = pix - oy * OW;
    const uint32_t dy = tap / kw, dx = tap - dy * kw;
    const int iy = (int)(oy * stride + dy) - pad, ix = (int)(ox * stride + dx) - pad;
    const bool valid = iy >= 0 && iy < (int)H && ix >= 0 && ix < (int)W;
    const T* src = in + (((int64_t)img * H + (valid ? iy : 0)) * W + (valid ? ix : 0)) * Cu;
    T* dst = X + (int64_t)p * ldx + (int64_t)tap * Cu;
    for (uint32_t c = lane; c < Cu; c += 32) {
      T v;
      if (valid) v = __ldg(src + c);
      else memset(&v, 0, sizeof(T));
      dst[c] = v;
    }
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
  const int64_t npairs = npix * kh * kw;
  if (npairs < (1LL << 31) && H < (1LL << 31) && W < (1LL << 31)) {  // warp per (pixel, tap), 32-bit index math
    int64_t g2 = (npairs + 7) / 8;
    if (g2 > cap) g2 = cap;
    if (g2 < 1) g2 = 1;
    if (vec)
      im2col_warp_kernel<uint4><<<(unsigned)g2, 256, 0, s>>>((const uint4*)in, (uint32_t)H, (uint32_t)W, (uint32_t)(C / per),
                                                              kh, kw, pad, stride, (uint32_t)OH, (uint32_t)OW,
                                                              (uint32_t)npairs, (uint4*)X, ldx / per);
    else if (es == 2)
      im2col_warp_kernel<uint16_t><<<(unsigned)g2, 256, 0, s>>>((const uint16_t*)in, (uint32_t)H, (uint32_t)W, (uint32_t)C,
                                                                 kh, kw, pad, stride, (uint32_t)OH, (uint32_t)OW,
                                                                 (uint32_t)npairs, (uint16_t*)X, ldx);
    else
      im2col_warp_kernel<uint32_t><<<(unsigned)g2, 256, 0, s>>>((const uint32_t*)in, (uint32_t)H, (uint32_t)W, (uint32_t)C,
                                                                 kh, kw, pad, stride, (uint32_t)OH, (uint32_t)OW,
                                                                 (uint32_t)npairs, (uint32_t*)X, ldx);
    return cudaGetLastError();
  }
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
