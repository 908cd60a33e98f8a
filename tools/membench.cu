// membench.cu: HBM read-pattern microbenchmark for the SpMV streaming design (tools only, not product).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench tools/membench.cu && ./membench
//
// Patterns (each reads ~1.2 GB once per iteration, CUDA-event timed, best of 5):
//   seq     : grid-stride, warp w reads 512-byte chunk w, w+NW, ... (copy-like locality)
//   warp1   : each warp owns a contiguous region; 512 B per step; U steps in flight (rolling)
//   warp2   : as warp1 plus a second region of 256 B per step (values + indices, as the SPMV layout)
//   bulk    : each warp's lane 0 issues cp.async.bulk copies of CH bytes into a per-warp smem ring
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ldg_na(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_na8(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

__global__ void seq_kernel(const uint8_t* base, int64_t bytes, uint32_t* sink) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint32_t acc = 0;
  const int64_t chunks = bytes / 512;
#pragma unroll 4
  for (int64_t c = w; c < chunks; c += nw) {
    uint4 v = ldg_na(base + c * 512 + lane * 16);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) sink[0] = acc;
}

template <int U, bool TWO>
__global__ void warp_kernel(const uint8_t* base, const uint8_t* base2, int64_t per_warp_steps, uint32_t* sink) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint8_t* p = base + w * per_warp_steps * 512 + lane * 16;
  const uint8_t* q = base2 + w * per_warp_steps * 256 + lane * 8;
  uint4 buf[U];
  uint2 buf2[U];
  uint32_t acc = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    buf[u] = ldg_na(p + u * 512);
    if (TWO) buf2[u] = ldg_na8(q + u * 256);
  }
  for (int64_t j0 = 0; j0 < per_warp_steps; j0 += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc ^= buf[u].x ^ buf[u].y ^ buf[u].z ^ buf[u].w;
      if (TWO) acc += buf2[u].x ^ buf2[u].y;
      const int64_t j = j0 + u + U;
      if (j < per_warp_steps) {
        buf[u] = ldg_na(p + j * 512);
        if (TWO) buf2[u] = ldg_na8(q + j * 256);
      }
    }
  }
  if (acc == 0x12345678) sink[0] = acc;
}

// bulk: per warp, NS stages of CH bytes in smem; lane 0 issues cp.async.bulk, all lanes consume.
template <int NS>
__global__ void bulk_kernel(const uint8_t* base, int64_t per_warp_bytes, int CH, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  uint8_t* ring = sm + (size_t)wid * NS * CH;
  __shared__ __align__(8) uint64_t bar[32][NS];
  if (lane == 0)
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[wid][s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const uint8_t* src = base + w * per_warp_bytes;
  const int64_t nch = per_warp_bytes / CH;
  auto issue = [&](int64_t c) {
    const int s = (int)(c % NS);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[wid][s]);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(ring + (size_t)s * CH);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CH));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                 "l"(src + c * CH), "r"(CH), "r"(b) : "memory");
  };
  if (lane == 0)
    for (int64_t c = 0; c < NS && c < nch; ++c) issue(c);
  uint32_t acc = 0;
  for (int64_t c = 0; c < nch; ++c) {
    const int s = (int)(c % NS);
    const uint32_t phase = (uint32_t)((c / NS) & 1);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[wid][s]);
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(b), "r"(phase));
    }
    const uint4* r = (const uint4*)(ring + (size_t)s * CH);
    for (int i = lane; i < CH / 16; i += 32) { uint4 v = r[i]; acc ^= v.x ^ v.w; }
    __syncwarp();
    if (lane == 0 && c + NS < nch) issue(c + NS);
  }
  if (acc == 0x12345678) sink[0] = acc;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int it = 0; it < 6; ++it) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it > 0 && ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t total = 1207959552LL;  // 1.2 GB (the 65536^2 @ 90% packed size)
  uint8_t* buf;
  uint32_t* sink;
  CK(cudaMalloc(&buf, total + (1 << 26)));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(buf, 1, total + (1 << 26)));
  printf("{\"sms\": %d}\n", sms);
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    float ms = timeit([&] { seq_kernel<<<blocks, tpb>>>(buf, total, sink); });
    printf("{\"pattern\": \"seq\", \"tpb\": %d, \"blocks\": %d, \"GBps\": %.1f}\n", tpb, blocks, total / ms / 1e6);
  }
  // warp-owned contiguous regions
  for (int wps : {8, 16, 32, 48, 64}) {
    const int tpb = 512;
    const int blocks = sms * wps / 16;
    const int64_t nw = (int64_t)blocks * 16;
    for (int two = 0; two < 2; ++two) {
      const int64_t stepb = two ? 768 : 512;
      const int64_t steps = total / nw / stepb;
      const uint8_t* b2 = buf + steps * nw * 512;
      auto run = [&](int U) {
        float ms = 0;
        if (two) {
          if (U == 2) ms = timeit([&] { warp_kernel<2, true><<<blocks, tpb>>>(buf, b2, steps, sink); });
          if (U == 4) ms = timeit([&] { warp_kernel<4, true><<<blocks, tpb>>>(buf, b2, steps, sink); });
          if (U == 8) ms = timeit([&] { warp_kernel<8, true><<<blocks, tpb>>>(buf, b2, steps, sink); });
        } else {
          if (U == 2) ms = timeit([&] { warp_kernel<2, false><<<blocks, tpb>>>(buf, b2, steps, sink); });
          if (U == 4) ms = timeit([&] { warp_kernel<4, false><<<blocks, tpb>>>(buf, b2, steps, sink); });
          if (U == 8) ms = timeit([&] { warp_kernel<8, false><<<blocks, tpb>>>(buf, b2, steps, sink); });
        }
        printf("{\"pattern\": \"warp%d\", \"warps_per_sm\": %d, \"U\": %d, \"inflight_KB_per_sm\": %.0f, \"GBps\": %.1f}\n",
               two ? 2 : 1, wps, U, wps * U * stepb / 1024.0, steps * nw * stepb / ms / 1e6);
      };
      for (int U : {2, 4, 8}) run(U);
    }
  }
  // bulk copies: per-warp rings
  for (int wps : {4, 8, 16}) {
    for (int CH : {2048, 4096, 8192}) {
      for (int ns : {2, 4}) {
        const int tpb = 32 * wps;
        const size_t smem = (size_t)wps * ns * CH;
        if (smem > 200 * 1024) continue;
        const int blocks = sms;
        const int64_t nw = (int64_t)blocks * wps;
        const int64_t per = total / nw / CH * CH;
        float ms;
        if (ns == 2) {
          cudaFuncSetAttribute(bulk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
          ms = timeit([&] { bulk_kernel<2><<<blocks, tpb, smem>>>(buf, per, CH, sink); });
        } else {
          cudaFuncSetAttribute(bulk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
          ms = timeit([&] { bulk_kernel<4><<<blocks, tpb, smem>>>(buf, per, CH, sink); });
        }
        CK(cudaGetLastError());
        printf("{\"pattern\": \"bulk\", \"warps_per_sm\": %d, \"chunk\": %d, \"stages\": %d, \"inflight_KB_per_sm\": %zu, \"GBps\": %.1f}\n",
               wps, CH, ns, smem / 1024, per * nw / ms / 1e6);
      }
    }
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
