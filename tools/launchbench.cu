// launchbench.cu: fixed per-launch costs on B200 (tools only). Graph of 200 back-to-back launches of
// an (almost) empty persistent kernel; per-launch time for several smem sizes / prologues.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/launchbench tools/launchbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void empty_kernel(int* p) {
  extern __shared__ uint8_t sm[];
  if (threadIdx.x == 0 && p && blockIdx.x == 100000) p[0] = sm[0];
}

__global__ void mbar_kernel(int* p) {
  extern __shared__ uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[16][4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    for (int s = 0; s < 4; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[w][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && p && blockIdx.x == 100000) p[0] = sm[0];
}

// one DRAM round trip per CTA (lane 0 of each warp loads 4 bytes of a cold buffer)
__global__ void dram_kernel(const int* src, int* p, int64_t stride) {
  if ((threadIdx.x & 31) == 0) {
    int v = __ldcg(src + (blockIdx.x * 16 + (threadIdx.x >> 5)) * stride);
    if (v == 0x12345) p[0] = v;
  }
}

template <typename L>
float graph_time(L launch, int n) {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) launch(s, i);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best * 1000.f / n;
}

int main() {
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(mbar_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  int* buf;
  cudaMalloc(&buf, 1 << 30);
  for (int smem : {0, 64 * 1024, 128 * 1024, 200 * 1024, 227 * 1024}) {
    for (int tpb : {128, 512, 1024}) {
      float us = graph_time([&](cudaStream_t s, int) { empty_kernel<<<148, tpb, smem, s>>>(nullptr); }, 200);
      printf("{\"kernel\": \"empty\", \"grid\": 148, \"tpb\": %d, \"smem_KB\": %d, \"us\": %.3f}\n", tpb, smem / 1024, us);
    }
  }
  float us = graph_time([&](cudaStream_t s, int) { mbar_kernel<<<148, 512, 200 * 1024, s>>>(nullptr); }, 200);
  printf("{\"kernel\": \"mbar_init+fence\", \"tpb\": 512, \"smem_KB\": 200, \"us\": %.3f}\n", us);
  // one dependent DRAM round trip per warp, different cold lines each launch
  us = graph_time([&](cudaStream_t s, int i) { dram_kernel<<<148, 512, 0, s>>>(buf + (i % 64) * 4096 * 1024, buf, 64); }, 200);
  printf("{\"kernel\": \"one_dram_roundtrip\", \"tpb\": 512, \"us\": %.3f}\n", us);
  cudaDeviceSynchronize();
  return 0;
}
