// NVLink peer bandwidth, SM-issued: pull (GPU 0 loads from GPU 1, stores locally) vs push
// (GPU 0 loads locally, stores to GPU 1), 16-byte vectors, 8 in flight per thread; and the
// copy engine (cudaMemcpyPeerAsync). nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy16(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) __stcs(dst + i + u * stride, v[u]);
  }
  for (; i < n; i += stride) __stcs(dst + i, __ldcs(src + i));
}

int main() {
  const size_t bytes = 4ull << 30, n = bytes / 16;
  void *a0, *b0, *a1;
  cudaSetDevice(1);
  cudaMalloc(&a1, bytes);
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaMalloc(&a0, bytes);
  cudaMalloc(&b0, bytes);
  cudaSetDevice(1);
  cudaDeviceEnablePeerAccess(0, 0);
  cudaSetDevice(0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int blocksPerSm : {4, 8, 16}) {
    for (int mode = 0; mode < 3; ++mode) {
      float best = 1e9;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) copy16<<<148 * blocksPerSm, 256>>>((uint4*)b0, (const uint4*)a1, n);  // pull
        else if (mode == 1) copy16<<<148 * blocksPerSm, 256>>>((uint4*)a1, (const uint4*)a0, n);  // push
        else cudaMemcpyPeerAsync(a1, 1, a0, 0, bytes);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("%s blocks/SM %2d: %.1f GB/s\n", mode == 0 ? "pull (SM loads) " : mode == 1 ? "push (SM stores)" : "copy engine     ",
             blocksPerSm, bytes / best / 1e6);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
