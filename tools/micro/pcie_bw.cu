// H2D, D2H and concurrent bidirectional PCIe bandwidth with pinned host memory.
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t n = 1ull << 30;
  void *h1, *h2, *d1, *d2;
  cudaHostAlloc(&h1, n, cudaHostAllocPortable);
  cudaHostAlloc(&h2, n, cudaHostAllocPortable);
  cudaMalloc(&d1, n);
  cudaMalloc(&d2, n);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int pass = 0; pass < 2; ++pass) {
    float ms;
    cudaEventRecord(e0, a);
    cudaMemcpyAsync(d1, h1, n, cudaMemcpyHostToDevice, a);
    cudaEventRecord(e1, a); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("H2D %.1f GB/s\n", n / ms / 1e6);
    cudaEventRecord(e0, a);
    cudaMemcpyAsync(h2, d2, n, cudaMemcpyDeviceToHost, a);
    cudaEventRecord(e1, a); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("D2H %.1f GB/s\n", n / ms / 1e6);
    cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    cudaStreamWaitEvent(a, e0, 0); cudaStreamWaitEvent(b, e0, 0);
    cudaMemcpyAsync(d1, h1, n, cudaMemcpyHostToDevice, a);
    cudaMemcpyAsync(h2, d2, n, cudaMemcpyDeviceToHost, b);
    cudaDeviceSynchronize();
    cudaEventRecord(e1, 0); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("bidir %.1f GB/s total (%.1f per direction)\n", 2 * n / ms / 1e6, n / ms / 1e6);
    // chunked (64 MiB) alternating streams
    cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    cudaStreamWaitEvent(a, e0, 0); cudaStreamWaitEvent(b, e0, 0);
    const size_t s = 64ull << 20;
    for (size_t o = 0; o < n; o += s) {
      cudaMemcpyAsync((char*)d1 + o, (char*)h1 + o, s, cudaMemcpyHostToDevice, a);
      cudaMemcpyAsync((char*)h2 + o, (char*)d2 + o, s, cudaMemcpyDeviceToHost, b);
    }
    cudaDeviceSynchronize();
    cudaEventRecord(e1, 0); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("bidir 64MiB slabs %.1f GB/s total\n", 2 * n / ms / 1e6);
  }
  return 0;
}
