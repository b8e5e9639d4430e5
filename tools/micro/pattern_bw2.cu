// Copy 2 GiB where each warp owns 32 pages of PAGE bytes and moves SEG bytes of every
// page per step (reads and writes follow the same pattern).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int PAGE, int SEG>
__global__ void __launch_bounds__(512) k(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                         size_t nbytes) {
  constexpr int LPP = SEG / 16;          // lanes per page per instruction
  constexpr int PPI = 32 / LPP;          // pages per instruction
  constexpr int NI = 32 / PPI;           // instructions per step (32 pages)
  const int lane = threadIdx.x & 31;
  const size_t gw = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = (size_t(gridDim.x) * blockDim.x) >> 5;
  const size_t ntasks = nbytes / (32ull * PAGE);
  for (size_t t = gw; t < ntasks; t += nw) {
    const size_t base = t * 32ull * PAGE / 16;
    for (int s = 0; s < PAGE / SEG; ++s) {
      uint4 v[NI];
#pragma unroll
      for (int kk = 0; kk < NI; ++kk)
        v[kk] = __ldcs(src + base + size_t(kk * PPI + lane / LPP) * (PAGE / 16) + s * LPP + lane % LPP);
#pragma unroll
      for (int kk = 0; kk < NI; ++kk)
        __stcs(dst + base + size_t(kk * PPI + lane / LPP) * (PAGE / 16) + s * LPP + lane % LPP, v[kk]);
    }
  }
}

int main() {
  const size_t n = 2ull << 30;
  uint4 *a, *b;
  cudaMalloc(&a, n); cudaMalloc(&b, n);
  cudaMemset(a, 1, n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name) {
    kern<<<148, 512>>>(a, b, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<148, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-24s %7.3f ms  %7.1f GB/s (R+W)\n", name, ms, 2.0 * n / ms / 1e6);
  };
  run(k<4096, 128>, "page 4K seg 128");
  run(k<4096, 256>, "page 4K seg 256");
  run(k<4096, 512>, "page 4K seg 512");
  run(k<2048, 128>, "page 2K seg 128");
  run(k<1024, 128>, "page 1K seg 128");
  run(k<512, 128>, "page 512 seg 128");
  run(k<65536, 128>, "page 64K seg 128");
  run(k<65536, 512>, "page 64K seg 512");
  return 0;
}
