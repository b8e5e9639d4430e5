// Copy micro (dev tool): the fused K1's per-warp pattern (32 pages x 256 B per step, loaded
// to registers, lane stores) with the warp's 32 pages at different strides: 4 KiB (consecutive
// pages, the kernel's layout), 64 KiB (one page of each of 32 chunks), 2 MiB.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int STRIDE_PAGES>
__global__ void __launch_bounds__(512, 1) k(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                           size_t npages) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t gw = size_t(blockIdx.x) * 16 + warp, nw = size_t(gridDim.x) * 16;
  const size_t ntasks = npages / 32;
  const uint32_t u = lane & 15, q = lane >> 4;
  for (size_t t = gw; t < ntasks; t += nw) {
    // task t: pages p(t, j) = base + j * STRIDE for j < 32, tasks tile the page space
    const size_t group = t / STRIDE_PAGES, off = t % STRIDE_PAGES;
    const size_t base = group * 32 * STRIDE_PAGES + off;
    for (int s = 0; s < 16; ++s) {
      uint4 v[16];
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const size_t page = base + size_t(kk * 2 + q) * STRIDE_PAGES;
        v[kk] = __ldcs(src + page * 256 + s * 16 + u);
      }
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const size_t page = base + size_t(kk * 2 + q) * STRIDE_PAGES;
        __stcs(dst + page * 256 + s * 16 + u, v[kk]);
      }
    }
  }
}

int main() {
  const size_t n = 2ull << 30, npages = n / 4096;
  uint4 *a, *b;
  cudaMalloc(&a, n);
  cudaMalloc(&b, n);
  cudaMemset(a, 1, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name) {
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      kern<<<148, 512>>>(a, b, npages);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    printf("%-26s %7.3f ms  %7.1f GB/s (R+W)  %s\n", name, best, 2.0 * n / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int i = 0; i < 2; ++i) {
    run(k<1>, "stride 4 KiB (consecutive)");
    run(k<16>, "stride 64 KiB");
    run(k<512>, "stride 2 MiB");
    run(k<3>, "stride 12 KiB");
  }
  return 0;
}
