// Contiguous 2 GiB device copy through three engines: LDG/STG (16 B per lane, streaming),
// TMA bulk (cp.async.bulk global->smem->global, 4-stage ring of 32 KiB per CTA), and
// cudaMemcpyAsync D2D. GB/s counts read + write bytes.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_ldst(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n16) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) if (i + k * size_t(gridDim.x) * blockDim.x < n16) v[k] = __ldcs(s + i + k * size_t(gridDim.x) * blockDim.x);
#pragma unroll
    for (int k = 0; k < 4; ++k) if (i + k * size_t(gridDim.x) * blockDim.x < n16) __stcs(d + i + k * size_t(gridDim.x) * blockDim.x, v[k]);
  }
}

__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int ST, int PIECE>
__global__ void __launch_bounds__(32) k_tma(const uint8_t* __restrict__ s, uint8_t* __restrict__ d, size_t n) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[ST];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < ST; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const size_t npieces = n / PIECE;
  size_t p0 = blockIdx.x;
  const size_t stride = gridDim.x;
  // issue ST loads
  int issued = 0;
  size_t p = p0;
  uint32_t phase[ST] = {};
  for (int k = 0; k < ST && p < npieces; ++k, p += stride, ++issued) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[k])), "r"(PIECE));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su(sm + k * PIECE)), "l"(s + p * PIECE), "r"(PIECE), "r"(su(&bar[k])) : "memory");
  }
  size_t q = p0;
  for (int k = 0; q < npieces; q += stride, k = (k + 1) % ST) {
    asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}"
                 ::"r"(su(&bar[k])), "r"(phase[k]) : "memory");
    phase[k] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + q * PIECE), "r"(su(sm + k * PIECE)), "r"(PIECE) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (p < npieces) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // slot k's store read done
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[k])), "r"(PIECE));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su(sm + k * PIECE)), "l"(s + p * PIECE), "r"(PIECE), "r"(su(&bar[k])) : "memory");
      p += stride;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t n = 2ull << 30;
  uint8_t *a, *b;
  cudaMalloc(&a, n);
  cudaMalloc(&b, n);
  cudaMemset(a, 1, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](auto f, const char* name) {
    f();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%-36s %7.3f ms %7.1f GB/s (R+W)  %s\n", name, ms, 2.0 * n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  time([&] { k_ldst<<<148 * 4, 512>>>((const uint4*)a, (uint4*)b, n / 16); }, "LDG/STG 148x4 CTAs x 512");
  time([&] { k_ldst<<<148 * 2, 512>>>((const uint4*)a, (uint4*)b, n / 16); }, "LDG/STG 148x2 CTAs x 512");
  cudaFuncSetAttribute(k_tma<4, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
  cudaFuncSetAttribute(k_tma<6, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
  cudaFuncSetAttribute(k_tma<4, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384);
  time([&] { k_tma<4, 32768><<<148, 32, 4 * 32768>>>(a, b, n); }, "TMA bulk 148 CTAs, 4 x 32 KiB");
  time([&] { k_tma<6, 32768><<<148, 32, 6 * 32768>>>(a, b, n); }, "TMA bulk 148 CTAs, 6 x 32 KiB");
  time([&] { k_tma<4, 16384><<<296, 32, 4 * 16384>>>(a, b, n); }, "TMA bulk 296 CTAs, 4 x 16 KiB");
  time([&] { cudaMemcpyAsync(b, a, n, cudaMemcpyDeviceToDevice); }, "cudaMemcpyAsync D2D");
  return 0;
}
