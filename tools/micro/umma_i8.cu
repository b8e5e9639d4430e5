// tcgen05.mma kind::i8 (M=128, K=32, A in TMEM or SMEM, B in SMEM) issue/latency probe:
// cycles for R MMAs issued back to back by one thread and completed through one commit,
// for N in {16, 32, 64, 128, 256} and 1 or 4 destination accumulators.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3fff) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

template <int N, int NACC, bool TS, int R, int M = 128>
__global__ void k(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(s)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tslot;
  const uint32_t id = (2u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint32_t bb = smem_u32(s), ab = smem_u32(s + 32768);
    long long best = 1ll << 60;
    for (int rep = 0; rep < 4; ++rep) {
      const long long t0 = clock64();
#pragma unroll 1
      for (int r = 0; r < R; ++r) {
        const uint32_t d = t + 256 + (r % NACC) * (N > 64 ? 0 : N);
        if (TS) mma_ts(d, t + (r % 8) * 8, desc(bb + (r & 3) * 32), id, r >= NACC);
        else mma_ss(d, desc(ab + (r & 3) * 32), desc(bb + (r & 3) * 32), id, r >= NACC);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)), "r"(rep & 1));
      const long long dt = clock64() - t0;
      best = dt < best ? dt : best;
    }
    out[0] = best;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int N, int NACC, bool TS, int R, int M = 128>
void run(long long* d) {
  cudaFuncSetAttribute(k<N, NACC, TS, R, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  k<N, NACC, TS, R, M><<<1, 128, 66 * 1024>>>(d);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("M=%d %s N=%3d acc=%d R=%3d: %7lld cycles, %6.1f per MMA  (%s)\n", M, TS ? "TS" : "SS", N, NACC, R, h,
         double(h) / R, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<16, 1, true, 256>(d);
  run<16, 1, true, 256, 64>(d);
  run<64, 1, true, 256, 64>(d);
  run<256, 1, true, 256, 64>(d);
  run<16, 1, false, 256, 64>(d);
  run<256, 1, false, 256, 64>(d);
  run<256, 1, false, 256>(d);
  return 0;
}
