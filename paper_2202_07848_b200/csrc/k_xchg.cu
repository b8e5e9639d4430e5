// k_xchg.cu — the cross-GPU barrier that completes the digest exchange fused
// into K1 (the one exchange step of the multi-rank snapshot).
//
// K1 has already stored every chunk digest into each rank's gathered vector
// over NVLink (CUDA-IPC-mapped windows) and fenced at system scope. Thread q
// then publishes "my digests are in place" into flag slot `rank` of rank q's
// window (st.release.sys) and waits until rank q has published the same epoch
// into this rank's window (ld.acquire.sys): after that, every peer's stores
// into this rank's vector are visible to the selection kernels that follow on
// the stream. Epochs only grow, so flags never need resetting.
#include <cuda_runtime.h>

#include "snap_internal.h"

namespace snap {
namespace {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

constexpr uint32_t kFlagStride = 16;  // u64 words: one 128-byte line per flag

__global__ void k_peer_barrier(uint64_t* const* __restrict__ xflag, const uint64_t* myflag,
                               uint32_t rank, uint32_t n, uint64_t epoch) {
  const uint32_t q = threadIdx.x;
  if (q >= n) return;
  __threadfence_system();
  st_release_sys(xflag[q] + rank * kFlagStride, epoch);
  const uint64_t* f = myflag + q * kFlagStride;
  const long long t0 = clock64();
  while (ld_acquire_sys(f) < epoch) {
    __nanosleep(256);
    // ~30 s at 2 GHz: a peer never reached its barrier (it failed or is not
    // running the same collective sequence) — fail loudly instead of hanging
    if (clock64() - t0 > 60000000000ll) __trap();
  }
}

}  // namespace

int launch_peer_barrier(uint64_t* const* xflag, const uint64_t* myflag, uint32_t rank, uint32_t n,
                        uint64_t epoch, cudaStream_t s) {
  if (n == 0) return 0;
  k_peer_barrier<<<1, 32 * ((n + 31) / 32), 0, s>>>(xflag, myflag, rank, n, epoch);
  return 1;
}

}  // namespace snap
