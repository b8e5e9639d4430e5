// k_allreduce.cu — fixed-order device-level gradient allreduce over peer
// memory (the reference's CollectiveEngine sum, collectives.cpp:137-154:
// p.sum[i] += contrib[i] in issue order; north star: fixed-order fp32 sums).
//
// One kernel per GPU is the whole collective: GPU `me` owns the slice
// [me, me+1) * nvec / N of the 16-byte vectors. For every vector of its slice
// it loads that vector of EVERY source (the sliced ranks' gradients of every
// GPU, read over NVLink from the peers' CUDA-IPC-mapped arenas), adds them in
// the global key order — u64 mod 2^64, f32 IEEE round-to-nearest, bf16 in f32
// with one final rounding — and stores the result into EVERY GPU's
// destination (NVLink stores). That is a reduce-scatter and an all-gather
// fused into one pass: no intermediate buffer, no second launch, each source
// byte read once, each result byte written once per GPU. The summation order
// never depends on N, on the slicing or on timing, so every GPU holds the same
// bits as a CPU left-to-right sum.
//
// Cross-GPU ordering (use_flags): CTA 0 publishes "my sources are final" into
// flag slot `me` of every peer (st.release.sys; the kernel starts only after
// every earlier op of its stream, so the sources and the destination are
// final/free), and every CTA waits for all N ready flags before its first
// peer load (ld.acquire.sys). The last CTA to finish (threadfence_system +
// counter) publishes "my slice is in every destination" and waits for all N
// done flags, so when the kernel completes this GPU's destination holds the
// whole result and no peer reads its sources any more. Epochs only grow.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "snap_internal.h"

namespace snap {
namespace {

constexpr int kThreads = 256;
constexpr uint32_t kFlag = 16;  // u64 words: one 128-byte line per flag
constexpr int kBatch = 8;       // sources loaded before their adds (loads in flight)

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_flag(const uint64_t* f, uint64_t epoch) {
  const long long t0 = clock64();
  while (ld_acquire_sys(f) < epoch) {
    __nanosleep(128);
    // ~30 s at 2 GHz: a peer never joined this collective — fail loudly
    if (clock64() - t0 > 60000000000ll) __trap();
  }
}

// Accumulator of one 16-byte vector per dtype.
template <int DT>
struct Acc;
template <>
struct Acc<SNAP_U64> {
  unsigned long long v[2];
  __device__ void init(const uint4& x) {
    const ulonglong2 y = reinterpret_cast<const ulonglong2&>(x);
    v[0] = y.x, v[1] = y.y;
  }
  __device__ void add(const uint4& x) {
    const ulonglong2 y = reinterpret_cast<const ulonglong2&>(x);
    v[0] += y.x, v[1] += y.y;
  }
  __device__ uint4 out() const {
    ulonglong2 y{v[0], v[1]};
    return reinterpret_cast<const uint4&>(y);
  }
};
template <>
struct Acc<SNAP_F32> {
  float v[4];
  __device__ void init(const uint4& x) {
    const float4 y = reinterpret_cast<const float4&>(x);
    v[0] = y.x, v[1] = y.y, v[2] = y.z, v[3] = y.w;
  }
  __device__ void add(const uint4& x) {
    const float4 y = reinterpret_cast<const float4&>(x);
    v[0] = __fadd_rn(v[0], y.x), v[1] = __fadd_rn(v[1], y.y);
    v[2] = __fadd_rn(v[2], y.z), v[3] = __fadd_rn(v[3], y.w);
  }
  __device__ uint4 out() const {
    float4 y{v[0], v[1], v[2], v[3]};
    return reinterpret_cast<const uint4&>(y);
  }
};
template <>
struct Acc<SNAP_BF16> {
  float v[8];
  __device__ static float lo(uint32_t w) { return __uint_as_float(w << 16); }
  __device__ static float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
  __device__ void init(const uint4& x) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) v[2 * k] = lo(w[k]), v[2 * k + 1] = hi(w[k]);
  }
  __device__ void add(const uint4& x) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      v[2 * k] = __fadd_rn(v[2 * k], lo(w[k])), v[2 * k + 1] = __fadd_rn(v[2 * k + 1], hi(w[k]));
  }
  __device__ uint4 out() const {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t a = __bfloat16_as_ushort(__float2bfloat16_rn(v[2 * k]));
      const uint32_t b = __bfloat16_as_ushort(__float2bfloat16_rn(v[2 * k + 1]));
      w[k] = a | (b << 16);
    }
    return uint4{w[0], w[1], w[2], w[3]};
  }
};

template <int DT>
__device__ __forceinline__ void scalar_elem(const ArArgs& a, uint64_t i) {
  if constexpr (DT == SNAP_U64) {
    unsigned long long s = reinterpret_cast<const unsigned long long*>(a.src[0])[i];
    for (uint32_t r = 1; r < a.R; ++r) s += reinterpret_cast<const unsigned long long*>(a.src[r])[i];
    for (uint32_t q = 0; q < a.N; ++q) reinterpret_cast<unsigned long long*>(a.dst[q])[i] = s;
  } else if constexpr (DT == SNAP_F32) {
    float s = reinterpret_cast<const float*>(a.src[0])[i];
    for (uint32_t r = 1; r < a.R; ++r) s = __fadd_rn(s, reinterpret_cast<const float*>(a.src[r])[i]);
    for (uint32_t q = 0; q < a.N; ++q) reinterpret_cast<float*>(a.dst[q])[i] = s;
  } else {
    auto f = [](const uint8_t* p, uint64_t i) {
      return __uint_as_float(uint32_t(reinterpret_cast<const uint16_t*>(p)[i]) << 16);
    };
    float s = f(a.src[0], i);
    for (uint32_t r = 1; r < a.R; ++r) s = __fadd_rn(s, f(a.src[r], i));
    const uint16_t o = __bfloat16_as_ushort(__float2bfloat16_rn(s));
    for (uint32_t q = 0; q < a.N; ++q) reinterpret_cast<uint16_t*>(a.dst[q])[i] = o;
  }
}

template <int DT, int U>
__global__ void __launch_bounds__(kThreads)
k_ordered_allreduce(ArArgs a, uint64_t v0, uint64_t v1, uint64_t t0, uint64_t t1) {
  if (a.use_flags) {
    if (blockIdx.x == 0 && threadIdx.x < a.N) {
      __threadfence_system();
      st_release_sys(a.flags[threadIdx.x] + a.me * kFlag, a.epoch);
    }
    if (threadIdx.x == 0)
      for (uint32_t q = 0; q < a.N; ++q) wait_flag(a.myflag + q * kFlag, a.epoch);
    __syncthreads();
  }
  // U vectors per thread and iteration (i, i + stride/U, ...): U x kBatch
  // independent 16-byte loads in flight per thread over NVLink
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  const uint64_t span = v1 - v0, per = (span + U - 1) / U;
  for (uint64_t j = uint64_t(blockIdx.x) * kThreads + threadIdx.x; j < per; j += stride) {
    Acc<DT> acc[U];
    uint4 x[U][kBatch];
    for (uint32_t r0 = 0; r0 < a.R; r0 += kBatch) {
      const uint32_t nb = min(uint32_t(kBatch), a.R - r0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = v0 + j + uint64_t(u) * per;
#pragma unroll
        for (int b = 0; b < kBatch; ++b)
          if (b < int(nb) && i < v1) x[u][b] = __ldcs(reinterpret_cast<const uint4*>(a.src[r0 + b]) + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
          if (b >= int(nb)) break;
          if (r0 + b == 0)
            acc[u].init(x[u][b]);
          else
            acc[u].add(x[u][b]);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = v0 + j + uint64_t(u) * per;
      if (i >= v1) continue;
      const uint4 o = acc[u].out();
      for (uint32_t q = 0; q < a.N; ++q) __stcs(reinterpret_cast<uint4*>(a.dst[q]) + i, o);
    }
  }
  for (uint64_t i = t0 + uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < t1; i += stride)
    scalar_elem<DT>(a, i);
  if (a.use_flags) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned prev = atomicAdd(a.cta_count, 1u);
      if (prev == gridDim.x - 1) {
        *a.cta_count = 0;
        __threadfence_system();
        for (uint32_t q = 0; q < a.N; ++q) st_release_sys(a.flags[q] + (a.N + a.me) * kFlag, a.epoch);
        for (uint32_t q = 0; q < a.N; ++q) wait_flag(a.myflag + (a.N + q) * kFlag, a.epoch);
      }
    }
  }
}

}  // namespace

int launch_ordered_allreduce(const ArArgs& a, cudaStream_t s) {
  const uint64_t esz = a.dtype == SNAP_U64 ? 8 : a.dtype == SNAP_F32 ? 4 : 2;
  const uint64_t per = 16 / esz;
  const uint64_t nvec = a.elems / per;
  const uint64_t v0 = nvec * a.me / a.N, v1 = nvec * (a.me + 1) / a.N;
  const uint64_t t0 = a.me == a.N - 1 ? nvec * per : 0, t1 = a.me == a.N - 1 ? a.elems : 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // tuning knobs (A/B on the box): SNAP_AR_CTAS per SM, SNAP_AR_UNROLL 1 | 2 | 4
  static const int cps = [] {
    const char* e = getenv("SNAP_AR_CTAS");
    return e && atoi(e) > 0 ? atoi(e) : 4;
  }();
  static const int unroll = [] {
    const char* e = getenv("SNAP_AR_UNROLL");
    const int v = e ? atoi(e) : 1;
    return v == 2 || v == 4 ? v : 1;
  }();
  uint64_t blocks = (v1 - v0 + uint64_t(kThreads) * unroll - 1) / (uint64_t(kThreads) * unroll);
  blocks = std::max<uint64_t>(1, std::min<uint64_t>(blocks, uint64_t(sms) * cps));
#define SNAP_AR_LAUNCH(DT)                                                                       \
  do {                                                                                          \
    if (unroll == 4)                                                                            \
      k_ordered_allreduce<DT, 4><<<unsigned(blocks), kThreads, 0, s>>>(a, v0, v1, t0, t1);      \
    else if (unroll == 2)                                                                       \
      k_ordered_allreduce<DT, 2><<<unsigned(blocks), kThreads, 0, s>>>(a, v0, v1, t0, t1);      \
    else                                                                                        \
      k_ordered_allreduce<DT, 1><<<unsigned(blocks), kThreads, 0, s>>>(a, v0, v1, t0, t1);      \
  } while (0)
  switch (a.dtype) {
    case SNAP_U64: SNAP_AR_LAUNCH(SNAP_U64); break;
    case SNAP_F32: SNAP_AR_LAUNCH(SNAP_F32); break;
    default: SNAP_AR_LAUNCH(SNAP_BF16); break;
  }
#undef SNAP_AR_LAUNCH
  return 1;
}

}  // namespace snap
