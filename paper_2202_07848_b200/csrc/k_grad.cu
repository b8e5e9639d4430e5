// k_grad.cu — K5: spliced-replica gradient reduction.
//
// Time-sliced DP ranks sharing one GPU contribute their gradients locally
// before the one device-level allreduce (reference: CollectiveEngine::issue
// sums every member's contribution, collectives.cpp:137-144; the local
// accumulation of a sliced rank is charged as a D2D stream op,
// worker.cpp:290-297; only the local closer triggers the cross-GPU op,
// collectives.cpp:147-154).
//
// dst[i] = s_0[i] + s_1[i] + ... in ascending (dp) order; u64 wraps mod 2^64
// (the reference's arithmetic), f32 adds left to right with IEEE
// round-to-nearest (no FMA contraction is possible for a pure add chain), so
// the result is identical to the CPU fixed-order sum; bf16 (C5's gradients)
// adds the same chain in f32 and rounds once to bf16 (RN-even). One pass reads every
// source once and writes dst once: HBM-bound, 16-byte vector accesses.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "snap_internal.h"

namespace snap {
namespace {

constexpr int kMaxSrc = 16;
struct Srcs {
  const uint8_t* p[kMaxSrc];
};

template <typename T>
__device__ __forceinline__ void add4(uint4& a, const uint4& b);
template <>
__device__ __forceinline__ void add4<uint64_t>(uint4& a, const uint4& b) {
  ulonglong2& x = reinterpret_cast<ulonglong2&>(a);
  const ulonglong2& y = reinterpret_cast<const ulonglong2&>(b);
  x.x += y.x;
  x.y += y.y;
}
template <>
__device__ __forceinline__ void add4<float>(uint4& a, const uint4& b) {
  float4& x = reinterpret_cast<float4&>(a);
  const float4& y = reinterpret_cast<const float4&>(b);
  x.x = __fadd_rn(x.x, y.x);
  x.y = __fadd_rn(x.y, y.y);
  x.z = __fadd_rn(x.z, y.z);
  x.w = __fadd_rn(x.w, y.w);
}

template <typename T>
__global__ void __launch_bounds__(256)
k_grad_sum(Srcs srcs, uint32_t nsrc, uint8_t* __restrict__ dst, uint64_t n16, int accumulate) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint4* d = reinterpret_cast<uint4*>(dst);
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
    uint4 acc;
    uint32_t r = 0;
    if (accumulate) {
      acc = d[i];
    } else {
      acc = __ldcs(reinterpret_cast<const uint4*>(srcs.p[0]) + i);
      r = 1;
    }
    for (; r < nsrc; ++r) add4<T>(acc, __ldcs(reinterpret_cast<const uint4*>(srcs.p[r]) + i));
    d[i] = acc;
  }
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t bf_pack(float a, float b) {
  return uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(a))) |
         (uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(b))) << 16);
}

__global__ void __launch_bounds__(256)
k_grad_sum_bf16(Srcs srcs, uint32_t nsrc, uint8_t* __restrict__ dst, uint64_t n16, int accumulate) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint4* d = reinterpret_cast<uint4*>(dst);
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
    float acc[8];
    uint32_t r = 0;
    uint4 x = accumulate ? d[i] : __ldcs(reinterpret_cast<const uint4*>(srcs.p[0]) + i);
    r = accumulate ? 0 : 1;
    const uint32_t w0[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[2 * k] = bf_lo(w0[k]), acc[2 * k + 1] = bf_hi(w0[k]);
    for (; r < nsrc; ++r) {
      const uint4 y = __ldcs(reinterpret_cast<const uint4*>(srcs.p[r]) + i);
      const uint32_t w[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        acc[2 * k] = __fadd_rn(acc[2 * k], bf_lo(w[k])),
        acc[2 * k + 1] = __fadd_rn(acc[2 * k + 1], bf_hi(w[k]));
    }
    d[i] = uint4{bf_pack(acc[0], acc[1]), bf_pack(acc[2], acc[3]), bf_pack(acc[4], acc[5]),
                 bf_pack(acc[6], acc[7])};
  }
}

__global__ void k_grad_sum_tail_bf16(Srcs srcs, uint32_t nsrc, uint8_t* dst, uint64_t first,
                                     uint64_t n, int accumulate) {
  const uint64_t i = first + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint16_t* d = reinterpret_cast<uint16_t*>(dst);
  auto f = [&](const uint8_t* p) {
    return __uint_as_float(uint32_t(reinterpret_cast<const uint16_t*>(p)[i]) << 16);
  };
  float acc = accumulate ? __uint_as_float(uint32_t(d[i]) << 16) : f(srcs.p[0]);
  for (uint32_t r = accumulate ? 0 : 1; r < nsrc; ++r) acc = __fadd_rn(acc, f(srcs.p[r]));
  d[i] = __bfloat16_as_ushort(__float2bfloat16_rn(acc));
}

template <typename T>
__global__ void k_grad_sum_tail(Srcs srcs, uint32_t nsrc, uint8_t* dst, uint64_t first,
                                uint64_t n, int accumulate) {
  const uint64_t i = first + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T* d = reinterpret_cast<T*>(dst);
  T acc = accumulate ? d[i] : reinterpret_cast<const T*>(srcs.p[0])[i];
  for (uint32_t r = accumulate ? 0 : 1; r < nsrc; ++r) {
    if constexpr (sizeof(T) == 4)
      acc = __fadd_rn(acc, reinterpret_cast<const T*>(srcs.p[r])[i]);
    else
      acc += reinterpret_cast<const T*>(srcs.p[r])[i];
  }
  d[i] = acc;
}

}  // namespace

int launch_grad_sum(int dtype, uint8_t* arena, const uint64_t* src_addrs, uint32_t nsrc,
                    uint64_t dst_addr, uint64_t elems, int accumulate, cudaStream_t s) {
  if (nsrc > kMaxSrc || elems == 0) return 0;
  Srcs srcs{};
  for (uint32_t r = 0; r < nsrc; ++r) srcs.p[r] = arena + src_addrs[r];
  const uint64_t esz = dtype == SNAP_F32 ? 4 : dtype == SNAP_BF16 ? 2 : 8;
  const uint64_t per16 = 16 / esz;
  const uint64_t n16 = elems / per16;
  int launches = 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (n16) {
    uint64_t blocks = (n16 + 255) / 256;
    if (blocks > uint64_t(sms) * 8) blocks = uint64_t(sms) * 8;
    if (dtype == SNAP_BF16)
      k_grad_sum_bf16<<<unsigned(blocks), 256, 0, s>>>(srcs, nsrc, arena + dst_addr, n16, accumulate);
    else if (dtype == SNAP_F32)
      k_grad_sum<float><<<unsigned(blocks), 256, 0, s>>>(srcs, nsrc, arena + dst_addr, n16, accumulate);
    else
      k_grad_sum<uint64_t><<<unsigned(blocks), 256, 0, s>>>(srcs, nsrc, arena + dst_addr, n16, accumulate);
    ++launches;
  }
  const uint64_t first = n16 * per16;
  if (first < elems) {
    const unsigned tb = unsigned((elems - first + 31) / 32);
    if (dtype == SNAP_BF16)
      k_grad_sum_tail_bf16<<<tb, 32, 0, s>>>(srcs, nsrc, arena + dst_addr, first, elems, accumulate);
    else if (dtype == SNAP_F32)
      k_grad_sum_tail<float><<<1, 32, 0, s>>>(srcs, nsrc, arena + dst_addr, first, elems, accumulate);
    else
      k_grad_sum_tail<uint64_t><<<1, 32, 0, s>>>(srcs, nsrc, arena + dst_addr, first, elems, accumulate);
    ++launches;
  }
  return launches;
}

}  // namespace snap
