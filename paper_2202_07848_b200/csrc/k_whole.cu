// k_whole.cu — the reference's WHOLE-BUFFER digest, value-equal
// (Gpu::digest, vdev.cpp:118 = digest_of_words over every byte of the range,
// sim.hpp:55-70): the opt-in compatibility path of SURVEY §8(c). The snapshot
// path keys buffers by a chunk-Merkle digest instead (equality-equivalent, and
// parallel); this path exists so a caller can get the exact reference value.
//
// FNV-1a is one serial chain per buffer, but it is affine in the state up to
// its low byte: with l = h mod 256 and u = l ^ b, (h ^ b) * P = h*P + (u - l)*P,
// so a segment of L bytes maps h -> h*P^L + D(h mod 256) where D depends only on
// the segment and the entry low byte (256 possibilities). Hence:
//   K-A (parallel): for every 64 KiB segment and every entry low byte l, run
//        FNV-1a from the state l over the segment: F(l) = l*P^L + D(l)
//        (one CTA per segment, 256 threads = 256 chains over the same bytes
//        staged once in shared memory, broadcast reads);
//   K-B (serial, tiny): per buffer, h <- (h - l)*P^L + F(l), l = h mod 256,
//        segment by segment — one 8-byte table lookup + one multiply-add per
//        64 KiB, the tables streamed through shared memory.
// 256 chains per byte makes K-A ~256x the work of one chain, but it spreads
// over every SM; the serial part shrinks from 1 step per byte to 1 per 64 KiB.
#include <cuda_runtime.h>

#include "snap_internal.h"

namespace snap {
namespace {

constexpr uint32_t kSegShift = 16;  // 64 KiB segments
constexpr uint32_t kSeg = 1u << kSegShift;
constexpr uint64_t kPrime = 0x100000001b3ull;

__device__ __forceinline__ uint64_t pow_prime(uint64_t e) {
  uint64_t r = 1, b = kPrime;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

// segment s of the list: buffer b = the last with seg_start[b] <= s
__device__ __forceinline__ uint32_t seg_buf(const uint64_t* seg_start, uint32_t nb, uint64_t s) {
  uint32_t lo = 0, hi = nb;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (seg_start[mid] <= s) lo = mid; else hi = mid;
  }
  return lo;
}

// K-A: F[s * 256 + l] = FNV-1a over segment s starting from the state l.
__global__ void __launch_bounds__(256)
k_whole_tables(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ addr,
               const uint64_t* __restrict__ bytes, const uint64_t* __restrict__ seg_start,
               uint32_t nb, uint64_t nseg, uint64_t* __restrict__ F) {
  extern __shared__ __align__(16) uint8_t seg[];
  for (uint64_t s = blockIdx.x; s < nseg; s += gridDim.x) {
    const uint32_t b = seg_buf(seg_start, nb, s);
    const uint64_t off = (s - seg_start[b]) << kSegShift;
    const uint64_t rem = bytes[b] - off;
    const uint32_t len = rem < kSeg ? uint32_t(rem) : kSeg;  // multiple of 256
    const uint4* src = reinterpret_cast<const uint4*>(arena + addr[b] + off);
    __syncthreads();  // previous segment consumed
    for (uint32_t i = threadIdx.x; i < (len >> 4); i += 256)
      reinterpret_cast<uint4*>(seg)[i] = __ldcs(src + i);
    __syncthreads();
    uint64_t h = threadIdx.x;
    const uint4* p = reinterpret_cast<const uint4*>(seg);
    for (uint32_t i = 0; i < (len >> 4); ++i) {
      const uint4 v = p[i];  // same address in every lane: broadcast
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          h ^= (w[k] >> (8 * j)) & 0xffu;
          h *= kPrime;
        }
      }
    }
    F[s * 256 + threadIdx.x] = h;
  }
}

// K-B: one CTA per buffer; its segments' tables are staged through shared
// memory in blocks, thread 0 walks the chain.
constexpr uint32_t kBlockSegs = 48;  // 48 x 2 KiB = 96 KiB of tables per block
__global__ void __launch_bounds__(256)
k_whole_combine(const uint64_t* __restrict__ bytes, const uint64_t* __restrict__ seg_start,
                uint32_t nb, const uint64_t* __restrict__ F, uint64_t* __restrict__ out) {
  extern __shared__ __align__(16) uint64_t tab[];
  __shared__ uint64_t s_h;
  const uint32_t b = blockIdx.x;
  if (b >= nb) return;
  const uint64_t s0 = seg_start[b], s1 = seg_start[b + 1], n = bytes[b];
  const uint64_t p_full = pow_prime(kSeg);
  if (threadIdx.x == 0) s_h = 14695981039346656037ull;  // digest_of({}), sim.hpp:57
  for (uint64_t sb = s0; sb < s1; sb += kBlockSegs) {
    const uint64_t ns = (s1 - sb) < kBlockSegs ? (s1 - sb) : kBlockSegs;
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < ns * 256; i += 256) tab[i] = __ldcs(F + sb * 256 + i);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t h = s_h;
      for (uint64_t k = 0; k < ns; ++k) {
        const uint64_t s = sb + k;
        const uint64_t seg_len = (s + 1 == s1) ? n - ((s - s0) << kSegShift) : kSeg;
        const uint64_t pl = seg_len == kSeg ? p_full : pow_prime(seg_len);
        const uint64_t l = h & 0xff;
        h = (h - l) * pl + tab[k * 256 + l];
      }
      s_h = h;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[b] = s_h;
}

}  // namespace

uint64_t whole_segments(uint64_t bytes) { return (bytes + kSeg - 1) >> kSegShift; }

int launch_whole_digest(const uint8_t* arena, const uint64_t* addr, const uint64_t* bytes,
                        const uint64_t* seg_start, uint32_t nb, uint64_t nseg, uint64_t* F,
                        uint64_t* out, cudaStream_t s) {
  if (nb == 0) return 0;
  static uint64_t attr = 0;
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_whole_tables, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSeg));
    cudaFuncSetAttribute(k_whole_combine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kBlockSegs * 256 * 8));
  });
  int n = 0;
  if (nseg) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t blocks = nseg < uint64_t(sms) * 3 ? nseg : uint64_t(sms) * 3;
    k_whole_tables<<<unsigned(blocks), 256, kSeg, s>>>(arena, addr, bytes, seg_start, nb, nseg, F);
    ++n;
  }
  k_whole_combine<<<nb, 256, kBlockSegs * 256 * 8, s>>>(bytes, seg_start, nb, F, out);
  return n + 1;
}

}  // namespace snap
