// k_hash.cu — K1: per-page / per-chunk 64-bit FNV-1a content digests over
// every tracked allocation (replaces sim::digest_of_words, sim.hpp:55-70, as
// called by Gpu::digest vdev.cpp:118, GpuLedger::refresh_digests
// splice.cpp:150-159 / plan_switch splice.cpp:176 and BlobStore::put
// ckpt.cpp:17).
//
// FNV-1a is byte-serial inside one digest, so parallelism comes from hashing
// many pages at once: one lane = one page chain, one warp = 32 consecutive
// page slots (= 2 chunks of 16 pages by default). Data reaches the lanes
// through shared memory: per stage the warp issues coalesced 16-byte
// cp.async copies (8 lanes per 128-byte page slab, 4 pages per instruction)
// into an XOR-swizzled slab layout, so both the copy-in and each lane's
// 16-byte LDS of its own slab are bank-conflict free. kStages-deep
// pipelining keeps ~100 KB in flight per SM. The 16 page digests of a chunk
// are folded into the chunk digest with warp shuffles (digest_of_words over
// the page digests).
//
// Per byte the chain costs ~4.75 integer instructions: FNV prime
// 2^40 + 0x1b3 is applied on 32-bit halves as one IMAD.WIDE.U32 (low half
// and carry), one IMAD + one shift/add for the high half, plus the xor/byte
// extraction.
#include <cuda_runtime.h>

#include "snap_internal.h"

namespace snap {
namespace {

constexpr int kWarps = 16;                 // 512 threads, 1 CTA per SM
constexpr int kStages = 3;                 // cp.async pipeline depth
constexpr int kSlab = 128;                 // bytes of one page per stage
constexpr int kStageBytes = 32 * kSlab;    // one warp-stage (32 pages)
constexpr int kWarpBytes = kStages * kStageBytes;
constexpr uint32_t kFull = 0xffffffffu;

struct Desc {
  const uint8_t* src;
  uint32_t len;
  uint32_t pad;
};
constexpr size_t kSmemBytes = size_t(kWarps) * kWarpBytes + size_t(kWarps) * 64 * sizeof(Desc);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;\n" ::"r"(dst), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// One FNV-1a byte step on the (lo, hi) halves of the 64-bit state. Only the
// low 8 bits of `b` are used.
// h' = (h ^ b) * (2^40 + c) mod 2^64 with x = lo ^ b, t = x * c (64-bit):
//   lo' = lo(t),  hi' = hi * c + hi(t) + (x << 8).
// The (x << 8) + hi(t) term is written as one PTX shl+add so ptxas emits a
// single LEA (or an IMAD, whichever pipe is idle): 4.75 SASS ops per byte
// (LOP3, 3/4 SHF, LEA|IMAD, IMAD, IMAD.WIDE.U32), split evenly between the
// ALU and FMA pipes.
__device__ __forceinline__ void fnv_step(uint32_t& lo, uint32_t& hi, uint32_t b) {
  const uint32_t x = lo ^ (b & 0xffu);
  const uint64_t t = static_cast<uint64_t>(x) * kFnvPrimeLo;  // IMAD.WIDE.U32
  uint32_t y;
  asm("{\n\t.reg .u32 s;\n\tshl.b32 s, %1, 8;\n\tadd.u32 %0, s, %2;\n\t}"
      : "=r"(y)
      : "r"(x), "r"(static_cast<uint32_t>(t >> 32)));
  hi = hi * kFnvPrimeLo + y;
  lo = static_cast<uint32_t>(t);
}
__device__ __forceinline__ void fnv_word(uint32_t& lo, uint32_t& hi, uint32_t w) {
  fnv_step(lo, hi, w);
  fnv_step(lo, hi, w >> 8);
  fnv_step(lo, hi, w >> 16);
  fnv_step(lo, hi, w >> 24);
}

// Last buffer b with cstart[b] <= gc (cstart has nbufs + 1 entries).
__device__ __forceinline__ uint32_t find_buf(const GridDev& g, uint64_t gc) {
  uint32_t lo = 0, hi = g.nbufs;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(g.cstart + mid) <= gc) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kWarps * 32, 1)
k_hash(const uint8_t* __restrict__ arena, GridDev g, uint64_t* __restrict__ chunk_dig) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint8_t* wbuf = smem + warp * kWarpBytes;
  Desc* desc = reinterpret_cast<Desc*>(smem + kWarps * kWarpBytes) + warp * 64;

  const uint32_t ppc_shift = g.chunk_shift - g.page_shift;  // pages per chunk (log2)
  const uint32_t ns_shift = g.page_shift - 7;               // stages per page (log2)
  const uint32_t ns = 1u << ns_shift;
  const uint64_t nslots = g.nchunks << ppc_shift;
  const uint64_t ntasks = (nslots + 31) >> 5;
  const uint64_t gw = uint64_t(blockIdx.x) * kWarps + warp;
  const uint64_t nw = uint64_t(gridDim.x) * kWarps;
  if (gw >= ntasks) return;
  const uint64_t my_tasks = (ntasks - gw + nw - 1) / nw;
  const uint64_t nsteps = my_tasks << ns_shift;

  // Producer: slot descriptors at the first stage of a task, then 8 coalesced
  // 16-byte cp.async per lane per stage (lanes 8q..8q+7 cover one 128 B slab).
  auto issue = [&](uint64_t p) {
    if (p < nsteps) {
      const uint64_t i = p >> ns_shift;
      const uint32_t s = static_cast<uint32_t>(p) & (ns - 1);
      Desc* dt = desc + (i & 1) * 32;
      if (s == 0) {
        const uint64_t slot = (gw + i * nw) * 32 + lane;
        const uint64_t gc = slot >> ppc_shift;
        Desc d{nullptr, 0u, 0u};
        if (gc < g.nchunks) {
          const uint32_t b = find_buf(g, gc);
          const uint64_t k = gc - __ldg(g.cstart + b);
          const uint64_t off = (k << g.chunk_shift) +
                               ((slot & ((1u << ppc_shift) - 1)) << g.page_shift);
          const uint64_t bytes = __ldg(g.bytes + b);
          if (off < bytes) {
            const uint64_t rem = bytes - off;
            d.len = static_cast<uint32_t>(rem < (1ull << g.page_shift) ? rem : (1ull << g.page_shift));
            d.src = arena + __ldg(g.addr + b) + off;
          }
        }
        dt[lane] = d;
        __syncwarp();
      }
      const uint32_t sbase = smem_u32(wbuf + (p % kStages) * kStageBytes);
      const uint32_t u = lane & 7;
      const uint32_t off = s * kSlab + u * 16;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = k * 4 + (lane >> 3);
        const Desc d = dt[j];
        if (off < d.len) cp_async16(sbase + j * kSlab + ((u ^ (j & 7)) << 4), d.src + off);
      }
    }
    cp_commit();
  };

#pragma unroll
  for (int p = 0; p < kStages - 1; ++p) issue(p);

  uint32_t lo = 0, hi = 0, mylen = 0;
  for (uint64_t t = 0; t < nsteps; ++t) {
    issue(t + kStages - 1);
    cp_wait<kStages - 1>();
    __syncwarp();
    const uint64_t i = t >> ns_shift;
    const uint32_t s = static_cast<uint32_t>(t) & (ns - 1);
    if (s == 0) {
      mylen = desc[(i & 1) * 32 + lane].len;
      lo = static_cast<uint32_t>(kFnvOffset);
      hi = static_cast<uint32_t>(kFnvOffset >> 32);
    }
    if (s * kSlab < mylen) {
      const uint8_t* slab = wbuf + (t % kStages) * kStageBytes + lane * kSlab;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint4 v = *reinterpret_cast<const uint4*>(slab + ((u ^ (lane & 7)) << 4));
        fnv_word(lo, hi, v.x);
        fnv_word(lo, hi, v.y);
        fnv_word(lo, hi, v.z);
        fnv_word(lo, hi, v.w);
      }
    }
    __syncwarp();
    if (s == ns - 1) {
      // Task complete: every lane holds one page digest (or nothing).
      const uint64_t slot0 = (gw + i * nw) * 32;
      if (ppc_shift == 0) {
        const uint64_t gc = slot0 + lane;
        if (mylen > 0) chunk_dig[gc] = (uint64_t(hi) << 32) | lo;
      } else {
        // chunk digest = digest_of_words(page digests): every lane of a group
        // folds the same 8-byte words (warp-uniform shuffles), the group's
        // first lane stores it.
        const uint32_t ppc = 1u << ppc_shift;
        const int base = lane & ~static_cast<int>(ppc - 1);
        uint32_t flo = static_cast<uint32_t>(kFnvOffset);
        uint32_t fhi = static_cast<uint32_t>(kFnvOffset >> 32);
        for (uint32_t q = 0; q < ppc; ++q) {
          const uint32_t plo = __shfl_sync(kFull, lo, base + q);
          const uint32_t phi = __shfl_sync(kFull, hi, base + q);
          const uint32_t pl = __shfl_sync(kFull, mylen, base + q);
          if (pl > 0) {
            fnv_word(flo, fhi, plo);
            fnv_word(flo, fhi, phi);
          }
        }
        const uint64_t gc = (slot0 + lane) >> ppc_shift;
        if (lane == base && mylen > 0) chunk_dig[gc] = (uint64_t(fhi) << 32) | flo;
      }
    }
  }
  cp_wait<0>();
}

// Buffer digest = digest_of_words(chunk digests of the buffer); one thread
// per buffer (digest vectors are 1/8192 of the data).
__global__ void k_buf_fold(GridDev g, const uint64_t* __restrict__ chunk_dig,
                           uint64_t* __restrict__ buf_dig) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= g.nbufs) return;
  uint32_t lo = static_cast<uint32_t>(kFnvOffset), hi = static_cast<uint32_t>(kFnvOffset >> 32);
  for (uint64_t c = g.cstart[b]; c < g.cstart[b + 1]; ++c) {
    const uint64_t d = chunk_dig[c];
    fnv_word(lo, hi, static_cast<uint32_t>(d));
    fnv_word(lo, hi, static_cast<uint32_t>(d >> 32));
  }
  buf_dig[b] = (uint64_t(hi) << 32) | lo;
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void k_fill_mix64(uint64_t* __restrict__ dst, uint64_t n, uint64_t seed, uint64_t base) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * 2;
  for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2; i < n; i += stride) {
    if (i + 1 < n) {
      ulonglong2 v{mix64(seed ^ (base + i)), mix64(seed ^ (base + i + 1))};
      *reinterpret_cast<ulonglong2*>(dst + i) = v;
    } else {
      dst[i] = mix64(seed ^ (base + i));
    }
  }
}

__global__ void k_xor_words(uint8_t* arena, const uint64_t* __restrict__ addrs, uint64_t n,
                            uint64_t value) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    *reinterpret_cast<uint64_t*>(arena + addrs[i]) ^= value;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

int launch_hash(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig, cudaStream_t s) {
  if (g.nchunks == 0) return 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_hash, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes));
    attr = true;
  }
  const uint64_t ntasks = ((g.nchunks << (g.chunk_shift - g.page_shift)) + 31) >> 5;
  uint64_t blocks = (ntasks + kWarps - 1) / kWarps;
  const uint64_t cap = uint64_t(sm_count());
  if (blocks > cap) blocks = cap;
  k_hash<<<unsigned(blocks), kWarps * 32, kSmemBytes, s>>>(arena, g, chunk_dig);
  return 1;
}

int launch_buf_fold(const GridDev& g, const uint64_t* chunk_dig, uint64_t* buf_dig,
                    cudaStream_t s) {
  if (g.nbufs == 0) return 0;
  k_buf_fold<<<(g.nbufs + 127) / 128, 128, 0, s>>>(g, chunk_dig, buf_dig);
  return 1;
}

int launch_fill_mix64(uint64_t* dst, uint64_t nwords, uint64_t seed, uint64_t base,
                      cudaStream_t s) {
  if (nwords == 0) return 0;
  uint64_t blocks = (nwords / 2 + 255) / 256;
  const uint64_t cap = uint64_t(sm_count()) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  k_fill_mix64<<<unsigned(blocks), 256, 0, s>>>(dst, nwords, seed, base);
  return 1;
}

int launch_xor_words(uint8_t* arena, const uint64_t* addrs, uint64_t n, uint64_t value,
                     cudaStream_t s) {
  if (n == 0) return 0;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_xor_words<<<unsigned(blocks), 256, 0, s>>>(arena, addrs, n, value);
  return 1;
}

}  // namespace snap
