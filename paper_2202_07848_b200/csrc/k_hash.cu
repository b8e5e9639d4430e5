// k_hash.cu — K1: per-page / per-chunk 64-bit FNV-1a content digests over
// every tracked allocation (replaces sim::digest_of_words, sim.hpp:55-70, as
// called by Gpu::digest vdev.cpp:118, GpuLedger::refresh_digests
// splice.cpp:150-159 / plan_switch splice.cpp:176 and BlobStore::put
// ckpt.cpp:17), optionally fused with K3 stream compaction.
//
// FNV-1a is byte-serial inside one digest, so parallelism comes from hashing
// many pages at once: one lane = one page chain, one warp = 32 consecutive
// chunk-aligned page slots (= 2 chunks of 16 pages by default). Each lane
// streams its page through a private ring of 128-byte shared-memory slabs
// filled by its own TMA bulk copies (cp.async.bulk, one mbarrier per slab),
// hashes each slab with conflict-free 16-byte LDS (slabs padded to 144 B),
// and — when the chunk is predicted to be staged — writes the same slab to
// the staging image with a TMA bulk store (cp.async.bulk.global.shared), so
// the image is read from HBM exactly once for hash + compaction. The 16 page
// digests of a chunk are folded into the chunk digest with warp shuffles
// (digest_of_words over the page digests).
#include <cuda_runtime.h>

#include "snap_internal.h"

namespace snap {
namespace {

// Per-lane TMA pipeline: 15 warps x 32 lanes = 480 page chains per SM; each
// lane owns kStages slabs of 128 B (+16 B pad so the 16-byte LDS of 8
// consecutive lanes hit 8 different bank groups) and one mbarrier per slab.
constexpr int kWarps = 15;
constexpr int kStages = 3;                       // slab ring per lane
constexpr int kSlab = 128;                       // bytes of a page per step
constexpr int kSlabStride = kSlab + 16;
constexpr int kStageBytes = 32 * kSlabStride;    // one warp-stage
constexpr size_t kSmemBytes =
    size_t(kWarps) * kStages * kStageBytes + size_t(kWarps) * kStages * 32 * 8;
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared (completes tx bytes on `bar`).
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// TMA bulk copy shared -> global (bulk async-group completion).
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// h' = (h ^ b) * (2^40 + c) mod 2^64 with x = lo ^ b, t = x * c (64-bit):
//   lo' = lo(t),  hi' = hi * c + hi(t) + (x << 8).
// The (x << 8) + hi(t) term is written as one PTX shl+add so ptxas emits a
// single LEA (or an IMAD, whichever pipe is idle): 4.75 SASS ops per byte
// (LOP3, 3/4 SHF, LEA|IMAD, IMAD, IMAD.WIDE.U32). The integer multiplies all
// issue on the FMA-heavy pipe (IMAD 2, IMAD.WIDE 4 cycles per warp), which
// bounds the kernel at ~6 pipe cycles per byte-step per SM sub-partition.
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

// K1 (+ fused K3 when spec_off != nullptr): one lane hashes one page slot of
// a warp task (32 consecutive chunk-aligned page slots), pulling its page
// through its own slab ring with per-lane TMA bulk loads; if the page's chunk
// has a speculative staging offset (spec_off[chunk] != ~0), every slab is
// also written to the staging image with a TMA bulk store straight from
// shared memory, so compaction costs no second HBM read of the chunk.
__global__ void __launch_bounds__(kWarps * 32, 1)
k_hash(const uint8_t* __restrict__ arena, GridDev g, uint64_t* __restrict__ chunk_dig,
       const uint64_t* __restrict__ spec_off, uint8_t* __restrict__ staging) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint8_t* slab0 = smem + (warp * kStages * 32 + lane) * kSlabStride;  // + st * kStageBytes
  const uint32_t slab0_u = smem_u32(slab0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(kWarps) * kStages * kStageBytes);
  const uint32_t bar0 = smem_u32(bars + warp * kStages * 32 + lane);  // + st * 256

  const uint32_t ppc_shift = g.chunk_shift - g.page_shift;  // pages per chunk (log2)
  const uint32_t ns_shift = g.page_shift - 7;               // steps per page (log2)
  const uint32_t ns = 1u << ns_shift;
  const uint64_t nslots = g.nchunks << ppc_shift;
  const uint64_t ntasks = (nslots + 31) >> 5;
  const uint64_t gw = uint64_t(blockIdx.x) * kWarps + warp;
  const uint64_t nw = uint64_t(gridDim.x) * kWarps;
  if (gw >= ntasks) return;
  const uint64_t my_tasks = (ntasks - gw + nw - 1) / nw;
  const uint64_t nsteps = my_tasks << ns_shift;

#pragma unroll
  for (int st = 0; st < kStages; ++st) mbar_init(bar0 + st * 256, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

  // producer-side descriptor of the task being loaded
  const uint8_t* p_src = nullptr;
  uint8_t* p_dst = nullptr;
  uint32_t p_len = 0;
  auto produce = [&](uint64_t p) {
    if (p >= nsteps) return;
    const uint64_t i = p >> ns_shift;
    const uint32_t s = static_cast<uint32_t>(p) & (ns - 1);
    if (s == 0) {
      const uint64_t slot = (gw + i * nw) * 32 + lane;
      const uint64_t gc = slot >> ppc_shift;
      p_src = nullptr;
      p_dst = nullptr;
      p_len = 0;
      if (gc < g.nchunks) {
        const uint32_t b = find_buf(g, gc);
        const uint64_t k = gc - __ldg(g.cstart + b);
        const uint64_t in_chunk = (slot & ((1u << ppc_shift) - 1)) << g.page_shift;
        const uint64_t off = (k << g.chunk_shift) + in_chunk;
        const uint64_t bytes = __ldg(g.bytes + b);
        if (off < bytes) {
          const uint64_t rem = bytes - off;
          p_len = static_cast<uint32_t>(rem < (1ull << g.page_shift) ? rem : (1ull << g.page_shift));
          p_src = arena + __ldg(g.addr + b) + off;
          if (spec_off) {
            const uint64_t so = __ldg(spec_off + gc);
            if (so != ~0ull) p_dst = staging + so + in_chunk;
          }
        }
      }
    }
    const uint32_t st = static_cast<uint32_t>(p % kStages);
    const uint32_t bar = bar0 + st * 256;
    if (s * kSlab < p_len) {
      mbar_arrive_tx(bar, kSlab);
      bulk_load(slab0_u + st * kStageBytes, p_src + s * kSlab, kSlab, bar);
    } else {
      mbar_arrive(bar);
    }
  };

  produce(0);
  uint32_t lo = 0, hi = 0, c_len = 0;
  uint8_t* c_dst = nullptr;
  for (uint64_t t = 0; t < nsteps; ++t) {
    // the slab reloaded now was stored two steps ago: its TMA read must be done
    bulk_wait_read<1>();
    produce(t + 1);
    const uint32_t st = static_cast<uint32_t>(t % kStages);
    mbar_wait(bar0 + st * 256, static_cast<uint32_t>((t / kStages) & 1));
    const uint64_t i = t >> ns_shift;
    const uint32_t s = static_cast<uint32_t>(t) & (ns - 1);
    if (s == 0) {  // the producer is still on this task (ahead by one step < ns)
      c_len = p_len;
      c_dst = p_dst;
      lo = static_cast<uint32_t>(kFnvOffset);
      hi = static_cast<uint32_t>(kFnvOffset >> 32);
    }
    if (s * kSlab < c_len) {
      const uint8_t* slab = slab0 + st * kStageBytes;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint4 v = *reinterpret_cast<const uint4*>(slab + u * 16);
        fnv_word(lo, hi, v.x);
        fnv_word(lo, hi, v.y);
        fnv_word(lo, hi, v.z);
        fnv_word(lo, hi, v.w);
      }
      if (c_dst) bulk_store(c_dst + s * kSlab, slab0_u + st * kStageBytes, kSlab);
    }
    bulk_commit();
    if (s == ns - 1) {
      // Task complete: every lane holds one page digest (or nothing).
      __syncwarp();
      const uint64_t slot0 = (gw + i * nw) * 32;
      if (ppc_shift == 0) {
        if (c_len > 0) chunk_dig[slot0 + lane] = (uint64_t(hi) << 32) | lo;
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
          const uint32_t pl = __shfl_sync(kFull, c_len, base + q);
          if (pl > 0) {
            fnv_word(flo, fhi, plo);
            fnv_word(flo, fhi, phi);
          }
        }
        const uint64_t gc = (slot0 + lane) >> ppc_shift;
        if (lane == base && c_len > 0) chunk_dig[gc] = (uint64_t(fhi) << 32) | flo;
      }
    }
  }
  bulk_wait_all();
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

int launch_hash(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig,
                const uint64_t* spec_off, uint8_t* staging, cudaStream_t s) {
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
  k_hash<<<unsigned(blocks), kWarps * 32, kSmemBytes, s>>>(arena, g, chunk_dig, spec_off, staging);
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
