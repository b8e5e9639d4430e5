// k_copy.cu — K3 (stream compaction gather into the staging image) and K4
// (inverse scatter-restore), plus the digest comparison used by verified
// restores.
//
// K3 replaces the per-buffer copies of build_manifest's dump
// (content_of + BlobStore::put, ckpt.cpp:161-163) and the swap-out copies of
// execute_switch (host_cache_put, splice.cpp:79-82,266); K4 replaces
// restore_job's Gpu::write_words at the recorded address (ckpt.cpp:522-523)
// and the swap-in writes of execute_switch (splice.cpp:293-303).
//
// One warp moves one chunk: 32 lanes x 16 B per access, 8 independent
// 16-byte loads in flight per lane (4 KiB per warp) before the stores, so a
// persistent grid of 148 x 32 warps keeps ~19 MB of reads in flight. Loads
// and stores use the streaming (.cs / evict-first) hints: neither side is
// re-read soon.
#include <cuda_runtime.h>

#include <algorithm>

#include "snap_internal.h"
#include "table.cuh"

namespace snap {
namespace {

constexpr int kThreads = 512;
constexpr int kUnroll = 8;

__device__ __forceinline__ uint32_t find_buf(const GridDev& g, uint64_t gc) {
  if (g.chunk_buf) return __ldg(g.chunk_buf + gc);
  uint32_t lo = 0, hi = g.nbufs;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(g.cstart + mid) <= gc) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ const uint8_t* chunk_ptr(const uint8_t* arena, const GridDev& g,
                                                    uint64_t gc) {
  if (g.chunk_addr) return arena + __ldg(g.chunk_addr + gc);
  const uint32_t b = find_buf(g, gc);
  return arena + __ldg(g.addr + b) + ((gc - __ldg(g.cstart + b)) << g.chunk_shift);
}

// Warp copy of `len` bytes (multiple of 256, both pointers 256-B aligned).
__device__ __forceinline__ void warp_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                          uint32_t len, int lane) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  const uint32_t n16 = len >> 4;
  uint32_t i = lane;
  for (; i + (kUnroll - 1) * 32 < n16; i += kUnroll * 32) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = __ldcs(s + i + u * 32);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) __stcs(d + i + u * 32, v[u]);
  }
  for (; i < n16; i += 32) __stcs(d + i, __ldcs(s + i));
}

// K3 gather / fix-up. For the k-th staged chunk gc = sel_list[k] with staging
// offset `off`: when the fused hash pass already wrote it there
// (spec_cur[gc] == off) nothing moves; otherwise the chunk is copied from the
// arena (never from the speculative image, so there is no overlap hazard).
// spec_next[gc] = off records the layout as the next snapshot's prediction.
__global__ void __launch_bounds__(kThreads)
k_gather(const uint8_t* __restrict__ arena, GridDev g, const uint32_t* __restrict__ lens,
         const uint32_t* __restrict__ sel_list, const uint64_t* __restrict__ totals,
         const uint64_t* __restrict__ offsets, int by_list, const uint64_t* __restrict__ spec_cur,
         uint64_t* __restrict__ spec_next, uint8_t* __restrict__ staging,
         uint32_t* __restrict__ moved, unsigned int* __restrict__ nmoved) {
  griddep_wait();
  const uint64_t nsel = totals[0];
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * kThreads) >> 5;
  if (spec_cur) {
    // speculative layout: almost every chunk is already in place — check 32
    // list entries per warp step (one per lane, coalesced), copy only the
    // mismatches with the whole warp
    for (uint64_t b = w0 * 32; b < nsel; b += nw * 32) {
      const uint64_t k = b + lane;
      uint32_t gc = 0;
      uint64_t off = 0;
      bool need = false;
      if (k < nsel) {
        gc = sel_list[k];
        off = offsets[by_list ? k : gc];
        if (spec_next) spec_next[gc] = off;
        need = spec_cur[gc] != off;
      }
      unsigned m = __ballot_sync(0xffffffffu, need);
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t gj = __shfl_sync(0xffffffffu, gc, j);
        const uint64_t oj = __shfl_sync(0xffffffffu, off, j);
        warp_copy(staging + oj, chunk_ptr(arena, g, gj), lens[gj], lane);
        if (moved && lane == 0) moved[atomicAdd(nmoved, 1u)] = static_cast<uint32_t>(b + j);
      }
    }
    return;
  }
  for (uint64_t w = w0; w < nsel; w += nw) {
    const uint32_t gc = sel_list[w];
    const uint64_t off = offsets[by_list ? w : gc];
    if (spec_next && lane == 0) spec_next[gc] = off;
    warp_copy(staging + off, chunk_ptr(arena, g, gc), lens[gc], lane);
    if (moved && lane == 0) moved[atomicAdd(nmoved, 1u)] = static_cast<uint32_t>(w);
  }
}

__global__ void __launch_bounds__(kThreads)
k_scatter(uint8_t* __restrict__ arena, GridDev g, const uint32_t* __restrict__ lens,
          const uint8_t* __restrict__ image, const uint64_t* __restrict__ src_off) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * kThreads) >> 5;
  for (uint64_t gc = w0; gc < g.nchunks; gc += nw) {
    uint8_t* dst = const_cast<uint8_t*>(chunk_ptr(arena, g, gc));
    warp_copy(dst, image + src_off[gc], lens[gc], lane);
  }
}

// K4 across GPUs (restore_job materialization after a resize, ckpt.cpp:517-528):
// chunk g of rank `src_rank`'s layout is read from the shard of the rank that
// wrote its first occurrence — over NVLink when that shard lives on a peer GPU
// (CUDA-IPC-mapped staging pointers) — and written at its recorded address.
// One pass: no intermediate gathered image in HBM.
__global__ void __launch_bounds__(kThreads)
k_scatter_shards(uint8_t* __restrict__ arena, GridDev g, const uint32_t* __restrict__ lens,
                 uint64_t row, const uint64_t* __restrict__ owner,
                 const int32_t* __restrict__ writer, const uint64_t* __restrict__ shard_off,
                 const uint8_t* const* __restrict__ shards, unsigned long long* __restrict__ missing) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * kThreads) >> 5;
  unsigned long long miss = 0;
  for (uint64_t gc = w0; gc < g.nchunks; gc += nw) {
    const uint64_t o = owner[row + gc];
    const int32_t w = o == ~0ull ? -1 : writer[o];
    if (w < 0) {
      miss += 1;
      continue;
    }
    uint8_t* dst = const_cast<uint8_t*>(chunk_ptr(arena, g, gc));
    warp_copy(dst, shards[w] + shard_off[o], lens[gc], lane);
  }
  if (lane == 0 && miss) atomicAdd(missing, miss);
}

// K3 from an image instead of the arena: list entry k (chunk sel_list[k]) is
// copied from image + src_off[chunk] to dst + offsets[chunk] (splice cache
// seeding from restored blobs).
__global__ void __launch_bounds__(kThreads)
k_gather_from(const uint8_t* __restrict__ image, const uint64_t* __restrict__ src_off,
              const uint32_t* __restrict__ lens, const uint32_t* __restrict__ sel_list,
              const uint64_t* __restrict__ totals, const uint64_t* __restrict__ offsets,
              int by_list, uint8_t* __restrict__ dst) {
  griddep_wait();
  const uint64_t nsel = totals[0];
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * kThreads) >> 5;
  for (uint64_t w = w0; w < nsel; w += nw) {
    const uint32_t gc = sel_list[w];
    warp_copy(dst + offsets[by_list ? w : gc], image + src_off[gc], lens[gc], lane);
  }
}

__global__ void k_compare(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                          uint64_t n, unsigned long long* nbad) {
  unsigned long long bad = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    bad += a[i] != b[i];
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(nbad, bad);
}

// Splice swap-out bookkeeping, before the gather: list entry k (chunk
// sel_list[k]) takes the free cache slot free_stack[free_n - 1 - k]; its
// gather destination is list_off[k] = slot << slot_shift and its digest is
// indexed digest -> slot (the B200 replacement of host_cache_put's
// digest-keyed std::map, splice.cpp:79-82). The host guarantees
// totals[0] <= free_n.
__global__ void k_cache_assign(TableDev cache, const uint64_t* __restrict__ dig,
                               const uint32_t* __restrict__ sel_list,
                               const uint64_t* __restrict__ totals,
                               const uint32_t* __restrict__ lens,
                               const uint32_t* __restrict__ free_stack, uint64_t free_n,
                               uint32_t slot_shift, uint64_t* __restrict__ list_off,
                               uint32_t* __restrict__ slot_len) {
  griddep_wait();
  const uint64_t n = totals[0];
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n && k < free_n;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t g = sel_list[k];
    const uint32_t slot = free_stack[free_n - 1 - k];
    list_off[k] = uint64_t(slot) << slot_shift;
    slot_len[slot] = lens[g];
    const uint64_t s = table_find_or_insert(cache, dig[g]);
    cache.vals[s] = slot;
  }
}

// Splice cache reclamation (no reference counterpart: the reference's host
// cache is an unbounded std::map, splice.hpp:128; the B200 cache is a fixed
// HBM slot array). Every entry of the old index whose digest is still recorded
// by some rank (`live`) is re-indexed into `fresh`; the slots of the others go
// back on the free stack (cnt[0] slots freed, cnt[1] bytes freed, cnt[2] kept).
__global__ void k_cache_gc(TableDev old, TableDev live, TableDev fresh,
                           uint32_t* __restrict__ free_stack, uint64_t free_n,
                           const uint32_t* __restrict__ slot_len,
                           unsigned long long* __restrict__ cnt) {
  const uint64_t n = old.mask + 2;
  for (uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < n;
       s += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned long long key = s == old.mask + 1 ? kEmptyKey : old.keys[s];
    const unsigned long long slot = old.vals[s];
    if (s == old.mask + 1 ? slot == ~0ull : key == kEmptyKey) continue;
    if (table_find(live, key) != ~0ull) {
      const uint64_t f = table_find_or_insert(fresh, key);
      fresh.vals[f] = slot;
      atomicAdd(cnt + 2, 1ull);
    } else {
      free_stack[free_n + atomicAdd(cnt + 0, 1ull)] = uint32_t(slot);
      atomicAdd(cnt + 1, static_cast<unsigned long long>(slot_len[slot]));
    }
  }
}

// Byte-range copies (result installs): range r copies bytes[r] (multiple of
// 16) from src[r] to dst[r]; every CTA takes a slice of every range.
__global__ void __launch_bounds__(kThreads)
k_copy_ranges(uint8_t* const* __restrict__ dst, const uint8_t* const* __restrict__ src,
              const uint64_t* __restrict__ bytes, uint32_t nr) {
  for (uint32_t r = 0; r < nr; ++r) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src[r]);
    uint4* d4 = reinterpret_cast<uint4*>(dst[r]);
    const uint64_t n16 = bytes[r] >> 4;
    for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < n16;
         i += uint64_t(gridDim.x) * kThreads)
      __stcs(d4 + i, __ldcs(s4 + i));
  }
}

// Splice swap-in (plan_switch swap-in phase + execute_switch, splice.cpp:186-226,
// 293-303, with the stale-digest fix of SURVEY App. A-1): chunk g of the
// incoming rank is already resident when the outgoing rank's fresh digest of
// the same address range equals the incoming rank's recorded digest;
// otherwise its bytes come from the device chunk cache by digest. A digest
// missing from the cache is counted (content lost -> SimFault on the host).
// End of a splice switch: the swap-in counters and the selection totals go
// to mapped pinned host memory in one tiny launch (no device memset, no
// pageable read-backs), and the counters are re-armed for the next switch.
__global__ void k_splice_report(unsigned long long* counters, const uint64_t* totals,
                                unsigned long long* host) {
  griddep_wait();
  if (threadIdx.x == 0) {
    volatile unsigned long long* h = host;
    for (int i = 0; i < 3; ++i) {
      h[i] = counters[i];
      counters[i] = 0;
    }
    h[3] = totals ? totals[0] : 0;
    h[4] = totals ? totals[1] : 0;
    __threadfence_system();
  }
}

__global__ void __launch_bounds__(kThreads)
k_splice_in(uint8_t* __restrict__ arena, GridDev to, const uint32_t* __restrict__ lens,
            const uint64_t* __restrict__ want, const int64_t* __restrict__ match,
            const uint64_t* __restrict__ dig_from, TableDev cache,
            const uint8_t* __restrict__ cache_base, uint32_t slot_shift,
            unsigned long long* __restrict__ counters) {
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * kThreads) >> 5;
  unsigned long long swapped = 0, resident = 0, missing = 0;
  // resident test of 8 chunks per warp step (lanes 0-7; the grid keeps about
  // one step per warp, so swap-ins still spread over every warp); the chunks
  // that need bytes from the cache are copied one at a time by the whole warp
  constexpr int kTest = 8;
  const int tl = lane & (kTest - 1);
  for (uint64_t b = w0 * kTest; b < to.nchunks; b += nw * kTest) {
    const uint64_t g = b + tl;
    uint64_t d = 0;
    uint32_t len = 0;
    bool need = false;
    if (g < to.nchunks) {
      d = want[g];
      len = lens[g];
      const int64_t m = match ? match[g] : -1;
      if (m >= 0 && dig_from[m] == d) {
        if (lane < kTest) resident += len;
      } else {
        need = true;
      }
    }
    unsigned msk = __ballot_sync(0xffffffffu, need) & ((1u << kTest) - 1);
    while (msk) {
      const int q = __ffs(msk) - 1;
      msk &= msk - 1;
      const uint64_t gq = __shfl_sync(0xffffffffu, g, q);
      const uint64_t dq = __shfl_sync(0xffffffffu, d, q);
      const uint32_t lq = __shfl_sync(0xffffffffu, len, q);
      const uint64_t s = table_find(cache, dq);
      if (s == ~0ull) {
        if (lane == 0) missing += 1;
        continue;
      }
      uint8_t* dst = const_cast<uint8_t*>(chunk_ptr(arena, to, gq));
      warp_copy(dst, cache_base + (cache.vals[s] << slot_shift), lq, lane);
      if (lane == 0) swapped += lq;
    }
  }
  for (int o = 16; o > 0; o >>= 1) resident += __shfl_xor_sync(0xffffffffu, resident, o);
  if (lane == 0) {
    if (swapped) atomicAdd(counters + 0, swapped);
    if (resident) atomicAdd(counters + 1, resident);
    if (missing) atomicAdd(counters + 2, missing);
  }
}

unsigned copy_grid() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return unsigned(n) * 2;  // 2 CTAs x 16 warps per SM
}

}  // namespace

int launch_gather(const uint8_t* arena, const GridDev& g, const uint32_t* lens,
                  const uint32_t* sel_list, const uint64_t* totals, const uint64_t* offsets,
                  bool offsets_by_list, const uint64_t* spec_cur, uint64_t* spec_next,
                  uint8_t* staging, uint64_t max_sel, cudaStream_t s, uint32_t* moved,
                  unsigned int* nmoved) {
  if (max_sel == 0) return 0;
  // speculative path: one list entry per thread; otherwise one chunk per warp
  uint64_t blocks = ((spec_cur ? max_sel : max_sel * 32) + kThreads - 1) / kThreads;
  if (blocks > copy_grid()) blocks = copy_grid();
  launch_pdl(k_gather, unsigned(blocks), kThreads, 0, s, arena, g, lens, sel_list, totals, offsets,
             offsets_by_list ? 1 : 0, spec_cur, spec_next, staging, moved, nmoved);
  return 1;
}

int launch_scatter(uint8_t* arena, const GridDev& g, const uint32_t* lens, const uint8_t* image,
                   const uint64_t* src_off, cudaStream_t s) {
  if (g.nchunks == 0) return 0;
  uint64_t blocks = (g.nchunks * 32 + kThreads - 1) / kThreads;
  if (blocks > copy_grid()) blocks = copy_grid();
  k_scatter<<<unsigned(blocks), kThreads, 0, s>>>(arena, g, lens, image, src_off);
  return 1;
}

int launch_gather_from(const uint8_t* image, const uint64_t* src_off, const uint32_t* lens,
                       const uint32_t* sel_list, const uint64_t* totals, const uint64_t* offsets,
                       uint8_t* dst, uint64_t max_sel, cudaStream_t s, bool offsets_by_list) {
  if (max_sel == 0) return 0;
  uint64_t blocks = (max_sel * 32 + kThreads - 1) / kThreads;
  if (blocks > copy_grid()) blocks = copy_grid();
  launch_pdl(k_gather_from, unsigned(blocks), kThreads, 0, s, image, src_off, lens, sel_list,
             totals, offsets, offsets_by_list ? 1 : 0, dst);
  return 1;
}

int launch_cache_assign(TableDev cache, const uint64_t* dig, const uint32_t* sel_list,
                        const uint64_t* totals, const uint32_t* lens, const uint32_t* free_stack,
                        uint64_t free_n, uint32_t slot_shift, uint64_t* list_off,
                        uint32_t* slot_len, uint64_t max_n, cudaStream_t s) {
  if (max_n == 0 || free_n == 0) return 0;
  uint64_t blocks = (std::min(max_n, free_n) + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch_pdl(k_cache_assign, unsigned(blocks), 256, 0, s, cache, dig, sel_list, totals, lens,
             free_stack, free_n, slot_shift, list_off, slot_len);
  return 1;
}

int launch_cache_gc(TableDev old, TableDev live, TableDev fresh, uint32_t* free_stack,
                    uint64_t free_n, const uint32_t* slot_len, unsigned long long* cnt,
                    cudaStream_t s) {
  cudaMemsetAsync(cnt, 0, 3 * sizeof(unsigned long long), s);
  uint64_t blocks = (old.mask + 2 + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_cache_gc<<<unsigned(blocks), 256, 0, s>>>(old, live, fresh, free_stack, free_n, slot_len, cnt);
  return 1;
}

int launch_copy_ranges(uint8_t* const* dst, const uint8_t* const* src, const uint64_t* bytes,
                       uint32_t nr, uint64_t max_bytes, cudaStream_t s) {
  if (nr == 0 || max_bytes == 0) return 0;
  uint64_t blocks = (max_bytes / 16 + kThreads - 1) / kThreads;
  if (blocks > copy_grid()) blocks = copy_grid();
  k_copy_ranges<<<unsigned(blocks), kThreads, 0, s>>>(dst, src, bytes, nr);
  return 1;
}

int launch_splice_in(uint8_t* arena, const GridDev& to, const uint32_t* lens, const uint64_t* want,
                     const int64_t* match, const uint64_t* dig_from, TableDev cache,
                     const uint8_t* cache_base, uint32_t slot_shift, unsigned long long* counters,
                     cudaStream_t s) {
  // counters are zero on entry (zeroed at init, re-armed by k_splice_report)
  if (to.nchunks == 0) return 0;
  uint64_t blocks = (to.nchunks * 4 + kThreads - 1) / kThreads;  // 8 chunks per warp step
  if (blocks > copy_grid()) blocks = copy_grid();
  launch_pdl(k_splice_in, unsigned(blocks), kThreads, 0, s, arena, to, lens, want, match, dig_from,
             cache, cache_base, slot_shift, counters);
  return 1;
}

int launch_splice_report(unsigned long long* counters, const uint64_t* totals,
                         unsigned long long* host, cudaStream_t s) {
  launch_pdl(k_splice_report, 1, 32, 0, s, counters, totals, host);
  return 1;
}

int launch_scatter_shards(uint8_t* arena, const GridDev& g, const uint32_t* lens, uint64_t row,
                         const uint64_t* owner, const int32_t* writer, const uint64_t* shard_off,
                         const uint8_t* const* shards, unsigned long long* missing,
                         cudaStream_t s) {
  cudaMemsetAsync(missing, 0, sizeof(unsigned long long), s);
  if (g.nchunks == 0) return 0;
  uint64_t blocks = (g.nchunks * 32 + kThreads - 1) / kThreads;
  if (blocks > copy_grid()) blocks = copy_grid();
  k_scatter_shards<<<unsigned(blocks), kThreads, 0, s>>>(arena, g, lens, row, owner, writer,
                                                         shard_off, shards, missing);
  return 1;
}

int launch_compare(const uint64_t* a, const uint64_t* b, uint64_t n, unsigned long long* nbad,
                   cudaStream_t s) {
  cudaMemsetAsync(nbad, 0, sizeof(unsigned long long), s);
  if (n == 0) return 0;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_compare<<<unsigned(blocks), 256, 0, s>>>(a, b, n, nbad);
  return 1;
}

}  // namespace snap
