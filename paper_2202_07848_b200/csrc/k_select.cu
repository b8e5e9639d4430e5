// k_select.cu — K2: dedup table + dirty test + deterministic stream-compaction
// offsets, single GPU and cross-rank (after the NCCL allgather of digest
// vectors).
//
// Reference semantics (build_manifest, ckpt.cpp:97,147-167; BlobStore::put,
// ckpt.cpp:16-21): walking chunks in canonical (rank, slot, chunk) order, a
// chunk is staged iff its digest was not seen earlier in this snapshot AND is
// not already in the store (the "known" set). Order independence on the GPU:
// the dedup table keeps min(canonical index) per digest (atomicMin), so the
// first occurrence is found without ordering threads; staging offsets come
// from a single-pass decoupled look-back scan over canonical chunk order, so
// the staging image is bit-identical run to run.
//
// Cross-rank: every GPU builds the same global table from the
// allgathered vectors; the logical owner is the first occurrence, but the
// physical copy of a replicated chunk is striped over its holders (ranks whose
// chunk at the same local index has the same digest): writer =
// holders[local_index % |holders|]. Each GPU stages only the chunks it writes,
// in canonical order (its shard of the global image).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "snap_internal.h"
#include <algorithm>
#include <cstdlib>

#include "table.cuh"

namespace snap {
namespace {

// chunk address and warp copy (as in k_copy.cu) for the fix-up fused into the scan
__device__ __forceinline__ const uint8_t* chunk_ptr(const uint8_t* arena, const GridDev& g,
                                                    uint64_t gc) {
  if (g.chunk_addr) return arena + __ldg(g.chunk_addr + gc);
  if (g.chunk_buf) {
    const uint32_t b = __ldg(g.chunk_buf + gc);
    return arena + __ldg(g.addr + b) + ((gc - __ldg(g.cstart + b)) << g.chunk_shift);
  }
  uint32_t lo = 0, hi = g.nbufs;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(g.cstart + mid) <= gc) lo = mid; else hi = mid;
  }
  return arena + __ldg(g.addr + lo) + ((gc - __ldg(g.cstart + lo)) << g.chunk_shift);
}

__device__ __forceinline__ void warp_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                          uint32_t len, int lane) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  for (uint32_t i = lane; i < (len >> 4); i += 32) __stcs(d + i, __ldcs(s + i));
}

__global__ void k_table_clear(TableDev t) {
  const uint64_t n = t.mask + 2;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    t.keys[i] = kEmptyKey;
    t.vals[i] = ~0ull;
  }
}

__global__ void k_table_insert_min(TableDev t, const uint64_t* __restrict__ keys, uint64_t n,
                                   uint64_t base) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t s = table_find_or_insert(t, keys[i]);
    atomicMin(t.vals + s, static_cast<unsigned long long>(base + i));
  }
}

// Insert every live chunk (len > 0; padding entries of the allgathered
// vectors have len 0) with its canonical index; record its slot and whether
// the known set holds it, so the scan needs one load per chunk.
__global__ void k_dedup_insert(TableDev dedup, TableDev known, int use_known,
                               const uint64_t* __restrict__ dig, const uint32_t* __restrict__ lens,
                               uint64_t n, uint64_t* __restrict__ slot) {
  griddep_wait();
  for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < n;
       g += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t s = ~0ull;
    if (lens[g] != 0) {
      const unsigned long long d = dig[g];
      const bool is_known = use_known && table_find(known, d) != ~0ull;
      if (!is_known) {
        s = table_find_or_insert(dedup, d);
        atomicMin(dedup.vals + s, static_cast<unsigned long long>(g));
      }
    }
    slot[g] = s;
  }
}

// Multi-rank step (writer and owner only; the global staging offsets are
// computed on demand, snap_get_selection): per global chunk g, owner = first
// occurrence (the dedup table's min index), selected iff owner == g, and the
// stripe writer of a selected chunk: holders = ranks whose chunk at the same
// local index i has the same digest and length, writer = holders[i % |holders|]
// (rank-major global index, `maxn` per rank). Also zeroes the
// shard scan's state (the next kernel on the stream), so the step needs no memset.
__global__ void k_select_stripe(TableDev dedup, const uint64_t* __restrict__ slot,
                                const uint64_t* __restrict__ gdig, const uint32_t* __restrict__ glens,
                                uint32_t nranks, uint64_t maxn, uint8_t* __restrict__ sel,
                                uint64_t* __restrict__ owner, int32_t* __restrict__ writer,
                                uint64_t* __restrict__ scan_state, uint64_t scan_words,
                                uint64_t* __restrict__ spec_next, uint64_t nlocal) {
  griddep_wait();
  const uint64_t n = uint64_t(nranks) * maxn;
  const uint64_t end = n > scan_words ? n : scan_words;
  for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < end;
       g += uint64_t(gridDim.x) * blockDim.x) {
    if (g < scan_words) scan_state[g] = 0;
    if (spec_next && g < nlocal) spec_next[g] = ~0ull;
    if (g >= n) continue;
    const uint64_t s = slot[g];
    const uint64_t own = s == ~0ull ? ~0ull : dedup.vals[s];
    int32_t w = -1;
    if (own == g) {
      const uint64_t i = g % maxn;
      const uint64_t d = gdig[g];
      const uint32_t ln = glens[g];
      uint32_t hold = 0, nh = 0;  // holder ranks as a bit set (nranks <= 32 fast path)
      if (nranks <= 32) {
        for (uint32_t q = 0; q < nranks; ++q)
          if (glens[q * maxn + i] == ln && gdig[q * maxn + i] == d) hold |= 1u << q;
        nh = __popc(hold);
        uint32_t pick = static_cast<uint32_t>(i % nh);
        for (; pick; --pick) hold &= hold - 1;
        w = __ffs(hold) - 1;
      } else {
        for (uint32_t q = 0; q < nranks; ++q)
          nh += (glens[q * maxn + i] == ln && gdig[q * maxn + i] == d);
        uint32_t pick = static_cast<uint32_t>(i % nh), seen = 0;
        for (uint32_t q = 0; q < nranks; ++q)
          if (glens[q * maxn + i] == ln && gdig[q * maxn + i] == d) {
            if (seen == pick) {
              w = static_cast<int32_t>(q);
              break;
            }
            ++seen;
          }
      }
    }
    sel[g] = own == g;
    owner[g] = own;
    writer[g] = w;
  }
}

// ---- decoupled look-back scan -------------------------------------------
// Status word per tile: flag (2 bits) | chunk count (26 bits) | 256-byte units (36 bits).
constexpr int kThreads = 256;
constexpr int kItems = 4;
constexpr int kTile = kThreads * kItems;
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPre = 2ull << 62;
constexpr uint64_t kPayload = (1ull << 62) - 1;
constexpr uint64_t kUnitBits = 36;

__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Block-wide exclusive scan + tile prefix by decoupled look-back. Returns the
// exclusive prefix of this thread's first item; publishes totals from the
// last tile.
__device__ uint64_t tile_scan(uint64_t local, uint64_t tile, uint64_t ntiles, uint64_t* status,
                              uint64_t* totals) {
  __shared__ uint64_t s_warp[kThreads / 32];
  __shared__ uint64_t s_excl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint64_t w = lane < kThreads / 32 ? s_warp[lane] : 0;
    uint64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    const uint64_t agg = __shfl_sync(0xffffffffu, wi, kThreads / 32 - 1);
    if (lane < kThreads / 32) s_warp[lane] = wi - w;
    uint64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_status(status, kFlagPre | agg);
    } else {
      if (lane == 0) st_status(status + tile, kFlagAgg | agg);
      int64_t pred = int64_t(tile) - 1;
      for (;;) {
        const int64_t idx = pred - lane;
        uint64_t st = idx >= 0 ? ld_status(status + idx) : kFlagPre;
        while (__any_sync(0xffffffffu, (st >> 62) == 0)) {
          if ((st >> 62) == 0) st = ld_status(status + idx);
        }
        const unsigned pmask = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        const int first_p = pmask ? __ffs(pmask) - 1 : 31;
        uint64_t v = lane <= first_p ? (st & kPayload) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (pmask) break;
        pred -= 32;
      }
      if (lane == 0) st_status(status + tile, kFlagPre | (excl + agg));
    }
    if (lane == 0) {
      s_excl = excl;
      if (tile + 1 == ntiles) {
        const uint64_t tot = excl + agg;
        totals[0] = tot >> kUnitBits;
        totals[1] = (tot & ((1ull << kUnitBits) - 1)) << 8;
      }
    }
  }
  __syncthreads();
  return s_excl + s_warp[warp] + (incl - local);
}

__device__ __forceinline__ uint64_t next_tile(unsigned int* counter) {
  __shared__ unsigned int s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  return s_tile;
}

__global__ void __launch_bounds__(kThreads)
k_select_scan(TableDev dedup, const uint64_t* __restrict__ slot, const uint32_t* __restrict__ lens,
              uint64_t n, uint64_t* __restrict__ status, unsigned int* __restrict__ tile_counter,
              uint8_t* __restrict__ sel, uint64_t* owner,
              uint64_t* __restrict__ offsets, uint32_t* __restrict__ sel_list,
              uint64_t* __restrict__ totals, uint64_t* __restrict__ spec_next,
              const uint64_t* __restrict__ spec_cur, const uint8_t* __restrict__ arena,
              GridDev grid, uint8_t* __restrict__ staging) {
  griddep_wait();
  const uint64_t tile = next_tile(tile_counter);
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const uint64_t base = tile * kTile + uint64_t(threadIdx.x) * kItems;
  uint64_t val[kItems], own[kItems], local = 0;
  uint64_t s[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j)
    s[j] = base + j >= n ? ~0ull : slot ? slot[base + j] : owner[base + j];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    // slot == nullptr: the owners are already known (multi-rank, on demand)
    own[j] = s[j] == ~0ull ? ~0ull : slot ? dedup.vals[s[j]] : s[j];
    val[j] = own[j] == base + j ? (1ull << kUnitBits) | (lens[base + j] >> 8) : 0;
    local += val[j];
  }
  uint64_t run = tile_scan(local, tile, ntiles, status, totals);
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint64_t g = base + j;
    if (g < n) {
      const bool sl = val[j] != 0;
      sel[g] = sl;
      owner[g] = own[j];
      const uint64_t off = (run & ((1ull << kUnitBits) - 1)) << 8;
      offsets[g] = own[j] == ~0ull ? ~0ull : off;
      if (sl) sel_list[run >> kUnitBits] = static_cast<uint32_t>(g);
      if (spec_next) spec_next[g] = sl ? off : ~0ull;
    }
    run += val[j];
  }
  if (spec_cur) {
    // K3 fix-up fused (single GPU, speculative K1 layout): a selected chunk the
    // fused K1 did not already store at its final offset is copied from the
    // arena by the whole warp (rare: only when the layout changed)
    const int lane = threadIdx.x & 31;
    run = run - local;  // this thread's first exclusive prefix again
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const uint64_t g = base + j;
      const uint64_t off = (run & ((1ull << kUnitBits) - 1)) << 8;
      const bool need = g < n && val[j] != 0 && spec_cur[g] != off;
      unsigned m = __ballot_sync(0xffffffffu, need);
      while (m) {
        const int q = __ffs(m) - 1;
        m &= m - 1;
        const uint64_t gq = __shfl_sync(0xffffffffu, g, q);
        const uint64_t oq = __shfl_sync(0xffffffffu, off, q);
        warp_copy(staging + oq, chunk_ptr(arena, grid, gq), lens[gq], lane);
      }
      run += val[j];
    }
  }
}

// Shard scan for writer `me`: offsets of the chunks `me` writes, in canonical
// order (its shard of the global image); with write_list, my_list[k] = local
// chunk index of the k-th chunk of the shard and my_off[k] its offset.
__global__ void __launch_bounds__(kThreads)
k_shard_scan(const int32_t* __restrict__ writer, const uint32_t* __restrict__ glens, uint64_t n,
             uint64_t maxn, int32_t me, int write_list, uint64_t* __restrict__ status,
             unsigned int* __restrict__ tile_counter, uint64_t* __restrict__ shard_off,
             uint32_t* __restrict__ my_list, uint64_t* __restrict__ my_off,
             uint64_t* __restrict__ totals, TableDev clear, FixUp fix) {
  griddep_wait();
  if (clear.keys) {  // the dedup table the previous kernel consumed: left empty
    const uint64_t tab = clear.mask + 2;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < tab;
         i += uint64_t(gridDim.x) * blockDim.x) {
      clear.keys[i] = kEmptyKey;
      clear.vals[i] = ~0ull;
    }
  }
  const uint64_t tile = next_tile(tile_counter);
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const uint64_t base = tile * kTile + uint64_t(threadIdx.x) * kItems;
  uint64_t val[kItems], local = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint64_t g = base + j;
    val[j] = (g < n && writer[g] == me) ? (1ull << kUnitBits) | (glens[g] >> 8) : 0;
    local += val[j];
  }
  uint64_t run = tile_scan(local, tile, ntiles, status, totals);
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint64_t g = base + j;
    if (g < n) {
      const uint64_t off = (run & ((1ull << kUnitBits) - 1)) << 8;
      if (val[j]) {
        shard_off[g] = off;
        if (write_list) {
          my_list[run >> kUnitBits] = static_cast<uint32_t>(g % maxn);
          my_off[run >> kUnitBits] = off;
        }
      }
    }
    run += val[j];
  }
  if (fix.staging) {
    // K3 fix-up fused (speculative K1 layout): this rank's chunks whose final
    // shard offset differs from the speculated one are copied from the arena
    // (local chunk g % maxn holds the bytes: same digest and length)
    const int lane = threadIdx.x & 31;
    run = run - local;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const uint64_t g = base + j;
      const uint64_t off = (run & ((1ull << kUnitBits) - 1)) << 8;
      const uint64_t i = g % maxn;
      bool need = false;
      if (val[j]) {
        if (fix.spec_next) fix.spec_next[i] = off;
        need = fix.spec_cur[i] != off;
      }
      unsigned m = __ballot_sync(0xffffffffu, need);
      while (m) {
        const int q = __ffs(m) - 1;
        m &= m - 1;
        const uint64_t iq = __shfl_sync(0xffffffffu, i, q);
        const uint64_t oq = __shfl_sync(0xffffffffu, off, q);
        warp_copy(fix.staging + oq, chunk_ptr(fix.arena, fix.grid, iq), glens[iq + uint64_t(me) * maxn],
                  lane);
      }
      run += val[j];
    }
  }
}

// Duplicates point at their owner's staged bytes (restore source). The same
// pass resets the dedup table and the scan state the selection just consumed,
// so the next selection starts without a clear kernel or memset.
__global__ void k_resolve_dups(const uint8_t* __restrict__ sel, const uint64_t* __restrict__ owner,
                               uint64_t* __restrict__ offsets, uint64_t n, TableDev clear,
                               uint64_t* __restrict__ scan_state, uint64_t clear_words) {
  griddep_wait();
  const uint64_t tab = clear.keys ? clear.mask + 2 : 0;
  const uint64_t end = n > tab ? (n > clear_words ? n : clear_words)
                               : (tab > clear_words ? tab : clear_words);
  for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < end;
       g += uint64_t(gridDim.x) * blockDim.x) {
    if (g < n) {
      const uint64_t o = owner[g];
      if (!sel[g] && o != ~0ull) offsets[g] = offsets[o];
    }
    if (g < tab) {
      clear.keys[g] = kEmptyKey;
      clear.vals[g] = ~0ull;
    }
    if (g < clear_words) scan_state[g] = 0;
  }
}

// Small selections (n <= kSmallMax, e.g. C1's 4096 chunks): the insert, the
// scan, the K3 fix-up, the duplicate resolution and the table clean-up of the
// three-kernel path (k_dedup_insert -> k_select_scan -> k_resolve_dups) in ONE
// launch of ceil(n / 1024) CTAs, one chunk per thread, phases separated by a
// software grid barrier — at this size the three launches and their
// dependency gaps cost more than the work, and one chunk per thread keeps
// every phase at one or two memory round trips. Same outputs bit for bit.
// Scratch: sc[0] = barrier arrivals, sc[1 + b] = CTA b's aggregate; the scan
// state is zero on entry (the selection's invariant) and left zero on exit.
constexpr int kSmallThreads = 1024;
constexpr int kSmallCtas = 8;
constexpr uint64_t kSmallMax = uint64_t(kSmallThreads) * kSmallCtas;

__device__ __forceinline__ void grid_wait(unsigned long long* cnt, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(cnt, 1ull);
    while (ld_status(reinterpret_cast<const uint64_t*>(cnt)) < target) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSmallThreads, 1)
k_select_small(TableDev dedup, TableDev known, int use_known, const uint64_t* __restrict__ dig,
               const uint32_t* __restrict__ lens, uint64_t n, uint8_t* __restrict__ sel,
               uint64_t* owner, uint64_t* offsets, uint32_t* __restrict__ sel_list,
               uint64_t* __restrict__ totals, uint64_t* __restrict__ spec_next,
               const uint64_t* __restrict__ spec_cur, const uint8_t* __restrict__ arena,
               GridDev grid, uint8_t* __restrict__ staging, uint64_t* sc) {
  __shared__ uint64_t s_warp[kSmallThreads / 32];
  __shared__ uint64_t s_pre;
  griddep_wait();
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(sc);
  const unsigned G = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t g = uint64_t(blockIdx.x) * kSmallThreads + threadIdx.x;
  // phase 1: insert (first occurrence by atomicMin), known-set probe
  uint64_t slot = ~0ull;
  uint32_t len = 0;
  if (g < n) {
    len = lens[g];
    if (len != 0) {
      const unsigned long long d = dig[g];
      if (!(use_known && table_find(known, d) != ~0ull)) {
        slot = table_find_or_insert(dedup, d);
        atomicMin(dedup.vals + slot, static_cast<unsigned long long>(g));
      }
    }
  }
  grid_wait(cnt, G);
  // phase 2: owner, CTA scan, cross-CTA prefix from the published aggregates
  const uint64_t own =
      slot == ~0ull ? ~0ull : __ldcg(reinterpret_cast<const unsigned long long*>(dedup.vals) + slot);
  const uint64_t val = own == g ? (1ull << kUnitBits) | (len >> 8) : 0;
  uint64_t incl = val;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint64_t w = s_warp[lane];
    uint64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    s_warp[lane] = wi - w;
    if (lane == 31) st_status(sc + 1 + blockIdx.x, wi);
  }
  grid_wait(cnt, 2ull * G);
  if (threadIdx.x == 0) {
    uint64_t pre = 0, all = 0;
    for (unsigned b = 0; b < G; ++b) {
      const uint64_t a = ld_status(sc + 1 + b);
      if (b < blockIdx.x) pre += a;
      all += a;
    }
    s_pre = pre;
    if (blockIdx.x == G - 1) {
      totals[0] = all >> kUnitBits;
      totals[1] = (all & ((1ull << kUnitBits) - 1)) << 8;
    }
  }
  __syncthreads();
  const uint64_t run = s_pre + s_warp[warp] + (incl - val);
  const uint64_t off = (run & ((1ull << kUnitBits) - 1)) << 8;
  const bool sl = val != 0;
  if (g < n) {
    sel[g] = sl;
    owner[g] = own;
    offsets[g] = own == ~0ull ? ~0ull : off;
    if (sl) sel_list[run >> kUnitBits] = static_cast<uint32_t>(g);
    if (spec_next) spec_next[g] = sl ? off : ~0ull;
  }
  if (spec_cur) {  // K3 fix-up (see k_select_scan)
    const bool need = g < n && sl && spec_cur[g] != off;
    unsigned m = __ballot_sync(0xffffffffu, need);
    while (m) {
      const int q = __ffs(m) - 1;
      m &= m - 1;
      const uint64_t gq = __shfl_sync(0xffffffffu, g, q);
      const uint64_t oq = __shfl_sync(0xffffffffu, off, q);
      warp_copy(staging + oq, chunk_ptr(arena, grid, gq), lens[gq], lane);
    }
  }
  grid_wait(cnt, 3ull * G);
  // phase 3: duplicates point at their owner's bytes; the table and the
  // scratch go back to empty
  if (g < n && !sl && own != ~0ull)
    offsets[g] = __ldcg(reinterpret_cast<const unsigned long long*>(offsets) + own);
  for (uint64_t t = g; t < dedup.mask + 2; t += uint64_t(G) * kSmallThreads) {
    dedup.keys[t] = kEmptyKey;
    dedup.vals[t] = ~0ull;
  }
  if (g < G) sc[1 + g] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    // the last CTA out resets the counter (nobody reads it after its increment)
    if (atomicAdd(cnt, 1ull) == 4ull * G - 1) st_status(sc, 0);
  }
}

// Selections of up to 4096 chunks (C1): the whole K2 in ONE thread-block
// CLUSTER (one CTA per SM) — no global
// atomics, no grid barriers, nothing to clean up afterwards (the global dedup
// table and scan state are not touched; same outputs bit for bit as
// k_select_small / the three-kernel path). The first-occurrence table is
// partitioned across the CTAs' shared memories (distributed shared memory:
// slot s lives in CTA s / LOCAL), so the inserts' shared-memory atomics and
// the outputs' loads / stores spread over CTAS SMs; the scan carries CTA
// totals through DSMEM, and cluster barriers replace grid barriers. Table load
// <= 1/4: an insert is a chain of dependent DSMEM atomics along its probe
// sequence, so the longest linear-probing run, not the atomic throughput, sets
// the phase time (at load 1/2 the 4096-chunk insert took ~6 us, at 1/8 ~1 us).
// Chunk g = rank * THREADS * ITEMS + j * THREADS + t: coalesced. (A one-CTA
// version with the table in one shared memory took 11-14 us on C1 — one SM's
// atomic and load-store throughput — against ~7.3 us for 8 CTAs.)
template <int CTAS, int THREADS, int ITEMS, uint32_t LOCAL>
struct ClCfg {
  static constexpr uint32_t kPer = uint32_t(THREADS) * ITEMS;  // chunks per CTA
  static constexpr uint32_t kMax = uint32_t(CTAS) * kPer;
  static constexpr uint32_t kSlots = uint32_t(CTAS) * LOCAL;
  static constexpr size_t kSmem = size_t(LOCAL) * 12 + size_t(kPer) * 4;  // keys, mins, fix list
  static_assert((kSlots & (kSlots - 1)) == 0 && kSlots >= 4 * kMax, "table load <= 1/4");
};
// n <= 4096, load 1/8. (Measured and dropped: 16 CTAs x 1024 threads x 4
// chunks at load 1/4 for n <= 65536 — 26.7 us on C3's 64970 chunks and 30 us
// on a C2 rank's 32960 against 12 / 22.5 us for the three-kernel path: four
// dependent probe chains per thread in sequence.)
using ClSmall = ClCfg<8, 512, 1, 4096>;

template <int CTAS, int THREADS, int ITEMS, uint32_t LOCAL>
__global__ void __launch_bounds__(THREADS, 1)
k_select_cluster(TableDev known, int use_known, const uint64_t* __restrict__ dig,
                 const uint32_t* __restrict__ lens, uint32_t n, uint8_t* __restrict__ sel,
                 uint64_t* __restrict__ owner, uint64_t* __restrict__ offsets,
                 uint32_t* __restrict__ sel_list, uint64_t* __restrict__ totals,
                 uint64_t* __restrict__ spec_next, const uint64_t* __restrict__ spec_cur,
                 const uint8_t* __restrict__ arena, GridDev grid, uint8_t* __restrict__ staging) {
  using C = ClCfg<CTAS, THREADS, ITEMS, LOCAL>;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) unsigned long long keys[];  // [LOCAL]
  uint32_t* mins = reinterpret_cast<uint32_t*>(keys + LOCAL);
  uint32_t* s_fix = mins + LOCAL;                             // [kPer]
  __shared__ uint64_t s_warp[THREADS / 32];
  __shared__ uint64_t s_tot;
  __shared__ uint32_t s_nfix;
  __shared__ uint32_t s_empty_min;  // first occurrence of the kEmptyKey digest (CTA 0)
  __shared__ int s_dup;
  const uint32_t t = threadIdx.x;
  const uint32_t rank = cl.block_rank();
  const int lane = t & 31, warp = t >> 5;
  for (uint32_t i = t; i < LOCAL; i += THREADS) {
    keys[i] = kEmptyKey;
    mins[i] = 0xffffffffu;
  }
  if (t == 0) {
    s_nfix = 0;
    s_dup = 0;
    s_empty_min = 0xffffffffu;
  }
  // split cluster barrier: the partitions' initialisation is published now,
  // the wait (before the first remote atomic) hides behind the input loads
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  griddep_wait();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint32_t len[ITEMS];
  unsigned long long d[ITEMS];
  uint64_t sc[ITEMS];
  bool cand[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t g = rank * C::kPer + j * THREADS + t;
    len[j] = g < n ? __ldcg(lens + g) : 0;
    d[j] = g < n ? __ldcg(reinterpret_cast<const unsigned long long*>(dig) + g) : 0;
    sc[j] = (spec_cur && g < n) ? __ldg(spec_cur + g) : 0;
  }
#pragma unroll
  for (int j = 0; j < ITEMS; ++j)
    cand[j] = len[j] != 0 && !(use_known && table_find(known, d[j]) != ~0ull);
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // partitions ready
  // insert: a CAS claims a free slot (the claimer stores its index), an equal
  // key makes the chunk a duplicate (rare), resolved by atomicMin below
  uint32_t slot[ITEMS];
  uint32_t dup = 0;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    slot[j] = 0xffffffffu;
    if (!cand[j]) continue;
    const uint32_t g = rank * C::kPer + j * THREADS + t;
    if (d[j] == kEmptyKey) {  // a legal digest: its own word in CTA 0
      slot[j] = C::kSlots;
      dup |= 1u << j;
      continue;
    }
    uint32_t h = uint32_t(tmix64(d[j])) & (C::kSlots - 1);
    for (;;) {
      unsigned long long* k = cl.map_shared_rank(keys, h / LOCAL) + (h % LOCAL);
      const unsigned long long prev = atomicCAS(k, kEmptyKey, d[j]);
      if (prev == kEmptyKey) {
        *(cl.map_shared_rank(mins, h / LOCAL) + (h % LOCAL)) = g;
        break;
      }
      if (prev == d[j]) {
        dup |= 1u << j;
        break;
      }
      h = (h + 1) & (C::kSlots - 1);
    }
    slot[j] = h;
  }
  if (dup) s_dup = 1;
  cl.sync();  // claims visible; every CTA's s_dup final
  int any_dup = 0;
  for (uint32_t r = 0; r < CTAS; ++r) any_dup |= *cl.map_shared_rank(&s_dup, r);
  if (any_dup) {
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if (dup >> j & 1) {
        const uint32_t g = rank * C::kPer + j * THREADS + t;
        uint32_t* m = slot[j] == C::kSlots
                          ? cl.map_shared_rank(&s_empty_min, 0)
                          : cl.map_shared_rank(mins, slot[j] / LOCAL) + (slot[j] % LOCAL);
        atomicMin(m, g);
      }
    cl.sync();
  }
  // owners, then the CTA-local scan (ITEMS block scans with a carry)
  uint64_t own[ITEMS], run[ITEMS];
  bool sl[ITEMS];
  uint64_t carry = 0;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t g = rank * C::kPer + j * THREADS + t;
    own[j] = slot[j] == 0xffffffffu ? ~0ull
             : slot[j] == C::kSlots
                 ? uint64_t(*cl.map_shared_rank(&s_empty_min, 0))
                 : uint64_t(*(cl.map_shared_rank(mins, slot[j] / LOCAL) + (slot[j] % LOCAL)));
    sl[j] = own[j] == g;
    const uint64_t val = sl[j] ? (1ull << kUnitBits) | (len[j] >> 8) : 0;
    uint64_t incl = val;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint64_t w = lane < THREADS / 32 ? s_warp[lane] : 0;
      uint64_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      if (lane < THREADS / 32) s_warp[lane] = wi - w;
      if (lane == THREADS / 32 - 1) s_tot = wi;
    }
    __syncthreads();
    run[j] = carry + s_warp[warp] + incl - val;
    carry += s_tot;
    __syncthreads();  // s_warp / s_tot reused
  }
  if (t == 0) s_tot = carry;
  cl.sync();  // every CTA's total published
  uint64_t pre = 0, all = 0;
  for (uint32_t r = 0; r < CTAS; ++r) {
    const uint64_t a = *cl.map_shared_rank(&s_tot, r);
    if (r < rank) pre += a;
    all += a;
  }
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t g = rank * C::kPer + j * THREADS + t;
    if (g >= n) continue;
    const uint64_t r = pre + run[j];
    const uint64_t off = (r & ((1ull << kUnitBits) - 1)) << 8;
    sel[g] = sl[j];
    owner[g] = own[j];
    if (sl[j]) {
      offsets[g] = off;
      sel_list[r >> kUnitBits] = g;
      if (spec_cur && sc[j] != off) s_fix[atomicAdd(&s_nfix, 1u)] = g;  // K3 fix-up
    } else if (own[j] == ~0ull) {
      offsets[g] = ~0ull;
    }
    if (spec_next) spec_next[g] = sl[j] ? off : ~0ull;
  }
  if (rank == CTAS - 1 && t == 0) {
    totals[0] = all >> kUnitBits;
    totals[1] = (all & ((1ull << kUnitBits) - 1)) << 8;
  }
  if (any_dup) {
    cl.sync();  // the owners' offsets (global, written above) visible cluster-wide
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const uint32_t g = rank * C::kPer + j * THREADS + t;
      if (g < n && !sl[j] && own[j] != ~0ull) offsets[g] = __ldcg(offsets + own[j]);
    }
  }
  // last remote shared-memory access done: arrive now, wait only before exit
  // (no CTA may leave while another can still read its shared memory)
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  __syncthreads();  // this CTA's fix-up list and offsets complete
  const uint32_t nfix = s_nfix;
  for (uint32_t q = warp; q < nfix; q += THREADS / 32) {
    const uint32_t gq = s_fix[q];
    warp_copy(staging + __ldcg(offsets + gq), chunk_ptr(arena, grid, gq), lens[gq], lane);
  }
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

unsigned grid_for(uint64_t n, unsigned threads, unsigned cap) {
  uint64_t b = (n + threads - 1) / threads;
  if (b > cap) b = cap;
  return b == 0 ? 1u : unsigned(b);
}

}  // namespace

uint64_t scan_state_words(uint64_t n) { return (n + kTile - 1) / kTile + 1; }

int launch_table_clear(TableDev t, cudaStream_t s) {
  k_table_clear<<<grid_for(t.mask + 2, 256, 148 * 16), 256, 0, s>>>(t);
  return 1;
}

int launch_table_insert_min(TableDev t, const uint64_t* keys, uint64_t n, uint64_t index_base,
                            cudaStream_t s) {
  if (n == 0) return 0;
  k_table_insert_min<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(t, keys, n, index_base);
  return 1;
}

int launch_dedup_insert(TableDev dedup, TableDev known, bool use_known, const uint64_t* dig,
                        const uint32_t* lens, uint64_t n, uint64_t* slot, cudaStream_t s) {
  if (n == 0) return 0;
  launch_pdl(k_dedup_insert, grid_for(n, 128, 148 * 32), 128, 0, s, dedup, known,
             use_known ? 1 : 0, dig, lens, n, slot);
  return 1;
}

int launch_select(TableDev dedup, const uint64_t* slot, const uint32_t* lens, uint64_t n,
                  uint64_t* scan_state, uint8_t* sel, uint64_t* owner, uint64_t* offsets,
                  uint32_t* sel_list, uint64_t* totals, uint64_t* spec_next, cudaStream_t s,
                  const uint64_t* spec_cur, const uint8_t* arena, const GridDev* grid,
                  uint8_t* staging) {
  const uint64_t tiles = (n + kTile - 1) / kTile;
  if (n == 0) {
    cudaMemsetAsync(totals, 0, 2 * sizeof(uint64_t), s);
    return 0;
  }
  launch_pdl(k_select_scan, unsigned(tiles), kThreads, 0, s, dedup, slot, lens, n, scan_state,
             reinterpret_cast<unsigned int*>(scan_state + tiles), sel, owner, offsets, sel_list,
             totals, spec_next, spec_cur, arena, grid ? *grid : GridDev{}, staging);
  return 1;
}

bool select_small_ok(uint64_t n) { return n > 0 && n <= kSmallMax; }
// the 16-CTA cluster needs 16 free SMs of one GPC (non-portable size):
// checked once per device, else the larger selections keep the other paths
template <class C, int CTAS, int THREADS, int ITEMS, uint32_t LOCAL>
bool cluster_fits() {
  static uint64_t done = 0;
  static int ok[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  once_per_device(done, [&] {
    auto k = k_select_cluster<CTAS, THREADS, ITEMS, LOCAL>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem));
    if (CTAS > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = CTAS;
    cfg.blockDim = THREADS;
    cfg.dynamicSmemBytes = C::kSmem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CTAS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k, &cfg);
    if (e != cudaSuccess) cudaGetLastError();
    if (dev >= 0 && dev < 64) ok[dev] = e == cudaSuccess && nc > 0;
  });
  return dev >= 0 && dev < 64 && ok[dev];
}

bool select_cluster_ok(uint64_t n) {
  return n > 0 && n <= ClSmall::kMax && cluster_fits<ClSmall, 8, 512, 1, 4096>();
}

int launch_select_cluster(TableDev known, bool use_known, const uint64_t* dig,
                          const uint32_t* lens, uint64_t n, uint8_t* sel, uint64_t* owner,
                          uint64_t* offsets, uint32_t* sel_list, uint64_t* totals,
                          uint64_t* spec_next, cudaStream_t s, const uint64_t* spec_cur,
                          const uint8_t* arena, const GridDev* grid, uint8_t* staging) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = 8;
  cfg.blockDim = 512;
  cfg.dynamicSmemBytes = ClSmall::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 8;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, k_select_cluster<8, 512, 1, 4096>, known, use_known ? 1 : 0, dig, lens,
                     uint32_t(n), sel, owner, offsets, sel_list, totals, spec_next, spec_cur,
                     arena, grid ? *grid : GridDev{}, staging);
  return 1;
}

int launch_select_small(TableDev dedup, TableDev known, bool use_known, const uint64_t* dig,
                        const uint32_t* lens, uint64_t n, uint8_t* sel, uint64_t* owner,
                        uint64_t* offsets, uint32_t* sel_list, uint64_t* totals,
                        uint64_t* spec_next, cudaStream_t s, uint64_t* scratch,
                        const uint64_t* spec_cur, const uint8_t* arena, const GridDev* grid,
                        uint8_t* staging) {
  const unsigned ctas = unsigned((n + kSmallThreads - 1) / kSmallThreads);
  launch_pdl(k_select_small, ctas, kSmallThreads, 0, s, dedup, known, use_known ? 1 : 0, dig, lens,
             n, sel, owner, offsets, sel_list, totals, spec_next, spec_cur, arena,
             grid ? *grid : GridDev{}, staging, scratch);
  return 1;
}

int launch_shard_scan(const int32_t* writer, const uint32_t* glens, uint32_t nranks, uint64_t maxn,
                      int32_t q, bool write_list, uint64_t* scan_state, uint64_t* shard_off,
                      uint32_t* my_list, uint64_t* my_off, uint64_t* totals, cudaStream_t s) {
  const uint64_t n = uint64_t(nranks) * maxn;
  const uint64_t tiles = (n + kTile - 1) / kTile;
  cudaMemsetAsync(scan_state, 0, (tiles + 1) * sizeof(uint64_t), s);
  if (n == 0) {
    cudaMemsetAsync(totals, 0, 2 * sizeof(uint64_t), s);
    return 0;
  }
  k_shard_scan<<<unsigned(tiles), kThreads, 0, s>>>(
      writer, glens, n, maxn, q, write_list ? 1 : 0, scan_state,
      reinterpret_cast<unsigned int*>(scan_state + tiles), shard_off, my_list, my_off, totals,
      TableDev{}, FixUp{});
  return 1;
}

int launch_select_stripe(TableDev dedup, const uint64_t* slot, const uint64_t* gdig,
                         const uint32_t* glens, uint32_t nranks, uint64_t maxn, int32_t me,
                         uint8_t* sel, uint64_t* owner, int32_t* writer, uint64_t* scan_state,
                         uint64_t* shard_off, uint32_t* my_list, uint64_t* my_off,
                         uint64_t* totals, cudaStream_t s, const FixUp& fix) {
  const uint64_t n = uint64_t(nranks) * maxn;
  const uint64_t tiles = (n + kTile - 1) / kTile;
  if (n == 0) {
    cudaMemsetAsync(totals, 0, 2 * sizeof(uint64_t), s);
    return 0;
  }
  launch_pdl(k_select_stripe, grid_for(n, 256, 148 * 16), 256, 0, s, dedup, slot, gdig, glens,
             nranks, maxn, sel, owner, writer, scan_state, tiles + 1,
             fix.staging ? fix.spec_next : nullptr, fix.nlocal);
  launch_pdl(k_shard_scan, unsigned(tiles), kThreads, 0, s, writer, glens, n, maxn, me, 1,
             scan_state, reinterpret_cast<unsigned int*>(scan_state + tiles), shard_off, my_list,
             my_off, totals, dedup, fix);
  return 2;
}

int launch_resolve_dups(const uint8_t* sel, const uint64_t* owner, uint64_t* offsets, uint64_t n,
                        TableDev clear, uint64_t* scan_state, uint64_t clear_words,
                        cudaStream_t s) {
  const uint64_t tab = clear.keys ? clear.mask + 2 : 0;
  const uint64_t end = std::max(n, std::max(tab, clear_words));
  if (end == 0) return 0;
  launch_pdl(k_resolve_dups, grid_for(end, 256, 148 * 8), 256, 0, s, sel, owner, offsets, n,
             clear, scan_state, clear_words);
  return 1;
}

}  // namespace snap
