// k_select.cu — K2: dedup table + dirty test + deterministic stream-compaction
// offsets.
//
// Reference semantics (build_manifest, ckpt.cpp:97,147-167; BlobStore::put,
// ckpt.cpp:16-21): walking chunks in canonical (rank, slot, chunk) order, a
// chunk is staged iff its digest was not seen earlier in this snapshot AND
// is not already in the store (the "known" set). Order independence on the
// GPU: the dedup table stores min(chunk index) per digest (atomicMin), so the
// first occurrence is found without any ordering between threads; staging
// offsets come from a single-pass decoupled look-back scan over canonical
// chunk order, so the staging image is bit-identical run to run.
#include <cuda_runtime.h>

#include "snap_internal.h"

namespace snap {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// Slot of key k; the digest value equal to kEmptyKey lives in the extra slot
// at index mask + 1 so every 64-bit digest is representable exactly.
__device__ __forceinline__ uint64_t table_find_or_insert(TableDev t, unsigned long long k) {
  if (k == kEmptyKey) return t.mask + 1;
  uint64_t h = mix64(k) & t.mask;
  for (;;) {
    const unsigned long long prev = atomicCAS(t.keys + h, kEmptyKey, k);
    if (prev == kEmptyKey || prev == k) return h;
    h = (h + 1) & t.mask;
  }
}
// Returns slot or UINT64_MAX when absent.
__device__ __forceinline__ uint64_t table_find(TableDev t, unsigned long long k) {
  if (k == kEmptyKey) return t.vals[t.mask + 1] != ~0ull ? t.mask + 1 : ~0ull;
  uint64_t h = mix64(k) & t.mask;
  for (;;) {
    const unsigned long long cur = t.keys[h];
    if (cur == k) return h;
    if (cur == kEmptyKey) return ~0ull;
    h = (h + 1) & t.mask;
  }
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

// ---- selection + decoupled look-back scan ---------------------------------
// Status word per tile: flag (2 bits) | chunk count (26 bits) | 256-byte units (36 bits).
constexpr int kThreads = 256;
constexpr int kItems = 8;
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

__global__ void __launch_bounds__(kThreads)
k_select_scan(TableDev dedup, TableDev known, int use_known, const uint64_t* __restrict__ dig,
              const uint32_t* __restrict__ lens, uint64_t n, uint64_t* __restrict__ status,
              unsigned int* __restrict__ tile_counter, uint8_t* __restrict__ sel,
              uint64_t* __restrict__ owner, uint64_t* __restrict__ offsets,
              uint32_t* __restrict__ sel_list, uint64_t* __restrict__ totals) {
  __shared__ unsigned int s_tile;
  __shared__ uint64_t s_warp[kThreads / 32];
  __shared__ uint64_t s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t base = tile * kTile + uint64_t(threadIdx.x) * kItems;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  uint64_t val[kItems];
  uint64_t own[kItems];
  uint64_t local = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint64_t g = base + j;
    val[j] = 0;
    own[j] = ~0ull;
    if (g < n) {
      const unsigned long long d = dig[g];
      bool is_known = false;
      if (use_known) is_known = table_find(known, d) != ~0ull;
      if (!is_known) {
        const uint64_t s = table_find(dedup, d);
        own[j] = dedup.vals[s];
        if (own[j] == g) val[j] = (1ull << kUnitBits) | (lens[g] >> 8);
      }
    }
    local += val[j];
  }
  // block-wide exclusive scan of per-thread sums
  uint64_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = lane < kThreads / 32 ? s_warp[lane] : 0;
    uint64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    const uint64_t agg = __shfl_sync(0xffffffffu, wi, kThreads / 32 - 1);
    if (lane < kThreads / 32) s_warp[lane] = wi - w;  // exclusive per warp
    // decoupled look-back over predecessor tiles
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
      if ((tile + 1) * kTile >= n) {  // last tile publishes the totals
        const uint64_t tot = excl + agg;
        totals[0] = tot >> kUnitBits;
        totals[1] = (tot & ((1ull << kUnitBits) - 1)) << 8;
      }
    }
  }
  __syncthreads();
  uint64_t run = s_excl + s_warp[warp] + (incl - local);
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint64_t g = base + j;
    if (g < n) {
      const bool s = val[j] != 0;
      sel[g] = s;
      owner[g] = own[j];
      offsets[g] = own[j] == ~0ull ? ~0ull : (run & ((1ull << kUnitBits) - 1)) << 8;
      if (s) sel_list[run >> kUnitBits] = static_cast<uint32_t>(g);
    }
    run += val[j];
  }
}

// Duplicates point at their owner's staged bytes (restore source).
__global__ void k_resolve_dups(const uint8_t* __restrict__ sel, const uint64_t* __restrict__ owner,
                               uint64_t* __restrict__ offsets, uint64_t n) {
  for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < n;
       g += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t o = owner[g];
    if (!sel[g] && o != ~0ull) offsets[g] = offsets[o];
  }
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

int launch_select(TableDev dedup, TableDev known, bool use_known, const uint64_t* dig,
                  const uint32_t* lens, uint64_t n, uint64_t* scan_state, uint8_t* sel,
                  uint64_t* owner, uint64_t* offsets, uint32_t* sel_list, uint64_t* totals,
                  cudaStream_t s) {
  const uint64_t tiles = (n + kTile - 1) / kTile;
  // scan_state = [tiles] status words + 1 word of tile counter
  cudaMemsetAsync(scan_state, 0, (tiles + 1) * sizeof(uint64_t), s);
  if (n == 0) {
    cudaMemsetAsync(totals, 0, 2 * sizeof(uint64_t), s);
    return 0;
  }
  k_select_scan<<<unsigned(tiles), kThreads, 0, s>>>(
      dedup, known, use_known ? 1 : 0, dig, lens, n, scan_state,
      reinterpret_cast<unsigned int*>(scan_state + tiles), sel, owner, offsets, sel_list, totals);
  return 1;
}

int launch_resolve_dups(const uint8_t* sel, const uint64_t* owner, uint64_t* offsets, uint64_t n,
                        cudaStream_t s) {
  if (n == 0) return 0;
  k_resolve_dups<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(sel, owner, offsets, n);
  return 1;
}

}  // namespace snap
