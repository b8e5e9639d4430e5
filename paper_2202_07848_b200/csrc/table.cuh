// table.cuh — open-addressing digest tables shared by the K2 (dedup / known
// set) and splice (chunk cache index) kernels. Power-of-two capacity, linear
// probing, key kEmptyKey = free; the digest value equal to kEmptyKey lives in
// the extra slot mask + 1, so every 64-bit digest is representable exactly.
#pragma once

#include "snap_internal.h"

namespace snap {

// PDL: wait until the previous kernel of the stream has completed and its
// writes are visible (no-op without a programmatic dependency)
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}


__device__ __forceinline__ uint64_t tmix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t table_find_or_insert(TableDev t, unsigned long long k) {
  if (k == kEmptyKey) return t.mask + 1;
  uint64_t h = tmix64(k) & t.mask;
  for (;;) {
    const unsigned long long prev = atomicCAS(t.keys + h, kEmptyKey, k);
    if (prev == kEmptyKey || prev == k) return h;
    h = (h + 1) & t.mask;
  }
}

// Slot of k, or UINT64_MAX when absent (the kEmptyKey slot counts as present
// once its value was set).
__device__ __forceinline__ uint64_t table_find(TableDev t, unsigned long long k) {
  if (k == kEmptyKey) return t.vals[t.mask + 1] != ~0ull ? t.mask + 1 : ~0ull;
  uint64_t h = tmix64(k) & t.mask;
  for (;;) {
    const unsigned long long cur = t.keys[h];
    if (cur == k) return h;
    if (cur == kEmptyKey) return ~0ull;
    h = (h + 1) & t.mask;
  }
}

// Arena offset and byte length of chunk gc: the grid's per-chunk maps when it
// carries them (one round of independent loads), else the buffer search.
__device__ __forceinline__ void chunk_loc(const GridDev& g, uint64_t gc, uint64_t& addr,
                                          uint32_t& len) {
  if (g.chunk_addr) {
    addr = __ldg(g.chunk_addr + gc);
    len = __ldg(g.chunk_len + gc);
    return;
  }
  uint32_t b;
  if (g.chunk_buf) {
    b = __ldg(g.chunk_buf + gc);
  } else {
    uint32_t lo = 0, hi = g.nbufs;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(g.cstart + mid) <= gc) lo = mid; else hi = mid;
    }
    b = lo;
  }
  const uint64_t off = (gc - __ldg(g.cstart + b)) << g.chunk_shift;
  const uint64_t rem = __ldg(g.bytes + b) - off;
  addr = __ldg(g.addr + b) + off;
  len = static_cast<uint32_t>(rem < (1ull << g.chunk_shift) ? rem : (1ull << g.chunk_shift));
}

// K1: store one finished chunk digest locally and, with the fused exchange, into
// every rank's gathered vector (8-byte NVLink stores, fire and forget).
__device__ __forceinline__ void k1_store_digest(const GridDev& g, uint64_t chunk, uint64_t d,
                                                uint64_t* chunk_dig) {
  chunk_dig[chunk] = d;
  if (g.expect != nullptr && g.expect[chunk] != d) {
    atomicAdd(g.nbad, 1ull);
    if (g.bad_flag) *reinterpret_cast<volatile unsigned int*>(g.bad_flag) = 1u;
  }
  if (g.xdig != nullptr)
    for (uint32_t q = 0; q < g.xn; ++q) g.xdig[q][g.xoff + chunk] = d;
}

// The K2 insert of one finished chunk digest, done by K1 itself on the
// single-GPU snapshot path (k_dedup_insert's body): known-set probe,
// first-occurrence atomicMin, slot record.
__device__ __forceinline__ void k1_insert(const GridDev& g, uint64_t chunk, uint64_t d) {
  uint64_t s = ~0ull;
  if (!(g.kn_use && table_find(g.kn, d) != ~0ull)) {
    s = table_find_or_insert(g.dd, d);
    atomicMin(g.dd.vals + s, static_cast<unsigned long long>(chunk));
  }
  g.dd_slot[chunk] = s;
}

}  // namespace snap
