// k_hash_tma.cu — K1 hash-only with TMA tensor loads (used when no
// speculative stores are needed: incremental snapshots, splice swap-out
// digests, restore verification).
//
// Same lane = page-chain scheme as k_hash.cu, but a warp's stage fill is ONE
// instruction: for a "regular" task (32 full, contiguous 4 KiB pages of one
// buffer) an elected lane issues cp.async.bulk.tensor.2d with a box of
// 32 pages x 128 B from the buffer's tensor map (rows = pages, pitch 4 KiB);
// the hardware SWIZZLE_128B layout is exactly the XOR layout the hash lanes
// read (16-B unit u of page j at u ^ (j & 7)), and completion is counted in
// bytes on one mbarrier per stage. Irregular tasks (buffer edges, tail pages)
// use one 1D bulk copy per valid page slab (unswizzled layout) on the same
// barrier. This removes the per-lane cp.async address math that costs ~1.2
// instructions per hashed byte in the cp.async kernel.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>

#include "snap_internal.h"
#include "table.cuh"

namespace snap {
namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kSlab = 128;
constexpr int kStageBytes = 32 * kSlab;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint4 ld_shared16(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx)
               : "memory");
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
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, int x, int y,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(tmap), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// FNV-1a byte step (see k_hash.cu for the instruction-level derivation)
__device__ __forceinline__ void fnv_step(uint32_t& lo, uint32_t& hi, uint32_t b) {
  const uint32_t x = lo ^ (b & 0xffu);
  const uint64_t t = static_cast<uint64_t>(x) * kFnvPrimeLo;
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
__device__ __forceinline__ uint32_t find_buf(const GridDev& g, uint64_t gc) {
  if (g.chunk_buf) return __ldg(g.chunk_buf + gc);
  uint32_t lo = 0, hi = g.nbufs;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(g.cstart + mid) <= gc) lo = mid; else hi = mid;
  }
  return lo;
}

// 4 KiB pages (PS = 12) only: the tensor maps describe a buffer as rows of 4 KiB.
template <int WARPS, int ST>
__global__ void __launch_bounds__(WARPS * 32, 1)
k_hash_tma(const uint8_t* __restrict__ arena, GridDev g, uint64_t* __restrict__ chunk_dig) {
  constexpr uint32_t page_shift = 12, ns_shift = page_shift - 7, ns = 1u << ns_shift;
  constexpr uint64_t pb = 1ull << page_shift;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KiB alignment: the 128B-swizzle atom is 8 rows x 128 B
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wbuf = smem + warp * ST * kStageBytes;
  const uint32_t wbuf_u = smem_u32(wbuf);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * ST * kStageBytes) + warp * ST;
  const uint32_t bar0 = smem_u32(bars);
  const CUtensorMap* maps = static_cast<const CUtensorMap*>(g.tmaps);

  const uint32_t ppc_shift = g.chunk_shift - page_shift;
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  const uint64_t slot_base = g.c_begin << ppc_shift;
  const uint64_t nslots = (c_end - g.c_begin) << ppc_shift;
  const uint64_t ntasks = (nslots + 31) >> 5;
  const uint64_t gw = uint64_t(blockIdx.x) * WARPS + warp;
  const uint64_t nw = uint64_t(gridDim.x) * WARPS;
  if (gw >= ntasks) return;
  const uint64_t nsteps = ((ntasks - gw + nw - 1) / nw) << ns_shift;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < ST; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // producer-side state of the task being loaded (warp-uniform except p_src/p_len)
  bool p_reg = false;
  uint32_t p_map = 0, p_row = 0;
  const uint8_t* p_src = nullptr;
  uint32_t p_len = 0;
  uint32_t reg_bits = 0;  // bit (i & 1): task i was loaded through the tensor path
  uint32_t ist = 0, cst = 0;

  auto issue = [&](uint64_t p) {
    const uint32_t st = ist;
    ist = ist + 1 == ST ? 0 : ist + 1;
    if (p >= nsteps) return;
    const uint64_t i = p >> ns_shift;
    const uint32_t s = static_cast<uint32_t>(p) & (ns - 1);
    if (s == 0) {
      const uint64_t slot = slot_base + (gw + i * nw) * 32 + lane;
      const uint64_t gc = slot >> ppc_shift;
      uint32_t b = 0xffffffffu, row = 0;
      p_src = nullptr;
      p_len = 0;
      if (gc < c_end) {
        b = find_buf(g, gc);
        const uint64_t k = gc - __ldg(g.cstart + b);
        const uint64_t off = (k << g.chunk_shift) + ((slot & ((1u << ppc_shift) - 1)) << page_shift);
        const uint64_t bytes = __ldg(g.bytes + b);
        if (off < bytes) {
          const uint64_t rem = bytes - off;
          p_len = static_cast<uint32_t>(rem < pb ? rem : pb);
          p_src = arena + __ldg(g.addr + b) + off;
          row = static_cast<uint32_t>(off >> page_shift);
        }
      }
      const uint32_t b0 = __shfl_sync(kFull, b, 0);
      const uint32_t r0 = __shfl_sync(kFull, row, 0);
      p_reg = __all_sync(kFull, b == b0 && p_len == pb && row == r0 + lane);
      p_map = b0;
      p_row = r0;
      if (p_reg) reg_bits |= 1u << (i & 1); else reg_bits &= ~(1u << (i & 1));
    }
    const uint32_t bar = bar0 + 8 * st;
    const uint32_t dst = wbuf_u + st * kStageBytes;
    if (p_reg) {
      if (lane == 0) {
        mbar_arrive_tx(bar, kStageBytes);
        tma_load_2d(dst, maps + p_map, static_cast<int>(s * kSlab), static_cast<int>(p_row), bar);
      }
    } else {
      const bool valid = s * kSlab < p_len;
      const uint32_t nvalid = __popc(__ballot_sync(kFull, valid));
      if (lane == 0) mbar_arrive_tx(bar, nvalid * kSlab);
      __syncwarp();
      if (valid) bulk_load(dst + lane * kSlab, p_src + s * kSlab, kSlab, bar);
    }
  };

#pragma unroll
  for (int p = 0; p < ST - 1; ++p) issue(p);

  uint32_t lo = 0, hi = 0, mylen = 0;
  const uint32_t hswz = wbuf_u + lane * kSlab;  // + ((uu ^ (lane & 7)) << 4) when swizzled
  for (uint64_t t = 0; t < nsteps; ++t) {
    issue(t + ST - 1);
    const uint32_t st = cst;
    cst = cst + 1 == ST ? 0 : cst + 1;
    const uint64_t i = t >> ns_shift;
    const uint32_t s = static_cast<uint32_t>(t) & (ns - 1);
    if (s == 0) {
      // own page length of task i (recomputed: the producer may already be ahead)
      const uint64_t slot = slot_base + (gw + i * nw) * 32 + lane;
      const uint64_t gc = slot >> ppc_shift;
      mylen = 0;
      if (gc < c_end) {
        const uint32_t b = find_buf(g, gc);
        const uint64_t k = gc - __ldg(g.cstart + b);
        const uint64_t off = (k << g.chunk_shift) + ((slot & ((1u << ppc_shift) - 1)) << page_shift);
        const uint64_t bytes = __ldg(g.bytes + b);
        if (off < bytes) mylen = static_cast<uint32_t>(bytes - off < pb ? bytes - off : pb);
      }
      lo = static_cast<uint32_t>(kFnvOffset);
      hi = static_cast<uint32_t>(kFnvOffset >> 32);
    }
    mbar_wait(bar0 + 8 * st, static_cast<uint32_t>((t / ST) & 1));
    const uint32_t sw = (reg_bits >> (i & 1)) & 1 ? static_cast<uint32_t>(lane & 7) << 4 : 0u;
    const uint32_t a = (hswz + st * kStageBytes) | sw;
    if (s * kSlab < mylen) {
#pragma unroll
      for (int uu = 0; uu < 8; ++uu) {
        const uint4 v = ld_shared16(a ^ (uu << 4));
        fnv_word(lo, hi, v.x);
        fnv_word(lo, hi, v.y);
        fnv_word(lo, hi, v.z);
        fnv_word(lo, hi, v.w);
      }
    }
    __syncwarp();  // the slot is refilled ST - 1 steps later by this warp's lane 0
    if (s == ns - 1) {
      const uint64_t slot0 = slot_base + (gw + i * nw) * 32;
      if (ppc_shift == 0) {
        if (mylen > 0) k1_store_digest(g, slot0 + lane, (uint64_t(hi) << 32) | lo, chunk_dig);
      } else {
        const uint32_t ppc = 1u << ppc_shift;
        const int base = lane & ~static_cast<int>(ppc - 1);
        uint32_t flo = static_cast<uint32_t>(kFnvOffset);
        uint32_t fhi = static_cast<uint32_t>(kFnvOffset >> 32);
        for (uint32_t qq = 0; qq < ppc; ++qq) {
          const uint32_t plo = __shfl_sync(kFull, lo, base + qq);
          const uint32_t phi = __shfl_sync(kFull, hi, base + qq);
          const uint32_t pl = __shfl_sync(kFull, mylen, base + qq);
          if (pl > 0) {
            fnv_word(flo, fhi, plo);
            fnv_word(flo, fhi, phi);
          }
        }
        if (lane == base && mylen > 0)
            k1_store_digest(g, (slot0 + lane) >> ppc_shift, (uint64_t(fhi) << 32) | flo, chunk_dig);
      }
    }
  }
  if (g.xdig != nullptr) __threadfence_system();
}


// Fused K1 (hash + speculative K3 stores) with TMA tensor loads: CfgE's
// geometry (12 warps, 2 stages, 256-byte slabs per page = two 32 x 128 B
// SWIZZLE_128B boxes per task) without the per-lane cp.async address math.
// After a stage is hashed, the warp writes the slabs of its predicted-staged
// pages to staging + spec_off[chunk] + page offset, 16 lanes per page
// (256 contiguous bytes), read back from the swizzled stage.
template <int WARPS, int ST>
__global__ void __launch_bounds__(WARPS * 32, 1)
k_hash_tma_fused(const uint8_t* __restrict__ arena, GridDev g, uint64_t* __restrict__ chunk_dig,
                 const uint64_t* __restrict__ spec_off, uint8_t* __restrict__ staging) {
  constexpr uint32_t page_shift = 12, SLAB = 256, ns = 4096 / SLAB;  // 16 stages per page
  constexpr uint32_t kStage = 32 * SLAB;                             // 2 boxes of 4 KiB
  constexpr uint64_t pb = 1ull << page_shift;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t wbuf_u = smem_u32(smem + warp * ST * kStage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * ST * kStage) + warp * ST;
  const uint32_t bar0 = smem_u32(bars);
  const CUtensorMap* maps = static_cast<const CUtensorMap*>(g.tmaps);

  const uint32_t ppc_shift = g.chunk_shift - page_shift;
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  const uint64_t slot_base = g.c_begin << ppc_shift;
  const uint64_t nslots = (c_end - g.c_begin) << ppc_shift;
  const uint64_t ntasks = (nslots + 31) >> 5;
  const uint64_t gw = uint64_t(blockIdx.x) * WARPS + warp;
  const uint64_t nw = uint64_t(gridDim.x) * WARPS;
  if (gw >= ntasks) return;
  const uint64_t nsteps = ((ntasks - gw + nw - 1) / nw) * ns;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < ST; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  auto page = [&](uint64_t i, const uint8_t*& src, uint32_t& len, uint32_t& b, uint32_t& row,
                  uint64_t& gc) {
    const uint64_t slot = slot_base + (gw + i * nw) * 32 + lane;
    gc = slot >> ppc_shift;
    b = 0xffffffffu;
    row = 0;
    src = nullptr;
    len = 0;
    if (gc < c_end) {
      b = find_buf(g, gc);
      const uint64_t k = gc - __ldg(g.cstart + b);
      const uint64_t off = (k << g.chunk_shift) + ((slot & ((1u << ppc_shift) - 1)) << page_shift);
      const uint64_t bytes = __ldg(g.bytes + b);
      if (off < bytes) {
        const uint64_t rem = bytes - off;
        len = static_cast<uint32_t>(rem < pb ? rem : pb);
        src = arena + __ldg(g.addr + b) + off;
        row = static_cast<uint32_t>(off >> page_shift);
      }
    }
  };

  bool p_reg = false;
  uint32_t p_map = 0, p_row = 0, p_len = 0;
  const uint8_t* p_src = nullptr;
  uint32_t reg_bits = 0;  // bit (i & 1): task i was loaded through the tensor path
  uint32_t ist = 0, cst = 0;

  auto issue = [&](uint64_t p) {
    const uint32_t st = ist;
    ist = ist + 1 == ST ? 0 : ist + 1;
    if (p >= nsteps) return;
    const uint64_t i = p / ns;
    const uint32_t s = static_cast<uint32_t>(p % ns);
    if (s == 0) {
      uint32_t b, row;
      uint64_t gc;
      page(i, p_src, p_len, b, row, gc);
      const uint32_t b0 = __shfl_sync(kFull, b, 0);
      const uint32_t r0 = __shfl_sync(kFull, row, 0);
      p_reg = __all_sync(kFull, b == b0 && p_len == pb && row == r0 + lane);
      p_map = b0;
      p_row = r0;
      if (p_reg) reg_bits |= 1u << (i & 1); else reg_bits &= ~(1u << (i & 1));
    }
    const uint32_t bar = bar0 + 8 * st;
    const uint32_t dst = wbuf_u + st * kStage;
    if (p_reg) {
      if (lane == 0) {
        mbar_arrive_tx(bar, kStage);
        tma_load_2d(dst, maps + p_map, static_cast<int>(s * SLAB), static_cast<int>(p_row), bar);
        tma_load_2d(dst + 4096, maps + p_map, static_cast<int>(s * SLAB + 128),
                    static_cast<int>(p_row), bar);
      }
    } else {
      const bool valid = s * SLAB < p_len;
      const uint32_t nvalid = __popc(__ballot_sync(kFull, valid));
      if (lane == 0) mbar_arrive_tx(bar, nvalid * SLAB);
      __syncwarp();
      if (valid) {
        bulk_load(dst + lane * 128, p_src + s * SLAB, 128, bar);
        bulk_load(dst + 4096 + lane * 128, p_src + s * SLAB + 128, 128, bar);
      }
    }
  };

#pragma unroll
  for (int p = 0; p < ST - 1; ++p) issue(p);

  uint32_t lo = 0, hi = 0, mylen = 0;
  uint8_t* mydst = nullptr;
  for (uint64_t t = 0; t < nsteps; ++t) {
    issue(t + ST - 1);
    const uint32_t st = cst;
    cst = cst + 1 == ST ? 0 : cst + 1;
    const uint64_t i = t / ns;
    const uint32_t s = static_cast<uint32_t>(t % ns);
    if (s == 0) {
      const uint8_t* src;
      uint32_t b, row;
      uint64_t gc;
      page(i, src, mylen, b, row, gc);
      mydst = nullptr;
      if (mylen > 0) {
        const uint64_t so = __ldg(spec_off + gc);
        if (so != ~0ull) {
          const uint64_t slot = slot_base + (gw + i * nw) * 32 + lane;
          mydst = staging + so + ((slot & ((1u << ppc_shift) - 1)) << page_shift);
        }
      }
      lo = static_cast<uint32_t>(kFnvOffset);
      hi = static_cast<uint32_t>(kFnvOffset >> 32);
    }
    mbar_wait(bar0 + 8 * st, static_cast<uint32_t>((t / ST) & 1));
    const bool reg = (reg_bits >> (i & 1)) & 1;
    const uint32_t sbase = wbuf_u + st * kStage;
    const uint32_t a = (sbase + lane * 128) | (reg ? static_cast<uint32_t>(lane & 7) << 4 : 0u);
    const bool valid = s * SLAB < mylen;
    if (valid) {
#pragma unroll
      for (int uu = 0; uu < 16; ++uu) {
        const uint4 v = ld_shared16((a ^ ((uu & 7) << 4)) + (uu >> 3) * 4096);
        fnv_word(lo, hi, v.x);
        fnv_word(lo, hi, v.y);
        fnv_word(lo, hi, v.z);
        fnv_word(lo, hi, v.w);
      }
    }
    // speculative compaction of this stage: 16 lanes per page, 2 pages per store
    const uint32_t vm = __ballot_sync(kFull, valid && mydst != nullptr);
    if (vm) {
      const uint32_t x = lane & 15, jj = lane >> 4;
#pragma unroll 4
      for (int k = 0; k < 16; ++k) {
        const uint32_t j = 2 * k + jj;
        uint8_t* d = reinterpret_cast<uint8_t*>(
            __shfl_sync(kFull, reinterpret_cast<uint64_t>(mydst), j));
        if ((vm >> j) & 1) {
          const uint32_t sw = reg ? (j & 7) : 0u;
          const uint4 v = ld_shared16(sbase + (x >> 3) * 4096 + j * 128 + (((x & 7) ^ sw) << 4));
          __stcs(reinterpret_cast<uint4*>(d + s * SLAB + x * 16), v);
        }
      }
    }
    __syncwarp();  // the slot is refilled ST - 1 steps later by this warp's lane 0
    if (s == ns - 1) {
      const uint64_t slot0 = slot_base + (gw + i * nw) * 32;
      if (ppc_shift == 0) {
        if (mylen > 0) k1_store_digest(g, slot0 + lane, (uint64_t(hi) << 32) | lo, chunk_dig);
      } else {
        const uint32_t ppc = 1u << ppc_shift;
        const int base = lane & ~static_cast<int>(ppc - 1);
        uint32_t flo = static_cast<uint32_t>(kFnvOffset);
        uint32_t fhi = static_cast<uint32_t>(kFnvOffset >> 32);
        for (uint32_t qq = 0; qq < ppc; ++qq) {
          const uint32_t plo = __shfl_sync(kFull, lo, base + qq);
          const uint32_t phi = __shfl_sync(kFull, hi, base + qq);
          const uint32_t pl = __shfl_sync(kFull, mylen, base + qq);
          if (pl > 0) {
            fnv_word(flo, fhi, plo);
            fnv_word(flo, fhi, phi);
          }
        }
        if (lane == base && mylen > 0)
          k1_store_digest(g, (slot0 + lane) >> ppc_shift, (uint64_t(fhi) << 32) | flo, chunk_dig);
      }
    }
  }
  if (g.xdig != nullptr) __threadfence_system();
}

constexpr int kTfWarps = 12, kTfStages = 2;
constexpr size_t kTfSmem = size_t(kTfWarps) * kTfStages * 32 * 256 + size_t(kTfWarps) * kTfStages * 8 + 1024;

constexpr int kTmaWarps = 16, kTmaStages = 3;
constexpr size_t kTmaSmem = size_t(kTmaWarps) * kTmaStages * kStageBytes +
                            size_t(kTmaWarps) * kTmaStages * 8 + 1024;

}  // namespace

bool hash_tma_ok(const GridDev& g) { return g.tmaps != nullptr && g.page_shift == 12; }

int launch_hash_tma(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig, cudaStream_t s) {
  static uint64_t attr = 0;
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_hash_tma<kTmaWarps, kTmaStages>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTmaSmem));
  });
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  if (c_end <= g.c_begin) return 0;
  const uint64_t ntasks = (((c_end - g.c_begin) << (g.chunk_shift - g.page_shift)) + 31) / 32;
  uint64_t blocks = (ntasks + kTmaWarps - 1) / kTmaWarps;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (blocks > uint64_t(sms)) blocks = uint64_t(sms);
  k_hash_tma<kTmaWarps, kTmaStages><<<unsigned(blocks), kTmaWarps * 32, kTmaSmem, s>>>(arena, g,
                                                                                     chunk_dig);
  return 1;
}

int launch_hash_tma_fused(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig,
                          const uint64_t* spec_off, uint8_t* staging, cudaStream_t s) {
  static uint64_t attr = 0;
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_hash_tma_fused<kTfWarps, kTfStages>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTfSmem));
  });
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  if (c_end <= g.c_begin) return 0;
  const uint64_t ntasks = (((c_end - g.c_begin) << (g.chunk_shift - g.page_shift)) + 31) / 32;
  uint64_t blocks = (ntasks + kTfWarps - 1) / kTfWarps;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (blocks > uint64_t(sms)) blocks = uint64_t(sms);
  k_hash_tma_fused<kTfWarps, kTfStages><<<unsigned(blocks), kTfWarps * 32, kTfSmem, s>>>(
      arena, g, chunk_dig, spec_off, staging);
  return 1;
}

// Host: one 2D tensor map per buffer (rows = its full 4 KiB pages, pitch 4 KiB,
// box 32 rows x 128 B, 128B swizzle). Buffers with no full page get an unused
// zeroed entry (their tasks are irregular).
int encode_tensor_maps(const uint8_t* arena, const uint64_t* addr, const uint64_t* bytes,
                       uint32_t nbufs, void* host_maps /* nbufs x 128 B */, int box_bytes,
                       int box_rows, uint64_t arena_bytes) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return -1;
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  CUtensorMap* maps = static_cast<CUtensorMap*>(host_maps);
  for (uint32_t b = 0; b < nbufs; ++b) {
    std::memset(&maps[b], 0, sizeof(CUtensorMap));
    // arena_bytes != 0: the buffer's partial last page is a row too (its tail
    // beyond the buffer is loaded but never hashed), if the row fits the arena
    cuuint64_t rows = bytes[b] >> 12;
    if (arena_bytes && (bytes[b] & 4095) && addr[b] + ((rows + 1) << 12) <= arena_bytes) ++rows;
    if (rows == 0) continue;
    const cuuint64_t dims[2] = {4096, rows};
    const cuuint64_t strides[1] = {4096};
    const cuuint32_t box[2] = {cuuint32_t(box_bytes), cuuint32_t(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&maps[b], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                        const_cast<uint8_t*>(arena + addr[b]), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        box_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return -2;
  }
  return 0;
}

// 16 arena-wide maps, one per 256-byte alignment class k of a page start:
// base = arena + 256 k, rows of 4096 B, ceil((arena_bytes - 256 k) / 4096) rows
// (the arena has one page of padding), box = box_rows x box_bytes. A page at
// arena offset a is row a >> 12 of map (a >> 8) & 15. Few maps for any number
// of buffers: the TMA descriptor cache stays warm (C3's 876 buffers: 5.28 TB/s
// with per-buffer maps vs 5.86 for one buffer of the same bytes).
int encode_arena_maps(const uint8_t* arena, uint64_t arena_bytes, int box_bytes, int box_rows,
                      void* host_maps /* 16 x 128 B */) {
  CUtensorMap* maps = static_cast<CUtensorMap*>(host_maps);
  for (uint32_t k = 0; k < 16; ++k) {
    std::memset(&maps[k], 0, sizeof(CUtensorMap));
    if (256ull * k >= arena_bytes) continue;
    const uint64_t span = arena_bytes - 256ull * k;
    const uint64_t rows = (span + 4095) >> 12;
    const uint64_t bytes = rows << 12;
    const uint64_t addr = 256ull * k;
    if (encode_tensor_maps(arena, &addr, &bytes, 1, &maps[k], box_bytes, box_rows) != 0) return -1;
  }
  return 0;
}

}  // namespace snap
