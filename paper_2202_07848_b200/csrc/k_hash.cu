// k_hash.cu — K1: per-page / per-chunk 64-bit FNV-1a content digests over
// every tracked allocation (replaces sim::digest_of_words, sim.hpp:55-70, as
// called by Gpu::digest vdev.cpp:118, GpuLedger::refresh_digests
// splice.cpp:150-159 / plan_switch splice.cpp:176 and BlobStore::put
// ckpt.cpp:17), optionally fused with K3 stream compaction.
//
// FNV-1a is byte-serial inside one digest, so parallelism comes from hashing
// many pages at once: one lane = one page chain, one warp = 32 consecutive
// chunk-aligned page slots (= 2 chunks of 16 pages by default). Data reaches
// the lanes through shared memory: per 128-byte step the warp fills 32 page
// slabs with coalesced 16-byte cp.async (3-stage ring), each lane hashes its
// own slab with conflict-free 16-byte LDS (XOR swizzle), and — when the chunk
// is predicted to be staged — the warp writes the same slabs to the staging
// image with coalesced streaming stores, so the image is read from HBM once
// for hash + compaction. (A per-lane TMA bulk-copy variant was measured at
// half this throughput: 128-byte bulk requests are dominated by per-request
// TMA cost.) The 16 page digests of a chunk are folded into the chunk digest
// with warp shuffles (digest_of_words over the page digests).
#include <cuda_runtime.h>

#include <cstdlib>

#include "snap_internal.h"
#include "table.cuh"

namespace snap {
namespace {

constexpr uint32_t kFull = 0xffffffffu;
__device__ __forceinline__ uint4 ld_shared16(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

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
__device__ __forceinline__ void st_stream16(uint8_t* p, uint4 v) {
  // streaming store (evict-first): the staging image is not re-read soon
  __stcs(reinterpret_cast<uint4*>(p), v);
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
  if (g.chunk_buf) return __ldg(g.chunk_buf + gc);
  uint32_t lo = 0, hi = g.nbufs;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(g.cstart + mid) <= gc) lo = mid; else hi = mid;
  }
  return lo;
}

// Kernel geometry. CH page chains per lane (independent FNV chains the
// scheduler can interleave), SLAB bytes of each page per pipeline step,
// STAGES-deep cp.async ring, WARPS warps per CTA (one CTA per SM).
template <int CH, int SLAB, int STAGES, int WARPS>
struct HashCfg {
  static constexpr int kCh = CH, kSlab = SLAB, kStages = STAGES, kWarps = WARPS;
  static constexpr int kPages = 32 * CH;                 // page slots per warp task
  static constexpr int kUnits = SLAB / 16;               // 16-byte units per slab
  static constexpr int kLanesPerPage = kUnits;           // copy-in: 1 unit per lane
  static constexpr int kPagesPerInstr = 32 / kUnits;
  static constexpr int kCopyInstr = kPages / kPagesPerInstr;
  static constexpr int kStageBytes = kPages * SLAB;
  static constexpr int kWarpBytes = STAGES * kStageBytes;
  static constexpr int kDescBytes = 2 * kPages * 16 + 2 * kPages * 4;  // src,dst | len
  static constexpr size_t kSmem = size_t(WARPS) * (kWarpBytes + kDescBytes);
  // swizzle: unit u of slab j is stored at unit u ^ sw(j) so that 8 lanes
  // reading the same unit of 8 consecutive slabs hit 8 distinct 16-B bank
  // groups (slab j starts at bank group (j * kUnits) mod 8).
  static constexpr int kSwShift = kUnits >= 8 ? 0 : (kUnits == 4 ? 1 : (kUnits == 2 ? 2 : 3));
  __device__ static __forceinline__ uint32_t sw(uint32_t j) {
    if constexpr (kUnits >= 8) return j & 7;
    else return (j >> kSwShift) & (kUnits - 1);
  }
};

// K1 (+ fused K3 when spec_off != nullptr). Warp task = 32*CH consecutive
// chunk-aligned page slots; lane l hashes slots l, l+32, ... (CH chains).
// Copy-in: per step, kUnits lanes move one page's SLAB-byte slab with one
// coalesced 16-byte cp.async each. A task whose pages are all full and
// contiguous in one buffer (the common case) takes the "regular" path: one
// base pointer plus fixed strides, no per-page descriptor loads. When a chunk
// has a speculative staging offset (spec_off[chunk] != ~0) the same slab is
// also written to staging + offset with coalesced 16-byte streaming stores
// read back from shared memory, so the image is read from HBM once for hash
// and compaction together.
template <class C, int PS, int PPC>
__global__ void __launch_bounds__(C::kWarps * 32, 1)
k_hash(const uint8_t* __restrict__ arena, GridDev g, uint64_t* __restrict__ chunk_dig,
       const uint64_t* __restrict__ spec_off, uint8_t* __restrict__ staging) {
  constexpr int CH = C::kCh, SLAB = C::kSlab, ST = C::kStages, NP = C::kPages;
  constexpr int NU = C::kUnits, PPI = C::kPagesPerInstr;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint8_t* wbuf = smem + warp * C::kWarpBytes;
  const uint32_t wbuf_u = smem_u32(wbuf);
  uint8_t* dsm = smem + C::kWarps * C::kWarpBytes + warp * C::kDescBytes;
  uint64_t* dptr = reinterpret_cast<uint64_t*>(dsm);               // [2][NP][2] src,dst
  uint32_t* dlen = reinterpret_cast<uint32_t*>(dsm + 2 * NP * 16);  // [2][NP]

  // PS != 0: page size known at compile time (4 KiB), so every page stride
  // below is an immediate offset
  const uint32_t page_shift = PS ? PS : g.page_shift;
  const uint32_t ppc_shift = g.chunk_shift - page_shift;
  constexpr uint32_t slab_shift =
      SLAB == 512 ? 9 : (SLAB == 256 ? 8 : (SLAB == 128 ? 7 : (SLAB == 64 ? 6 : 5)));
  const uint32_t ns_shift = page_shift - slab_shift;  // steps per page (log2)
  const uint32_t ns = 1u << ns_shift;
  const uint64_t pb = 1ull << page_shift;
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  const uint64_t slot_base = g.c_begin << ppc_shift;
  const uint64_t nslots = (c_end - g.c_begin) << ppc_shift;
  const uint64_t ntasks = (nslots + NP - 1) / NP;
  const uint64_t gw = uint64_t(blockIdx.x) * C::kWarps + warp;
  const uint64_t nw = uint64_t(gridDim.x) * C::kWarps;
  // launched with PDL: the CTAs become resident while the previous kernel of
  // the stream (e.g. the last snapshot's selection) drains; wait for it here
  griddep_wait();
  if (gw >= ntasks) return;
  const uint64_t my_tasks = (ntasks - gw + nw - 1) / nw;
  const uint64_t nsteps = my_tasks << ns_shift;
  const uint32_t u = lane % NU, q = lane / NU;  // copy role: unit u of page q + k*PPI
  // shared-memory byte offset of (page q + k*PPI, unit u) inside a stage:
  // (q + k*PPI)*SLAB + ((u ^ sw(q + k*PPI)) << 4); sw only depends on k
  // through (k*PPI) & 7, so two bases (even/odd k) + immediates cover all k
  auto copy_off = [&](int k) -> uint32_t {
    const int j = k * PPI + q;
    return uint32_t(j) * SLAB + ((u ^ C::sw(j)) << 4);
  };
  // per-lane hash read address (stage 0): slab `lane` with its swizzle bits;
  // unit uu is at (hbase ^ (uu << 4)) + stage * kStageBytes + c * 32 * SLAB
  const uint32_t hbase = wbuf_u + lane * SLAB + (C::sw(lane) << 4);

  bool reg0 = false, reg1 = false, wr0 = false, wr1 = false;
  const uint8_t *rsrc0 = nullptr, *rsrc1 = nullptr;
  // staging destinations of the regular path, one base per chunk of the task:
  // with <= 2 chunks per task (default geometry: 16 pages per chunk, 32 per
  // task) each chunk is either not staged or staged contiguously, so striped
  // layouts (alternate chunks of another rank) stay on the fast path; with
  // more chunks per task the whole task must be contiguous (wshift = 31)
  uint8_t *rdst0 = nullptr, *rdst1 = nullptr, *rdstb0 = nullptr, *rdstb1 = nullptr;
  const uint32_t jb = 1u << ppc_shift;  // first page of the task's second chunk
  const bool two_chunks = (uint32_t(NP) >> ppc_shift) <= 2;
  const uint32_t wshift = two_chunks ? ppc_shift : 31;
  uint32_t ist = 0, cst = 0;  // stage of the next issue / of the step being consumed

  // next task's chunk descriptors (arena offset, length, staging offset), loaded one
  // step before the task starts so the loads overlap the current step's hash
  uint64_t pf_ca[CH], pf_so[CH];
  uint32_t pf_clen[CH];
  uint64_t pf_i = ~0ull;
  auto prefetch = [&](uint64_t i) {
    if (!g.chunk_addr) return;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const uint64_t gc = (slot_base + (gw + i * nw) * NP + c * 32 + lane) >> ppc_shift;
      pf_ca[c] = 0;
      pf_clen[c] = 0;
      pf_so[c] = ~0ull;
      if (gc < c_end) {
        pf_ca[c] = __ldg(g.chunk_addr + gc);
        pf_clen[c] = __ldg(g.chunk_len + gc);
        if (spec_off) pf_so[c] = __ldg(spec_off + gc);
      }
    }
    pf_i = i;
  };

  auto issue = [&](uint64_t p) {
    const uint32_t st = ist;
    ist = ist + 1 == ST ? 0 : ist + 1;
    if (p < nsteps) {
      const uint64_t i = p >> ns_shift;
      const uint32_t s = static_cast<uint32_t>(p) & (ns - 1);
      const uint32_t par = static_cast<uint32_t>(i & 1);
      if (s == 0) {
        __syncwarp();
        bool allreg = true, anyw = false, dreg = true;
        const uint8_t* s0 = nullptr;
        uint8_t *d0 = nullptr, *db = nullptr;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int j = c * 32 + lane;
          const uint64_t slot = slot_base + (gw + i * nw) * NP + j;
          const uint64_t gc = slot >> ppc_shift;
          const uint8_t* src = nullptr;
          uint8_t* dst = nullptr;
          uint32_t len = 0;
          if (gc < c_end) {
            uint64_t ca, so = ~0ull;
            uint32_t clen;
            if (pf_i == i) {
              ca = pf_ca[c];
              clen = pf_clen[c];
              so = pf_so[c];
            } else {
              chunk_loc(g, gc, ca, clen);
              if (spec_off) so = __ldg(spec_off + gc);
            }
            const uint64_t in_chunk = (slot & ((1u << ppc_shift) - 1)) << page_shift;
            if (in_chunk < clen) {
              const uint64_t rem = clen - in_chunk;
              len = static_cast<uint32_t>(rem < pb ? rem : pb);
              if (g.reverse) {
                // verify-scatter: the image holds the chunk, the grid address gets it
                src = staging + so + in_chunk;
                dst = const_cast<uint8_t*>(arena) + ca + in_chunk;
              } else {
                src = arena + ca + in_chunk;
                if (so != ~0ull) dst = staging + so + in_chunk;
              }
            }
          }
          dptr[(par * NP + j) * 2] = reinterpret_cast<uint64_t>(src);
          dptr[(par * NP + j) * 2 + 1] = reinterpret_cast<uint64_t>(dst);
          dlen[par * NP + j] = len;
          if (c == 0) {
            s0 = reinterpret_cast<const uint8_t*>(__shfl_sync(kFull, reinterpret_cast<uint64_t>(src), 0));
            d0 = reinterpret_cast<uint8_t*>(__shfl_sync(kFull, reinterpret_cast<uint64_t>(dst), 0));
          }
          if (two_chunks && jb < uint32_t(NP) && c == int(jb >> 5))
            db = reinterpret_cast<uint8_t*>(__shfl_sync(kFull, reinterpret_cast<uint64_t>(dst), jb & 31));
          allreg = allreg && len == pb && src == s0 + uint64_t(j) * pb;
          anyw = anyw || dst != nullptr;
          dreg = dreg && d0 != nullptr && dst == d0 + uint64_t(j) * pb;
        }
        const bool w = __any_sync(kFull, anyw);
        const bool r = __all_sync(kFull, allreg) && (!w || two_chunks || __all_sync(kFull, dreg));
        if (par) {
          reg1 = r; wr1 = w; rsrc1 = s0; rdst1 = d0; rdstb1 = db;
        } else {
          reg0 = r; wr0 = w; rsrc0 = s0; rdst0 = d0; rdstb0 = db;
        }
        __syncwarp();
      }
      const uint32_t sbase = wbuf_u + st * C::kStageBytes;
      const uint32_t soff = s * SLAB + u * 16;
      if (par ? reg1 : reg0) {
        const uint8_t* src = (par ? rsrc1 : rsrc0) + q * pb + soff;
#pragma unroll
        for (int k = 0; k < C::kCopyInstr; ++k)
          cp_async16(sbase + copy_off(k), src + uint64_t(k) * PPI * pb);
      } else {
#pragma unroll
        for (int k = 0; k < C::kCopyInstr; ++k) {
          const int j = k * PPI + q;
          const uint32_t len = dlen[par * NP + j];
          if (soff < len)
            cp_async16(sbase + copy_off(k),
                       reinterpret_cast<const uint8_t*>(dptr[(par * NP + j) * 2]) + soff);
        }
      }
    }
    cp_commit();
  };

  // Speculative compaction of the consumed step: coalesced 16-byte streaming
  // stores (kUnits lanes per slab) read back from the swizzled stage buffer.
  auto store = [&](uint64_t t, uint32_t st) {
    const uint64_t i = t >> ns_shift;
    const uint32_t par = static_cast<uint32_t>(i & 1);
    if (!(par ? wr1 : wr0)) return;
    const uint32_t s = static_cast<uint32_t>(t) & (ns - 1);
    const uint8_t* sb = wbuf + st * C::kStageBytes;
    const uint32_t soff = s * SLAB + u * 16;
    if (par ? reg1 : reg0) {
      uint8_t* da = par ? rdst1 : rdst0;
      uint8_t* dbb = par ? rdstb1 : rdstb0;
      if constexpr (PPC != 0 && NP / (PPC ? PPC : 1) <= 2 && PPC % PPI == 0) {
        // pages per chunk known at compile time: the chunk split of the
        // unrolled store loop is static (pages k*PPI + q, q < PPI)
        constexpr int KA = PPC < NP ? PPC / PPI : C::kCopyInstr;
        if (da) {
          uint8_t* d = da + q * pb + soff;
#pragma unroll
          for (int k = 0; k < KA; ++k)
            st_stream16(d + uint64_t(k) * PPI * pb, *reinterpret_cast<const uint4*>(sb + copy_off(k)));
        }
        if (KA < C::kCopyInstr && dbb) {
          uint8_t* d = dbb + q * pb + soff;
#pragma unroll
          for (int k = KA; k < C::kCopyInstr; ++k)
            st_stream16(d + uint64_t(k - KA) * PPI * pb,
                        *reinterpret_cast<const uint4*>(sb + copy_off(k)));
        }
      } else {
#pragma unroll
        for (int k = 0; k < C::kCopyInstr; ++k) {
          const uint32_t j = uint32_t(k * PPI) + q;
          const uint32_t ch = j >> wshift;
          uint8_t* base = ch ? dbb : da;
          if (base)
            st_stream16(base + uint64_t(j - (ch << wshift)) * pb + soff,
                        *reinterpret_cast<const uint4*>(sb + copy_off(k)));
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < C::kCopyInstr; ++k) {
        const int j = k * PPI + q;
        uint8_t* dst = reinterpret_cast<uint8_t*>(dptr[(par * NP + j) * 2 + 1]);
        if (dst && soff < dlen[par * NP + j])
          st_stream16(dst + soff, *reinterpret_cast<const uint4*>(sb + copy_off(k)));
      }
    }
  };

#pragma unroll
  for (int p = 0; p < ST - 1; ++p) issue(p);

  uint32_t lo[CH], hi[CH], mylen[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) lo[c] = hi[c] = mylen[c] = 0;
  for (uint64_t t = 0; t < nsteps; ++t) {
    issue(t + ST - 1);
    if (((t + ST) & (ns - 1)) == 0 && t + ST < nsteps) prefetch((t + ST) >> ns_shift);
    cp_wait<ST - 1>();
    __syncwarp();
    const uint64_t i = t >> ns_shift;
    const uint32_t s = static_cast<uint32_t>(t) & (ns - 1);
    const uint32_t par = static_cast<uint32_t>(i & 1);
    if (s == 0) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        mylen[c] = dlen[par * NP + c * 32 + lane];
        lo[c] = static_cast<uint32_t>(kFnvOffset);
        hi[c] = static_cast<uint32_t>(kFnvOffset >> 32);
      }
    }
    const uint32_t st = cst;
    cst = cst + 1 == ST ? 0 : cst + 1;
    store(t, st);
    const uint32_t sadd = st * C::kStageBytes;
#pragma unroll
    for (int uu = 0; uu < NU; ++uu) {
      // CH independent chains interleaved unit by unit
      uint4 v[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c)
        v[c] = ld_shared16((hbase ^ (uu << 4)) + sadd + c * 32 * SLAB);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (s * SLAB < mylen[c]) {
          fnv_word(lo[c], hi[c], v[c].x);
          fnv_word(lo[c], hi[c], v[c].y);
          fnv_word(lo[c], hi[c], v[c].z);
          fnv_word(lo[c], hi[c], v[c].w);
        }
      }
    }
    __syncwarp();
    if (s == ns - 1) {
      // Task complete: each lane holds CH page digests (or nothing).
      const uint64_t slot0 = slot_base + (gw + i * nw) * NP;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const uint64_t myslot = slot0 + c * 32 + lane;
        if (ppc_shift == 0) {
          if (mylen[c] > 0) k1_store_digest(g, myslot, (uint64_t(hi[c]) << 32) | lo[c], chunk_dig);
        } else {
          // chunk digest = digest_of_words(page digests), folded with
          // warp-uniform shuffles inside each group of ppc lanes
          const uint32_t ppc = 1u << ppc_shift;
          const int base = lane & ~static_cast<int>(ppc - 1);
          uint32_t flo = static_cast<uint32_t>(kFnvOffset);
          uint32_t fhi = static_cast<uint32_t>(kFnvOffset >> 32);
          for (uint32_t qq = 0; qq < ppc; ++qq) {
            const uint32_t plo = __shfl_sync(kFull, lo[c], base + qq);
            const uint32_t phi = __shfl_sync(kFull, hi[c], base + qq);
            const uint32_t pl = __shfl_sync(kFull, mylen[c], base + qq);
            if (pl > 0) {
              fnv_word(flo, fhi, plo);
              fnv_word(flo, fhi, phi);
            }
          }
          if (lane == base && mylen[c] > 0)
            k1_store_digest(g, myslot >> ppc_shift, (uint64_t(fhi) << 32) | flo, chunk_dig);
        }
      }
    }
  }
  cp_wait<0>();
  if (g.dd.keys != nullptr) {
    // fused K2 insert: this warp's chunks (whole chunks per task, since NP is
    // a multiple of the pages per chunk), one chunk per lane, after the
    // streaming loop so no atomic round trip ever stalls a slab
    __syncwarp();
    const uint32_t cpt = uint32_t(NP) >> ppc_shift;
    for (uint64_t e = lane; e < my_tasks * cpt; e += 32) {
      const uint64_t i = e / cpt;
      const uint64_t c = ((slot_base + (gw + i * nw) * NP) >> ppc_shift) + (e - i * cpt);
      if (c < c_end) k1_insert(g, c, chunk_dig[c]);
    }
  }
  if (g.xdig != nullptr) __threadfence_system();  // NVLink digest stores before the barrier
}

// ---------------------------------------------------------------------------
// Warp-specialized K1: HW hash warps only hash (LDS + FNV), CW copy warps own
// all memory traffic — the coalesced cp.async fill of every hash warp's slab
// ring (completion signalled straight to a per-stage mbarrier with
// cp.async.mbarrier.arrive.noinc) and the speculative staging stores. The
// hash warps' instruction stream is then pure FNV (no address math, no
// cp.async bookkeeping), and memory latency never sits on their critical
// path. Copy warp c serves hash warps c, c + CW, ... round-robin, running
// ST - 1 steps ahead of them; a slab is refilled only after its hash warp
// released it (empty barrier) and after the copy warp stored it.
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
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
__device__ __forceinline__ void cp_async_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

template <int HW, int CW, int ST>
struct WsCfg {
  static constexpr int kHW = HW, kCW = CW, kST = ST;
  static constexpr int kSlab = 128;
  static constexpr int kStageBytes = 32 * kSlab;
  static constexpr int kPer = HW / CW;  // hash warps per copy warp
  static_assert(HW % CW == 0, "copy warps must divide hash warps");
  // smem: slabs [HW][ST][32][128] | full/empty mbarriers [HW][ST] x2 |
  // copy-side descriptors [HW][2 parities][32] x (src, dst) | lens [HW][2][32]
  static constexpr size_t kSlabBytes = size_t(HW) * ST * kStageBytes;
  static constexpr size_t kBarBytes = size_t(HW) * ST * 2 * 8;
  static constexpr size_t kDescBytes = size_t(HW) * 2 * 32 * 16;
  static constexpr size_t kLenBytes = size_t(HW) * 2 * 32 * 4;
  static constexpr size_t kStateBytes = size_t(HW) * 2 * 32;  // {src0, dst0, flags}
  static constexpr size_t kSmem = kSlabBytes + kBarBytes + kDescBytes + kLenBytes + kStateBytes;
};

// copy-side task state of one (hash warp, task parity), warp-uniform
struct WsTask {
  const uint8_t* src0;
  uint8_t* dst0;
  uint32_t regular;
  uint32_t writes;
};
static_assert(sizeof(WsTask) <= 32, "WsTask slot");

template <class C>
__global__ void __launch_bounds__((C::kHW + C::kCW) * 32, 1)
k_hash_ws(const uint8_t* __restrict__ arena, GridDev g, uint64_t* __restrict__ chunk_dig,
          const uint64_t* __restrict__ spec_off, uint8_t* __restrict__ staging) {
  constexpr int HW = C::kHW, CW = C::kCW, ST = C::kST, SLAB = C::kSlab;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* slabs = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kSlabBytes);  // full[h*ST+s], empty after
  uint64_t* desc = reinterpret_cast<uint64_t*>(smem + C::kSlabBytes + C::kBarBytes);
  uint32_t* lens = reinterpret_cast<uint32_t*>(smem + C::kSlabBytes + C::kBarBytes + C::kDescBytes);
  uint8_t* tstate = smem + C::kSlabBytes + C::kBarBytes + C::kDescBytes + C::kLenBytes;
  auto task_state = [&](int h, int par) -> WsTask& {
    return *reinterpret_cast<WsTask*>(tstate + (h * 2 + par) * 32);
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // page length of slot `slot` (0 when outside the grid / past its buffer)
  auto page_len = [&](uint64_t slot) -> uint32_t {
    const uint64_t gc = slot >> (g.chunk_shift - g.page_shift);
    if (gc >= (g.c_end ? g.c_end : g.nchunks)) return 0;
    const uint32_t b = find_buf(g, gc);
    const uint64_t kk = gc - __ldg(g.cstart + b);
    const uint64_t off = (kk << g.chunk_shift) +
                         ((slot & ((1u << (g.chunk_shift - g.page_shift)) - 1)) << g.page_shift);
    const uint64_t bytes = __ldg(g.bytes + b);
    if (off >= bytes) return 0;
    const uint64_t rem = bytes - off, pg = 1ull << g.page_shift;
    return static_cast<uint32_t>(rem < pg ? rem : pg);
  };

  const uint32_t ppc_shift = g.chunk_shift - g.page_shift;
  const uint32_t ns_shift = g.page_shift - 7;
  const uint32_t ns = 1u << ns_shift;
  const uint64_t pb = 1ull << g.page_shift;
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  const uint64_t slot_base = g.c_begin << ppc_shift;
  const uint64_t nslots = (c_end - g.c_begin) << ppc_shift;
  const uint64_t ntasks = (nslots + 31) >> 5;
  const uint64_t nw = uint64_t(gridDim.x) * HW;
  auto steps_of = [&](int h) -> uint64_t {
    const uint64_t gw = uint64_t(blockIdx.x) * HW + h;
    return gw >= ntasks ? 0 : ((ntasks - gw + nw - 1) / nw) << ns_shift;
  };
  auto full_bar = [&](int h, int s) { return smem_u32(bars + h * ST + s); };
  auto empty_bar = [&](int h, int s) { return smem_u32(bars + HW * ST + h * ST + s); };

  if (threadIdx.x == 0) {
    for (int h = 0; h < HW; ++h)
      for (int s = 0; s < ST; ++s) {
        mbar_init(full_bar(h, s), 32);   // one cp.async arrival per copy lane
        mbar_init(empty_bar(h, s), 32);  // every hash lane releases the slab
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp < HW) {
    // ------------------------------------------------------------ hash warp
    const int h = warp;
    const uint64_t gw = uint64_t(blockIdx.x) * HW + h;
    const uint64_t nsteps = steps_of(h);
    uint8_t* ring = slabs + size_t(h) * ST * C::kStageBytes;
    uint32_t lo = 0, hi = 0, mylen = 0;
    for (uint64_t t = 0; t < nsteps; ++t) {
      const uint32_t s = static_cast<uint32_t>(t) & (ns - 1);
      const uint64_t i = t >> ns_shift;
      const int st = static_cast<int>(t % ST);
      mbar_wait(full_bar(h, st), static_cast<uint32_t>((t / ST) & 1));
      if (s == 0) {
        mylen = page_len(slot_base + (gw + i * nw) * 32 + lane);
        lo = static_cast<uint32_t>(kFnvOffset);
        hi = static_cast<uint32_t>(kFnvOffset >> 32);
      }
      if (s * SLAB < mylen) {
        const uint8_t* slab = ring + st * C::kStageBytes + lane * SLAB;
#pragma unroll
        for (int uu = 0; uu < 8; ++uu) {
          const uint4 v = *reinterpret_cast<const uint4*>(slab + ((uu ^ (lane & 7)) << 4));
          fnv_word(lo, hi, v.x);
          fnv_word(lo, hi, v.y);
          fnv_word(lo, hi, v.z);
          fnv_word(lo, hi, v.w);
        }
      }
      mbar_arrive(empty_bar(h, st));
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
  } else {
    // ------------------------------------------------------------ copy warp
    const int c = warp - HW;
    const uint32_t u = lane & 7, q = lane >> 3;
    // steps of every served hash warp (copy warp c serves c, c + CW, ...)
    uint64_t nst[C::kPer];
    uint64_t maxsteps = 0;
#pragma unroll
    for (int k = 0; k < C::kPer; ++k) {
      nst[k] = steps_of(c + k * CW);
      maxsteps = nst[k] > maxsteps ? nst[k] : maxsteps;
    }
    // fill step p of served warp k
    auto fill = [&](int k, uint64_t p) {
      const int h = c + k * CW;
      const uint64_t gw = uint64_t(blockIdx.x) * HW + h;
      const uint64_t i = p >> ns_shift;
      const uint32_t s = static_cast<uint32_t>(p) & (ns - 1);
      const int par = static_cast<int>(i & 1);
      const int st = static_cast<int>(p % ST);
      mbar_wait(empty_bar(h, st), static_cast<uint32_t>(((p / ST) & 1) ^ 1));
      uint64_t* dsc = desc + (h * 2 + par) * 32 * 2;
      if (s == 0) {
        const uint64_t slot = slot_base + (gw + i * nw) * 32 + lane;
        const uint64_t gc = slot >> ppc_shift;
        const uint8_t* src = nullptr;
        uint8_t* dst = nullptr;
        uint32_t len = 0;
        if (gc < c_end) {
          const uint32_t b = find_buf(g, gc);
          const uint64_t kk = gc - __ldg(g.cstart + b);
          const uint64_t in_chunk = (slot & ((1u << ppc_shift) - 1)) << g.page_shift;
          const uint64_t off = (kk << g.chunk_shift) + in_chunk;
          const uint64_t bytes = __ldg(g.bytes + b);
          if (off < bytes) {
            const uint64_t rem = bytes - off;
            len = static_cast<uint32_t>(rem < pb ? rem : pb);
            src = arena + __ldg(g.addr + b) + off;
            if (spec_off) {
              const uint64_t so = __ldg(spec_off + gc);
              if (so != ~0ull) dst = staging + so + in_chunk;
            }
          }
        }
        dsc[lane * 2] = reinterpret_cast<uint64_t>(src);
        dsc[lane * 2 + 1] = reinterpret_cast<uint64_t>(dst);
        lens[(h * 2 + par) * 32 + lane] = len;
        const uint8_t* s0 = reinterpret_cast<const uint8_t*>(
            __shfl_sync(kFull, reinterpret_cast<uint64_t>(src), 0));
        uint8_t* d0 = reinterpret_cast<uint8_t*>(__shfl_sync(kFull, reinterpret_cast<uint64_t>(dst), 0));
        const bool w = __any_sync(kFull, dst != nullptr);
        const bool r = __all_sync(kFull, len == pb && src == s0 + lane * pb) &&
                       (!w || __all_sync(kFull, d0 != nullptr && dst == d0 + lane * pb));
        if (lane == 0) task_state(h, par) = WsTask{s0, d0, r ? 1u : 0u, w ? 1u : 0u};
        __syncwarp();
      }
      const WsTask ts = task_state(h, par);
      const uint32_t sbase = smem_u32(slabs + (size_t(h) * ST + st) * C::kStageBytes);
      const uint32_t soff = s * SLAB + u * 16;
      if (ts.regular) {
        const uint8_t* src = ts.src0 + q * pb + soff;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int j = kk * 4 + q;
          cp_async16(sbase + j * SLAB + ((u ^ (j & 7)) << 4), src);
          src += 4 * pb;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int j = kk * 4 + q;
          const uint32_t len = lens[(h * 2 + par) * 32 + j];
          if (soff < len)
            cp_async16(sbase + j * SLAB + ((u ^ (j & 7)) << 4),
                       reinterpret_cast<const uint8_t*>(dsc[j * 2]) + soff);
        }
      }
      cp_async_arrive(full_bar(h, st));
    };
    // speculative store of step t of served warp k (data must have landed)
    auto store = [&](int k, uint64_t t) {
      const int h = c + k * CW;
      const uint64_t i = t >> ns_shift;
      const int par = static_cast<int>(i & 1);
      const WsTask ts = task_state(h, par);
      if (!ts.writes) return;
      const uint32_t s = static_cast<uint32_t>(t) & (ns - 1);
      const int st = static_cast<int>(t % ST);
      mbar_wait(full_bar(h, st), static_cast<uint32_t>((t / ST) & 1));
      const uint8_t* sb = slabs + (size_t(h) * ST + st) * C::kStageBytes;
      const uint32_t soff = s * SLAB + u * 16;
      const uint64_t* dsc = desc + (h * 2 + par) * 32 * 2;
      if (ts.regular) {
        uint8_t* dst = ts.dst0 + q * pb + soff;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int j = kk * 4 + q;
          st_stream16(dst, *reinterpret_cast<const uint4*>(sb + j * SLAB + ((u ^ (j & 7)) << 4)));
          dst += 4 * pb;
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int j = kk * 4 + q;
          uint8_t* dst = reinterpret_cast<uint8_t*>(dsc[j * 2 + 1]);
          if (dst && soff < lens[(h * 2 + par) * 32 + j])
            st_stream16(dst + soff,
                        *reinterpret_cast<const uint4*>(sb + j * SLAB + ((u ^ (j & 7)) << 4)));
        }
      }
    };
    // prologue: ST - 1 steps ahead for every served warp
    for (int p = 0; p < ST - 1; ++p)
#pragma unroll
      for (int k = 0; k < C::kPer; ++k)
        if (uint64_t(p) < nst[k]) fill(k, p);
    for (uint64_t t = 0; t < maxsteps; ++t) {
#pragma unroll
      for (int k = 0; k < C::kPer; ++k) {
        if (t + ST - 1 < nst[k]) fill(k, t + ST - 1);
        if (t < nst[k]) store(k, t);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  if (g.xdig != nullptr) __threadfence_system();
}

// Buffer digest = digest_of_words(chunk digests of the buffer); one thread
// per buffer (digest vectors are 1/8192 of the data).
// K2 insert over the chunk range of a K1 launch (for the K1 variants that do
// not carry the fused epilogue: warp-specialized, TMA)
__global__ void k_insert_range(GridDev g, const uint64_t* __restrict__ chunk_dig) {
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  for (uint64_t c = g.c_begin + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < c_end;
       c += uint64_t(gridDim.x) * blockDim.x)
    k1_insert(g, c, chunk_dig[c]);
}

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

// Variant selection (SNAP_HASH_VARIANT env, 1-10; see choose_k1): all compute
// identical digests, they only differ in how the bytes reach shared memory and
// in latency hiding.
using CfgA = HashCfg<1, 128, 3, 16>;  // 512 chains/SM, 128-B slabs
using CfgB = HashCfg<2, 64, 2, 16>;   // 1024 chains/SM, 64-B slabs
using CfgC = HashCfg<2, 64, 3, 12>;   // 768 chains/SM, deeper ring
using CfgD = HashCfg<2, 128, 2, 12>;  // 768 chains/SM, 128-B slabs
using CfgE = HashCfg<1, 256, 2, 12>;  // 256-B slabs: DRAM-friendly write segments
using CfgF = HashCfg<1, 256, 2, 13>;
// one wave for small fused grids (C1: 2048 tasks <= 148 x 14 warps): 256-B
// slabs, one stage per warp — latency hidden across 14-16 warps per SM
using CfgG = HashCfg<1, 256, 1, 16>;
using CfgH = HashCfg<1, 256, 1, 14>;
// 512-B segments per page and step (fewer DRAM row switches per byte), one stage
using CfgI = HashCfg<1, 512, 1, 12>;
using CfgJ = HashCfg<1, 512, 1, 13>;
// fewer warps, each overlapping its own next slab with the hash of the current
// one (experimental: small fused grids)
using CfgK = HashCfg<1, 256, 2, 8>;
using CfgL = HashCfg<1, 256, 3, 8>;
using CfgM = HashCfg<1, 256, 2, 10>;
using WsA = WsCfg<16, 4, 3>;          // warp-specialized: 16 hash + 4 copy warps
using WsB = WsCfg<16, 2, 3>;          // 16 hash + 2 copy warps
using WsC = WsCfg<12, 4, 4>;          // 12 hash + 4 copy warps, deeper ring

template <class C>
int launch_hash_ws(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig,
                   const uint64_t* spec_off, uint8_t* staging, cudaStream_t s) {
  static uint64_t attr = 0;
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_hash_ws<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem));
  });
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  if (c_end <= g.c_begin) return 0;
  const uint64_t ntasks = (((c_end - g.c_begin) << (g.chunk_shift - g.page_shift)) + 31) / 32;
  uint64_t blocks = (ntasks + C::kHW - 1) / C::kHW;
  const uint64_t cap = uint64_t(sm_count());
  if (blocks > cap) blocks = cap;
  k_hash_ws<C><<<unsigned(blocks), (C::kHW + C::kCW) * 32, C::kSmem, s>>>(arena, g, chunk_dig,
                                                                         spec_off, staging);
  return 1;
}

template <class C>
int launch_hash_cfg(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig,
                    const uint64_t* spec_off, uint8_t* staging, cudaStream_t s) {
  static uint64_t attr = 0;
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_hash<C, 12, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem));
    cudaFuncSetAttribute(k_hash<C, 12, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem));
    cudaFuncSetAttribute(k_hash<C, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem));
  });
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  if (c_end <= g.c_begin) return 0;
  const uint64_t ntasks =
      (((c_end - g.c_begin) << (g.chunk_shift - g.page_shift)) + C::kPages - 1) / C::kPages;
  uint64_t blocks = (ntasks + C::kWarps - 1) / C::kWarps;
  const uint64_t cap = uint64_t(sm_count());
  if (blocks > cap) blocks = cap;
  // the reference's 4 KiB page (strides become immediates) and the default
  // 64 KiB chunk (static chunk split of the speculative stores)
  if (g.page_shift == 12 && g.chunk_shift == 16)
    launch_pdl(k_hash<C, 12, 16>, unsigned(blocks), C::kWarps * 32, C::kSmem, s, arena, g,
               chunk_dig, spec_off, staging);
  else if (g.page_shift == 12)
    launch_pdl(k_hash<C, 12, 0>, unsigned(blocks), C::kWarps * 32, C::kSmem, s, arena, g,
               chunk_dig, spec_off, staging);
  else
    launch_pdl(k_hash<C, 0, 0>, unsigned(blocks), C::kWarps * 32, C::kSmem, s, arena, g,
               chunk_dig, spec_off, staging);
  return 1;
}

int g_hash_variant = -1;
int hash_variant() {
  if (g_hash_variant < 0) {
    const char* e = getenv("SNAP_HASH_VARIANT");
    g_hash_variant = e ? atoi(e) : -1;
    if (g_hash_variant < 0) g_hash_variant = 99;  // default policy
  }
  return g_hash_variant;
}

void set_hash_variant(int v) { g_hash_variant = v < 0 ? 99 : v; }
const char* last_k1_name();

// tensor maps are built for every grid unless a cp.async variant is forced
bool hash_tma_selected() {
  const int v = hash_variant();
  return v == 10 || v == 11 || v == 12 || v == 13 || v == 99;
}

// The K1 kernel a launch uses (SNAP_HASH_VARIANT / snap_set_k1_variant force
// one; the default is the fastest measured per shape):
//  * fused hash + speculative stores, most of the grid staged, and the
//    verify-scatter: CfgG (below) — 256-B slabs keep the mixed read/write DRAM
//    pattern at ~6 TB/s (128-B segments cap it at ~5.2, tools/micro/pattern_bw2.cu);
//  * fused, less than 55 % of a >= 512 MiB grid staged: the tensor-core kernel
//    with fused stores;
//  * hash only, grids with tensor maps: the tensor-core FNV kernel (k_hash_mma.cu:
//    16 chain warps, or 8 in 512-page groups for grids of <= one group per SM);
//  * hash only without tensor maps (forced cp.async variants, 64 MiB+ buffers):
//    CfgB / CfgA (tools/hash_variants.py).
enum class K1 { A, B, C, D, E, F, G, H, I, J, K, L, M, WsA, WsB, WsC, Tma, Mma, MmaFL, TmaF };
// Fused launches (hash + stores, and the verify-scatter): CfgG, 16 warps per
// SM with one 256-byte stage each. Same-box A/B (tools/fused_variants.py,
// tools/c1_variants.py): C2 N = 1 K1 0.734-0.740 ms vs CfgE's 0.796-0.798
// (0.89 vs 0.82 of the copy roofline; 512 more page chains in flight per SM
// outweigh CfgE's second stage), C1 0.114 vs 0.163 ms (2048 tasks fit one wave
// of 148 x 16 warps; CfgE needed a second, mostly idle one), 512-B slabs lose
// (0.94 ms).
K1 fused_cfg(const GridDev&) { return K1::G; }

K1 choose_k1(const GridDev& g, const uint64_t* spec_off) {
  if (g.reverse) {  // the verify-scatter exists as a k_hash geometry only
    const int v = hash_variant();
    if (v == 7) return K1::E;
    if (v == 14) return K1::G;
    if (v == 15) return K1::H;
    if (v == 18) return K1::K;
    if (v == 19) return K1::L;
    if (v == 20) return K1::M;
    return fused_cfg(g);
  }
  switch (hash_variant()) {
    case 14: return K1::G;
    case 15: return K1::H;
    case 16: return K1::I;
    case 17: return K1::J;
    case 18: return K1::K;
    case 19: return K1::L;
    case 20: return K1::M;
    case 1: return K1::B;
    case 2: return K1::C;
    case 3: return K1::D;
    case 4: return K1::WsA;
    case 5: return K1::WsB;
    case 6: return K1::WsC;
    case 7: return K1::E;
    case 8: return K1::F;
    case 9: return K1::A;
    case 13:  // fused: TMA-load FNV kernel (CfgE geometry)
      if (spec_off) return hash_tma_ok(g) ? K1::TmaF : K1::E;
      return hash_tma_ok(g) ? K1::Tma : K1::A;
    case 11:
    case 12:  // the tensor-core kernels for every launch (hash only and fused)
      if (spec_off) return hash_mma_ok(g) ? K1::MmaFL : K1::E;
      return hash_mma_ok(g) ? K1::Mma : K1::A;
    default: {
      const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
      const uint64_t pages = (c_end - g.c_begin) << (g.chunk_shift - g.page_shift);
      // fused hash + speculative stores. Most chunks staged (single GPU, first
      // snapshot): CfgG — the mixed read/write DRAM stream bounds the pass
      // (0.74 ms on C2 vs 0.94 for the tensor-core kernel). Few staged
      // (multi-GPU striping: rank r writes its private state + 1/N of the
      // replicated state; several ranks in one buffer list): the hash dominates
      // -> tensor-core FNV with the stores fused (64-B segments) below 55 %
      // staged. Real 2-GPU runs of C2 (62 % staged): CfgG K1 0.670 ms vs 0.695
      // (6106-6123 vs 5890-5922 GB/s); at the N = 4 / 8 write fractions (44 / 38 %)
      // the tensor-core kernel wins (tools/stripe_emu.py: 0.741 / 0.703 vs ~0.83).
      if (spec_off) {
        const uint64_t grid_bytes = (c_end - g.c_begin) << g.chunk_shift;
        if (hash_mma_ok(g) && pages >= 128 * 1024 && g.spec_bytes * 100 < grid_bytes * 55)
          return K1::MmaFL;
        return fused_cfg(g);
      }
      // tensor-core FNV: one 1024-page group per SM at a time, so small grids
      // leave SMs idle (tools/hash_sizes.py: 256 MiB 2.56 vs 2.85 TB/s for the
      // TMA kernel, 384 MiB 3.75 vs 2.29, 512 MiB+ 4.8-6.0 vs 3.0-3.6)
      if (hash_mma_ok(g) && (pages >= 80 * 1024 || g.mma_cw == 81)) return K1::Mma;
      if (g.nbufs && (g.nchunks << g.chunk_shift) / g.nbufs >= (64ull << 20)) return K1::B;
      return hash_tma_ok(g) ? K1::Tma : K1::A;
    }
  }
}

int launch_k1(K1 k, const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig,
              const uint64_t* spec_off, uint8_t* staging, cudaStream_t s) {
  switch (k) {
    case K1::A: return launch_hash_cfg<CfgA>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::B: return launch_hash_cfg<CfgB>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::C: return launch_hash_cfg<CfgC>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::D: return launch_hash_cfg<CfgD>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::E: return launch_hash_cfg<CfgE>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::F: return launch_hash_cfg<CfgF>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::G: return launch_hash_cfg<CfgG>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::H: return launch_hash_cfg<CfgH>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::I: return launch_hash_cfg<CfgI>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::J: return launch_hash_cfg<CfgJ>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::K: return launch_hash_cfg<CfgK>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::L: return launch_hash_cfg<CfgL>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::M: return launch_hash_cfg<CfgM>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::WsA: return launch_hash_ws<WsA>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::WsB: return launch_hash_ws<WsB>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::WsC: return launch_hash_ws<WsC>(arena, g, chunk_dig, spec_off, staging, s);
    case K1::Tma: return launch_hash_tma(arena, g, chunk_dig, s);
    case K1::Mma: return launch_hash_mma(arena, g, chunk_dig, s);
    case K1::MmaFL: return launch_hash_mma_fused(arena, g, chunk_dig, spec_off, staging, s);
    case K1::TmaF: return launch_hash_tma_fused(arena, g, chunk_dig, spec_off, staging, s);
  }
  return 0;
}

// K1 launch; with g.dd set the K2 insert is fused into the k_hash epilogue, or
// (warp-specialized / TMA kernels) runs as a range kernel right after.
const char* k1_name(K1 k) {
  switch (k) {
    case K1::A: return "k_hash<CfgA> (FNV chain, cp.async)";
    case K1::B: return "k_hash<CfgB> (FNV chain, 2 chains/lane)";
    case K1::C: return "k_hash<CfgC>";
    case K1::D: return "k_hash<CfgD>";
    case K1::E: return "k_hash<CfgE> (FNV chain + fused K3 stores, 256-B slabs)";
    case K1::F: return "k_hash<CfgF>";
    case K1::G: return "k_hash<CfgG> (FNV chain + fused K3 stores, 16 warps x 1 stage of 256-B slabs)";
    case K1::H: return "k_hash<CfgH> (FNV chain + fused stores, 14 warps x 1 stage: one wave)";
    case K1::I: return "k_hash<CfgI> (FNV chain + fused stores, 512-B slabs, 12 warps)";
    case K1::J: return "k_hash<CfgJ> (FNV chain + fused stores, 512-B slabs, 13 warps)";
    case K1::K: return "k_hash<CfgK> (FNV chain + fused stores, 8 warps x 2 stages)";
    case K1::L: return "k_hash<CfgL> (FNV chain + fused stores, 8 warps x 3 stages)";
    case K1::M: return "k_hash<CfgM> (FNV chain + fused stores, 10 warps x 2 stages)";
    case K1::WsA: return "k_hash_ws<WsA>";
    case K1::WsB: return "k_hash_ws<WsB>";
    case K1::WsC: return "k_hash_ws<WsC>";
    case K1::Tma: return "k_hash_tma (FNV chain, TMA loads)";
    case K1::Mma: return "k_hash_mma (tensor-core FNV, hash only)";
    case K1::MmaFL: return "k_hash_mma fused-light (tensor-core FNV + fused K3 stores)";
    case K1::TmaF: return "k_hash_tma_fused (FNV chain, TMA loads + fused K3 stores)";
  }
  return "?";
}
const char* g_last_k1 = "";

int launch_hash(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig,
                const uint64_t* spec_off, uint8_t* staging, cudaStream_t s) {
  if (g.nchunks == 0) return 0;
  const K1 k = choose_k1(g, spec_off);
  g_last_k1 = k1_name(k);
  const bool epilogue = !(k == K1::WsA || k == K1::WsB || k == K1::WsC || k == K1::Tma || k == K1::Mma ||
                          k == K1::MmaFL || k == K1::TmaF);
  if (!g.dd.keys || epilogue) return launch_k1(k, arena, g, chunk_dig, spec_off, staging, s);
  GridDev h = g;
  h.dd = TableDev{};
  const int n = launch_k1(k, arena, h, chunk_dig, spec_off, staging, s);
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  uint64_t blocks = (c_end - g.c_begin + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks) k_insert_range<<<unsigned(blocks), 256, 0, s>>>(g, chunk_dig);
  return n + (blocks ? 1 : 0);
}

const char* last_k1_name() { return g_last_k1; }

bool k1_epilogue_insert(const GridDev& g, const uint64_t* spec_off) {
  const K1 k = choose_k1(g, spec_off);
  return !(k == K1::WsA || k == K1::WsB || k == K1::WsC || k == K1::Tma || k == K1::Mma ||
           k == K1::MmaFL || k == K1::TmaF);
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
