// k_hash_mma.cu — K1 hash-only on the tensor cores: FNV-1a-64 split into an
// 8-bit serial chain (CUDA cores) and a linear form (tcgen05 int8 MMA).
//
// FNV-1a step (sim.hpp:55-65): h' = (h ^ b) * P, P = 2^40 + 0x1b3.
// Write l = h mod 256 and u = l ^ b. Since h ^ b only changes the low byte,
// h ^ b = h + (u - l), so over a page of n bytes
//     h_n = h_0 P^n + sum_k (u_k - l_k) P^(n-k)            (mod 2^64)
// and the only serial dependency is the 8-bit chain
//     l_{k+1} = (u_k * 0xb3) mod 256,  u_k = l_k ^ b_k     (P = 0xb3 mod 256).
// The sum is a dot product of byte streams with fixed 64-bit weights: split
// each weight into 8 byte limbs and it is an int8 matrix product
//     D[page][limb] = sum_k u_k W_k[limb] + l_{k+1} Wl_{k+1}[limb]
// with u8 operands and s32 accumulation (max 8192 * 255 * 255 < 2^31), and
// sum_j D[j] << 8j recovers the 64-bit value mod 2^64. The CUDA cores run
// only the 8-bit chain, two pages per 32-bit register (16-bit lanes: the
// 16-bit product u * 179 < 2^16 never carries into the other lane):
//     X = PRMT(word_a, word_b)              byte k of each page -> bits 0, 16
//     U = (L ^ X) & 0x00ff00ff              LOP3
//     L = U * 179                           IMAD: low bytes = next l, the
//                                           high bytes are ignored (weight 0)
// i.e. 2 ALU + 1.5 FMA-pipe instructions per two byte-steps, against
// IMAD.WIDE + 2 IMAD (8 FMA-heavy cycles per warp) per byte-step for the
// direct 64-bit chain (k_hash.cu) — the bound of the other K1 kernels.
//
// Streams fed to the MMA (A operand in TMEM, one row = one page pair):
//   u words:  U_k + (U_{k+1} << 8)   = [u_a,k    u_a,k+1  u_b,k    u_b,k+1]
//   l words:  PRMT(L_k, L_{k+1})     = [l_a,k+1  l_a,k+2  l_b,k+1  l_b,k+2]
// B operand = the weight limbs of the batch's byte positions (N = 16: limbs
// of page a, limbs of page b), a 4 KiB slice per 64 byte-steps streamed from
// an L2-resident table by the MMA warp. After the 4096 steps of a page:
//     h = H0 P^n + P^-(4096-n) (S + l_4096 - 0x25 P^4096)
// with S = sum_j D[j] << 8j (the chain continues over zero bytes past a
// short page's end, where u = l makes every term vanish). Bit-exact with the
// reference digest: tests compare every chunk digest with the oracle.
//
// CTA = 4 compute warps (threads 0..127 = TMEM lanes 0..127; each thread
// owns 4 pages = 2 chain pairs) + 1 MMA warp. Group = 512 page slots
// (16 chunk-aligned tasks of 32 pages); warp w owns tasks 4w..4w+3 and loads
// them itself (TMA 2D box of 32 pages x 128 B per regular task, 1D bulk per
// page otherwise) into a 3-stage ring. Per 64 byte-steps the warps write
// 2 x 64 TMEM columns (3-deep ring) and the MMA warp issues 2 x 8 MMAs
// (M=128, N=16, K=32, kind::i8, A from TMEM) into per-group accumulators.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "snap_internal.h"
#include "table.cuh"

namespace snap {
namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kCW = 8;                        // compute warps (2 per SM sub-partition)
constexpr int kThreads = (kCW + 1) * 32;      // + MMA warp
constexpr int kSlab = 64;                     // bytes of a page per data stage
constexpr int kWarpStage = 4 * 32 * kSlab;    // 4 tasks x 32 pages x 64 B
constexpr int kST = 3;                        // data ring depth per warp
constexpr int kGroupPages = kCW * 128;        // page slots per group
constexpr int kStages = 4096 / kSlab;         // data stages per page
constexpr int kBSteps = 32;                   // byte-steps per MMA batch
constexpr int kBatches = 4096 / kBSteps;      // batches per 4 KiB page
constexpr int kBBytes = 16 * 128;             // one B slice: 16 rows x (64 B u | 64 B l)
constexpr int kBR = 8;                        // B-slice ring depth
// TMEM columns: kNA A buffers of 4 pair-sets x 32 columns (16 u words, 16 l
// words), then kNDB accumulator buffers of 4 pair-sets x 16 columns.
constexpr int kSets = 4, kNA = 3, kNDB = 2;
constexpr uint32_t kASet = 32, kABuf = kSets * kASet, kDCol = kNA * kABuf, kDBuf = kSets * 16;
static_assert(kDCol + kNDB * kDBuf <= 512, "TMEM budget");
constexpr uint64_t kP = 0x100000001b3ull;
// table tail (after the kBatches B slices): HP[17], IP[17], K0
constexpr size_t kBTab = size_t(kBatches) * kBBytes;
constexpr size_t kBTabAll = kBTab + (17 + 17 + 1) * 8;

constexpr size_t kSmemData = size_t(kCW) * kST * kWarpStage;
constexpr size_t kSmemB = size_t(kBR) * kBBytes;
constexpr size_t kSmemDig = size_t(kCW) * 128 * 8;
constexpr size_t kSmemZero = 128;             // zero slab: LDS source for absent pages
constexpr int kNBars = kCW * kST + kNA + kNA + kNDB + kNDB + kBR;
constexpr size_t kSmem = 1024 + kSmemData + kSmemB + kSmemDig + kSmemZero + kNBars * 8 + 16;

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
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
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

// ---- tcgen05 (TMEM, MMA) ----
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tc_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// D[tmem] (+)= A[tmem] x B[smem desc], M=128 N=16 K=32, u8 x u8 -> s32
__device__ __forceinline__ void tc_mma_i8(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}
// K-major operand, 128-byte swizzle, 8-row groups 1024 B apart (SBO)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3fff) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ uint32_t find_buf(const GridDev& g, uint64_t gc) {
  uint32_t lo = 0, hi = g.nbufs;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(g.cstart + mid) <= gc) lo = mid; else hi = mid;
  }
  return lo;
}

// FNV-1a over the 8 bytes of a page digest (chunk fold, digest_of_words)
__device__ __forceinline__ uint64_t fnv_u64(uint64_t h, uint64_t w) {
#pragma unroll
  for (int i = 0; i < 8; ++i) h = (h ^ ((w >> (8 * i)) & 0xffu)) * kP;
  return h;
}

__device__ __forceinline__ uint32_t lop_xor_and(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(r) : "r"(a), "r"(b), "r"(c));  // (a ^ b) & c
  return r;
}
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

// 16 byte-steps of one chain pair: bytes of page a from `va`, page b from `vb`.
// upk[m] = [u_a,2m u_a,2m+1 u_b,2m u_b,2m+1], lpk[m] = [l_a,2m+1 l_a,2m+2 l_b,2m+1 l_b,2m+2]
__device__ __forceinline__ void chain16(uint32_t& L, const uint4& va, const uint4& vb,
                                        uint32_t (&upk)[8], uint32_t (&lpk)[8]) {
  const uint32_t wa[4] = {va.x, va.y, va.z, va.w};
  const uint32_t wb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t sel = uint32_t(k) | (uint32_t(k) << 4) | (uint32_t(k + 4) << 8) |
                           (uint32_t(k + 4) << 12);
      const uint32_t x = __byte_perm(wa[i], wb[i], sel);
      const uint32_t u = lop_xor_and(L, x, 0x00ff00ffu);
      const uint32_t prev = L;
      L = mad_u32(u, 179u, 0u);
      if (k & 1) {
        upk[2 * i + (k >> 1)] = mad_u32(u, 256u, upk[2 * i + (k >> 1)]);
        lpk[2 * i + (k >> 1)] = __byte_perm(prev, L, 0x6240);
      } else {
        upk[2 * i + (k >> 1)] = u;
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
k_hash_mma(const uint8_t* __restrict__ arena, GridDev g, uint64_t* __restrict__ chunk_dig,
           const uint8_t* __restrict__ btab, int dbg) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // warp index through a shuffle: the compiler then treats it as warp-uniform
  // (TMEM addresses and ring offsets stay in uniform registers)
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  uint8_t* bring = smem + kSmemData;
  uint64_t* dsm = reinterpret_cast<uint64_t*>(bring + kSmemB);
  uint8_t* zero = reinterpret_cast<uint8_t*>(dsm + kCW * 128);
  uint64_t* bars = reinterpret_cast<uint64_t*>(zero + kSmemZero);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + kNBars);
  const uint32_t bar_full = smem_u32(bars);              // [kCW][kST]
  const uint32_t bar_afull = bar_full + 8 * kCW * kST;   // [kNA]
  const uint32_t bar_afree = bar_afull + 8 * kNA;        // [kNA]
  const uint32_t bar_dfull = bar_afree + 8 * kNA;        // [kNDB]
  const uint32_t bar_dfree = bar_dfull + 8 * kNDB;       // [kNDB]
  const uint32_t bar_bfull = bar_dfree + 8 * kNDB;       // [kBR]

  const uint32_t ppc_shift = g.chunk_shift - 12;
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  const uint64_t slot_base = g.c_begin << ppc_shift;
  const uint64_t nslots = (c_end - g.c_begin) << ppc_shift;
  const uint64_t ngroups = (nslots + kGroupPages - 1) / kGroupPages;
  if (blockIdx.x >= ngroups) return;
  const uint64_t ngl = (ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x;  // my groups

  if (threadIdx.x < kSmemZero / 16) reinterpret_cast<uint4*>(zero)[threadIdx.x] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kCW * kST; ++i) mbar_init(bar_full + 8 * i, 1);
    for (int i = 0; i < kNA; ++i) {
      mbar_init(bar_afull + 8 * i, kCW * 32);
      mbar_init(bar_afree + 8 * i, 1);
    }
    for (int i = 0; i < kNDB; ++i) {
      mbar_init(bar_dfull + 8 * i, 1);
      mbar_init(bar_dfree + 8 * i, kCW * 32);
    }
    for (int i = 0; i < kBR; ++i) mbar_init(bar_bfull + 8 * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kCW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == kCW) {
    // ------------------------------------------------------------ MMA warp
    // the whole warp runs the loop (warp-uniform operands stay in uniform
    // registers); one elected lane issues the TMA, MMA and commit instructions
    const uint64_t nb = ngl * kBatches;
    const uint32_t idesc = (2u << 4) | (2u << 17) | (8u << 24);  // s32; u8 x u8; N=16, M=128
    const uint32_t bring_u = smem_u32(bring);
    const bool leader = elect_one();
    auto load_b = [&](uint64_t j) {
      const uint32_t slot = static_cast<uint32_t>(j % kBR);
      if (leader) {
        mbar_arrive_tx(bar_bfull + 8 * slot, kBBytes);
        bulk_load(bring_u + slot * kBBytes, btab + (j % kBatches) * kBBytes, kBBytes,
                  bar_bfull + 8 * slot);
      }
    };
    for (uint64_t j = 0; j < kBR && j < nb; ++j) load_b(j);
    for (uint64_t gb = 0; gb < nb; ++gb) {
      const uint64_t i = gb / kBatches;
      const uint32_t b = static_cast<uint32_t>(gb % kBatches);
      const uint32_t ab = static_cast<uint32_t>(gb % kNA), db = static_cast<uint32_t>(i % kNDB);
      if (b == 0 && i >= kNDB)
        mbar_wait(bar_dfree + 8 * db, static_cast<uint32_t>((i / kNDB - 1) & 1));
      mbar_wait(bar_afull + 8 * ab, static_cast<uint32_t>((gb / kNA) & 1));
      // A buffer gb % kNA was refilled only after batch gb - kNA's MMAs
      // completed, so that batch's B slot is free: refill it kBR ahead
      if (gb >= kNA && gb - kNA + kBR < nb) load_b(gb - kNA + kBR);
      mbar_wait(bar_bfull + 8 * (gb % kBR), static_cast<uint32_t>((gb / kBR) & 1));
      tc_fence_after();
      if (leader) {
        const uint64_t bdesc = sw128_desc(bring_u + static_cast<uint32_t>(gb % kBR) * kBBytes);
        const uint32_t dcol = tbase + kDCol + db * kDBuf, acol = tbase + ab * kABuf;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int ps = 0; ps < kSets; ++ps)
            if (!(dbg & 2))
              tc_mma_i8(dcol + ps * 16, acol + ps * kASet + 8 * kk, bdesc + uint64_t(2 * kk), idesc,
                        (b > 0 || kk > 0) ? 1u : 0u);
        tc_commit(bar_afree + 8 * ab);
        if (b == kBatches - 1) tc_commit(bar_dfull + 8 * db);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------- compute warps
    // warp w: tasks 4w..4w+3 of each group; pair sets 2 (w / 4) + {0, 1}
    // in TMEM lanes 32 (w % 4) + lane
    const CUtensorMap* maps = static_cast<const CUtensorMap*>(g.tmaps64);
    const uint32_t ring = smem_u32(smem + warp * kST * kWarpStage);
    const uint32_t fbar = bar_full + 8 * warp * kST;
    const uint32_t trow = tbase + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                          static_cast<uint32_t>(warp >> 2) * 2 * kASet;
    const uint32_t drow = tbase + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + kDCol +
                          static_cast<uint32_t>(warp >> 2) * 32;
    const uint32_t nst = static_cast<uint32_t>(ngl) * kStages;  // data stages of this warp
    const uint64_t* htab = reinterpret_cast<const uint64_t*>(btab + kBTab);

    // producer state of the group being loaded
    uint32_t p_reg = 0, p_map[4] = {0, 0, 0, 0}, p_row[4] = {0, 0, 0, 0}, p_len[4];
    const uint8_t* p_src[4];
    uint32_t reg_bits[2] = {0, 0};  // per group parity: bit q = task q loaded by TMA 2D
    uint32_t ist = 0, cst = 0;

    auto page_info = [&](uint32_t i, int q, const uint8_t*& src, uint32_t& len, uint32_t& b,
                         uint32_t& row) {
      const uint64_t gi = blockIdx.x + uint64_t(i) * gridDim.x;
      const uint64_t rel = gi * kGroupPages + 128 * warp + 32 * q + lane;
      src = nullptr;
      len = 0;
      b = 0xffffffffu;
      row = 0;
      if (rel < nslots) {
        const uint64_t slot = slot_base + rel;
        const uint64_t gc = slot >> ppc_shift;
        b = find_buf(g, gc);
        const uint64_t k = gc - __ldg(g.cstart + b);
        const uint64_t off = (k << g.chunk_shift) + ((slot & ((1u << ppc_shift) - 1)) << 12);
        const uint64_t bytes = __ldg(g.bytes + b);
        if (off < bytes) {
          const uint64_t rem = bytes - off;
          len = static_cast<uint32_t>(rem < 4096 ? rem : 4096);
          src = arena + __ldg(g.addr + b) + off;
          row = static_cast<uint32_t>(off >> 12);
        }
      }
    };

    auto issue = [&](uint32_t p) {
      const uint32_t st = ist;
      ist = ist + 1 == kST ? 0 : ist + 1;
      if (p >= nst) return;
      const uint32_t i = p / kStages;
      const uint32_t s = p % kStages;
      if (s == 0) {
        p_reg = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t b, row;
          page_info(i, q, p_src[q], p_len[q], b, row);
          const uint32_t b0 = __shfl_sync(kFull, b, 0);
          const uint32_t r0 = __shfl_sync(kFull, row, 0);
          if (__all_sync(kFull, b == b0 && p_len[q] == 4096 && row == r0 + lane)) p_reg |= 1u << q;
          p_map[q] = b0;
          p_row[q] = r0;
        }
        reg_bits[i & 1] = p_reg;
      }
      const uint32_t bar = fbar + 8 * st;
      const uint32_t dst = ring + st * kWarpStage;
      if (p_reg == 0xfu) {
        // regular group: four TMA boxes, one elected lane
        if (lane == 0) {
          mbar_arrive_tx(bar, 4 * 32 * kSlab);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            tma_load_2d(dst + q * 32 * kSlab, maps + p_map[q], static_cast<int>(s * kSlab),
                        static_cast<int>(p_row[q]), bar);
        }
        return;
      }
      uint32_t tx = 0;
      uint32_t vmask[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        vmask[q] = __ballot_sync(kFull, s * kSlab < p_len[q]);
        tx += (p_reg >> q) & 1 ? 32u * kSlab : __popc(vmask[q]) * kSlab;
      }
      if (lane == 0) mbar_arrive_tx(bar, tx);
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if ((p_reg >> q) & 1) {
          if (lane == 0)
            tma_load_2d(dst + q * 32 * kSlab, maps + p_map[q], static_cast<int>(s * kSlab),
                        static_cast<int>(p_row[q]), bar);
        } else if ((vmask[q] >> lane) & 1) {
          bulk_load(dst + q * 32 * kSlab + lane * kSlab, p_src[q] + s * kSlab, kSlab, bar);
        }
      }
    };

#pragma unroll
    for (int p = 0; p < kST - 1; ++p) issue(p);

    uint32_t c_len[4] = {0, 0, 0, 0};
    uint32_t L0 = 0, L1 = 0;
    bool c_full = false;  // every page of the group is a full page of a TMA-loaded task
    const uint32_t zbase = smem_u32(zero);
    // SWIZZLE_64B: 16-B unit u of box row j lives at unit u ^ ((j >> 1) & 3)
    const uint32_t swz = static_cast<uint32_t>((lane >> 1) & 3) << 4;
    uint32_t ph_full = 0;  // parity of the data ring's next wrap
    for (uint32_t p = 0; p < nst; ++p) {
      issue(p + kST - 1);
      const uint32_t st = cst;
      cst = cst + 1 == kST ? 0 : cst + 1;
      const uint32_t i = p / kStages;
      const uint32_t s = p % kStages;
      if (s == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint8_t* src;
          uint32_t b, row;
          page_info(i, q, src, c_len[q], b, row);
        }
        c_full = reg_bits[i & 1] == 0xfu;
        L0 = L1 = 0x00250025u;  // l_0 = low byte of the FNV offset basis, both lanes
      }
      mbar_wait(fbar + 8 * st, ph_full);
      if (st == kST - 1) ph_full ^= 1u;
      // per page: slab address with its swizzle bits (unit uu at addr ^ (uu << 4));
      // pages without bytes in this stage read the zero slab (their chain
      // continues over zeros, which adds nothing to the digest sum)
      const uint32_t sbase = ring + st * kWarpStage + lane * kSlab;
      uint32_t pa[4];
      if (c_full) {
#pragma unroll
        for (int q = 0; q < 4; ++q) pa[q] = (sbase + q * 32 * kSlab) | swz;
      } else {
        const uint32_t rb = reg_bits[i & 1];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          pa[q] = s * kSlab < c_len[q] ? (sbase + q * 32 * kSlab) | ((rb >> q) & 1 ? swz : 0u) : zbase;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t gb = 2 * p + h;
        const uint32_t ab = gb % kNA;
        if (gb >= kNA) mbar_wait(bar_afree + 8 * ab, (gb / kNA - 1) & 1);
        tc_fence_after();
        const uint32_t acol = trow + ab * kABuf;
#pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
          const uint32_t unit = 2 * h + uu;
          uint4 v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) v[q] = ld_shared16(pa[q] ^ (unit << 4));
          uint32_t upk0[8], lpk0[8], upk1[8], lpk1[8];
          if (dbg & 1) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              upk0[j] = v[0].x + j; lpk0[j] = v[1].y + j; upk1[j] = v[2].z + j; lpk1[j] = v[3].w + j;
            }
          } else {
            chain16(L0, v[0], v[1], upk0, lpk0);
            chain16(L1, v[2], v[3], upk1, lpk1);
          }
          tc_st8(acol + 8 * uu, upk0);
          tc_st8(acol + 16 + 8 * uu, lpk0);
          tc_st8(acol + kASet + 8 * uu, upk1);
          tc_st8(acol + kASet + 16 + 8 * uu, lpk1);
        }
        tc_wait_st();
        tc_fence_before();
        mbar_arrive(bar_afull + 8 * ab);
      }
      __syncwarp();  // the stage slot is refilled by this warp's next issue
      if (s == kStages - 1) {
        // ---- epilogue of group i: accumulators -> page digests -> chunk digests
        const uint32_t db = i % kNDB;
        mbar_wait(bar_dfull + 8 * db, (i / kNDB) & 1);
        tc_fence_after();
        uint32_t d[32];  // d[16 ps + 8 pg + j] = limb j of page (pair ps, lane pg)
        tc_ld32(drow + db * kDBuf, d);
        tc_fence_before();
        mbar_arrive(bar_dfree + 8 * db);
        const uint64_t k0 = __ldg(htab + 34);
        uint32_t vm[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int ps = q >> 1, pg = q & 1;
          uint64_t S = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) S += static_cast<uint64_t>(d[16 * ps + 8 * pg + j]) << (8 * j);
          const uint32_t Lf = ps ? L1 : L0;
          const uint64_t ln = (Lf >> (16 * pg)) & 0xffu;
          const uint32_t n = c_len[q];
          uint64_t hv = 0;
          if (n > 0) {
            const uint32_t m = n >> 8;
            hv = __ldg(htab + m) + __ldg(htab + 17 + m) * (S + ln - k0);
          }
          dsm[warp * 128 + 32 * q + lane] = hv;
          vm[q] = __ballot_sync(kFull, n > 0);
        }
        __syncwarp();
        const uint64_t gi = blockIdx.x + uint64_t(i) * gridDim.x;
        const uint64_t slot0 = slot_base + gi * kGroupPages + 128 * warp;
        const uint32_t ppc = 1u << ppc_shift;
        for (uint32_t c = lane; c < (128u >> ppc_shift); c += 32) {
          const uint32_t p0 = c << ppc_shift;
          const uint32_t q0 = p0 >> 5;
          const uint32_t vq = q0 == 0 ? vm[0] : q0 == 1 ? vm[1] : q0 == 2 ? vm[2] : vm[3];
          if (!((vq >> (p0 & 31)) & 1)) continue;
          uint64_t hv;
          if (ppc_shift == 0) {
            hv = dsm[warp * 128 + p0];
          } else {
            // a chunk's pages lie in one task (ppc <= 32): valid pages are a prefix
            hv = kFnvOffset;
            for (uint32_t j = 0; j < ppc; ++j) {
              if (!((vq >> ((p0 + j) & 31)) & 1)) break;
              hv = fnv_u64(hv, dsm[warp * 128 + p0 + j]);
            }
          }
          k1_store_digest(g, (slot0 + p0) >> ppc_shift, hv, chunk_dig);
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kCW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
  if (g.xdig != nullptr) __threadfence_system();
}

// ---- host: weight-limb table ----
uint64_t powP(uint64_t e) {
  uint64_t r = 1, b = kP;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}
uint64_t inv64(uint64_t a) {  // a odd: Newton iteration mod 2^64
  uint64_t x = a;
  for (int i = 0; i < 6; ++i) x *= 2 - a * x;
  return x;
}

std::vector<uint8_t> make_btab() {
  std::vector<uint8_t> t(kBTabAll, 0);
  // logical B[n][kb] (n < 16, kb < 128) of batch bi -> SW128 K-major image:
  // 16 rows x 128 B, 16-B unit swizzled by n & 7
  auto put = [&](int bi, int n, int kb, uint8_t v) {
    const int c = kb >> 7, x = kb & 127;
    t[size_t(bi) * kBBytes + c * 2048 + n * 128 + ((((x >> 4) ^ (n & 7))) << 4) + (x & 15)] = v;
  };
  for (int bi = 0; bi < kBatches; ++bi) {
    const int t0 = kBSteps * bi;
    for (int m = 0; m < kBSteps / 2; ++m)
      for (int j = 0; j < 4; ++j) {
        const int pg = j >> 1, dt = j & 1;
        // u word m: [u_a,2m u_a,2m+1 u_b,2m u_b,2m+1] -> weight P^(4096 - t)
        const uint64_t wu = powP(uint64_t(4096 - (t0 + 2 * m + dt)));
        // l word m: [l_a,2m+1 l_a,2m+2 l_b,2m+1 l_b,2m+2] -> weight -P^(4096 - t)
        const uint64_t wl = 0 - powP(uint64_t(4096 - (t0 + 2 * m + 1 + dt)));
        for (int n = 0; n < 8; ++n) {
          put(bi, 8 * pg + n, 4 * m + j, uint8_t(wu >> (8 * n)));
          put(bi, 8 * pg + n, 2 * kBSteps + 4 * m + j, uint8_t(wl >> (8 * n)));
        }
      }
  }
  uint64_t* tail = reinterpret_cast<uint64_t*>(t.data() + kBTab);
  const uint64_t pinv = inv64(kP);
  for (int m = 0; m <= 16; ++m) {
    uint64_t ip = 1;
    for (int e = 0; e < 4096 - 256 * m; ++e) ip *= pinv;
    tail[m] = kFnvOffset * powP(uint64_t(256 * m));
    tail[17 + m] = ip;
  }
  tail[34] = 0x25ull * powP(4096);
  return t;
}

const uint8_t* device_btab() {
  static const uint8_t* tabs[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!tabs[dev]) {
    const std::vector<uint8_t> h = make_btab();
    void* d = nullptr;
    if (cudaMalloc(&d, h.size()) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    tabs[dev] = static_cast<const uint8_t*>(d);
  }
  return tabs[dev];
}

}  // namespace

bool hash_mma_ok(const GridDev& g) {
  return g.tmaps64 != nullptr && g.page_shift == 12 && g.chunk_shift >= 12 && g.chunk_shift <= 17;
}

int launch_hash_mma(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_hash_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmem));
    attr = true;
  }
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  if (c_end <= g.c_begin) return 0;
  const uint8_t* bt = device_btab();
  if (!bt) return -1;
  const uint64_t ngroups = (((c_end - g.c_begin) << (g.chunk_shift - 12)) + kGroupPages - 1) / kGroupPages;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t blocks = ngroups < uint64_t(sms) ? ngroups : uint64_t(sms);
  static const int dbg = getenv("SNAP_MMA_DEBUG") ? atoi(getenv("SNAP_MMA_DEBUG")) : 0;
  k_hash_mma<<<unsigned(blocks), kThreads, kSmem, s>>>(arena, g, chunk_dig, bt, dbg);
  return 1;
}

}  // namespace snap
