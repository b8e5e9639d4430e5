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
// CTA = 8 compute warps (threads 0..255; warp w writes TMEM lanes 32 (w % 4)
// + lane; each thread owns 4 pages = 2 chain pairs) + 1 MMA warp. Group =
// 1024 page slots (32 chunk-aligned tasks of 32 pages); warp w owns 4 tasks and
// loads them itself into a 3-stage ring (64-byte slabs): one TMA 2D box of
// 32 rows x 64 B per task that is contiguous in memory, one box per chunk
// otherwise (16 arena-wide tensor maps, one per 256-byte alignment class of a
// page start), per-page bulk copies only for chunk sizes below 8 pages. Per
// 32 byte-steps the warps write 4 pair-sets x 32 TMEM columns (3-deep ring)
// and the MMA warp issues 16 MMAs (M=128, N=16, K=32, kind::i8, A from TMEM)
// into double-buffered accumulators. The fused variant also stores each
// hashed slab of a predicted-staged page to the staging image.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "snap_internal.h"
#include "table.cuh"

namespace snap {
namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kBSteps = 32;                   // byte-steps per MMA batch
constexpr int kBatches = 4096 / kBSteps;      // batches per 4 KiB page
constexpr int kBBytes = 16 * 128;             // one B slice: 16 rows x (64 B u | 64 B l)
constexpr int kBR = 8;                        // B-slice ring depth
constexpr uint64_t kP = 0x100000001b3ull;
// table tail (after the kBatches B slices): HP[17], IP[17], K0
constexpr size_t kBTab = size_t(kBatches) * kBBytes;
constexpr size_t kBTabAll = kBTab + (17 + 17 + 1) * 8;

// Kernel geometry. CW compute warps (a multiple of 4: TMEM lane quadrants),
// PAIRS chain pairs per thread, SLAB bytes of each page per data stage (TMA
// boxes of 32 pages x BOXW bytes, SWIZZLE_64B / _128B), ST-deep ring per
// warp, FUSED: also write every predicted-staged chunk's slab to staging.
template <int CW_, int PAIRS_, int SLAB_, int ST_, bool FUSED_, int NA_ = 3, int NDB_ = 2>
struct MmaCfg {
  static constexpr int CW = CW_, PAIRS = PAIRS_, SLAB = SLAB_, ST = ST_;
  static constexpr bool FUSED = FUSED_;
  static constexpr int TPW = 2 * PAIRS;                 // 32-page tasks per warp
  static constexpr int PPW = 32 * TPW;                  // pages per warp
  static constexpr int GP = CW * PPW;                   // page slots per group
  static constexpr int BOXW = SLAB >= 128 ? 128 : 64;   // box width = swizzle span
  static constexpr int NBOX = SLAB / BOXW;              // boxes per task and stage
  static constexpr int SUB = 32 * BOXW;                 // bytes of one box
  static constexpr int TASKB = NBOX * SUB;              // bytes per task and stage
  static constexpr int WSTAGE = TPW * TASKB;            // bytes per warp and stage
  static constexpr int STAGES = 4096 / SLAB;            // data stages per page
  static constexpr int UNITS = SLAB / 16;               // 16-B units per page and stage
  static constexpr int UPB = BOXW / 16;                 // units per box row
  static constexpr int BPS = UNITS / 2;                 // 32-step batches per stage
  static constexpr int SETS = (CW / 4) * PAIRS;         // pair sets (M = 128 rows each)
  static constexpr int NA = NA_, NDB = NDB_;             // A ring, accumulator buffers
  static constexpr uint32_t ASET = 32, ABUF = SETS * ASET, DCOL = NA * ABUF, DBUF = SETS * 16;
  static constexpr uint32_t TUSED = DCOL + NDB * DBUF;
  static constexpr uint32_t TCOLS = TUSED <= 32 ? 32 : TUSED <= 64 ? 64 : TUSED <= 128 ? 128
                                  : TUSED <= 256 ? 256 : 512;
  static_assert(TUSED <= 512, "TMEM budget");
  static constexpr int THREADS = (CW + 1) * 32;         // + MMA warp
  static constexpr size_t SM_DATA = size_t(CW) * ST * WSTAGE;
  static constexpr size_t SM_B = size_t(kBR) * kBBytes;
  static constexpr size_t SM_DIG = size_t(GP) * 8;
  static constexpr size_t SM_ZERO = 128;                // zero slab: LDS source for absent pages
  static constexpr size_t SM_CTAB = size_t(CW) * (TPW * 16 + 4) * 4;  // per-warp TMA issue plan
  static constexpr int NBARS = CW * ST + NA + NA + NDB + NDB + kBR;
  static constexpr size_t SMEM = 1024 + SM_DATA + SM_B + SM_DIG + SM_ZERO + SM_CTAB + NBARS * 8 + 16;
  static_assert(SMEM <= 232448, "shared memory");
};
// hash only: 1024 pages in flight per SM (2 chain pairs per thread, 2 warps
// per SM sub-partition) for latency hiding; 64-byte slabs keep 3 stages in
// shared memory. Fused, few chunks staged (multi-GPU striping, the default
// when the predicted staging is < 55 % of the grid): the same geometry, each
// stage's staged slabs written right after it is hashed (64-byte segments,
// full prefetch depth). (Measured and dropped: 8 warps x 1 pair with 128-byte
// slabs and 128/256-byte segments, 3-7 % slower at the N = 2..8 write fractions.)
using MmaHash = MmaCfg<8, 2, 64, 3, false>;
using MmaFusedLight = MmaCfg<8, 2, 64, 3, true>;
// 12 chain warps = 1536 pages in flight per SM; TMEM (480 of 512 columns) and
// shared memory (2 stages) pay for the extra warps (forced only, SNAP_MMA_CW=12)
using MmaHash12 = MmaCfg<12, 2, 64, 2, false, 2, 1>;
// default (mma_cw_for): 16 chain warps x 1 chain pair, same 1024-page groups
using MmaHash16 = MmaCfg<16, 1, 64, 3, false, 3, 2>;
using MmaFused16 = MmaCfg<16, 1, 64, 3, true, 3, 2>;
// small hash-only grids (mma_cw_for): 512-page groups (8 chain warps x 1 pair)
using MmaHash8x1 = MmaCfg<8, 1, 64, 3, false, 3, 2>;
using MmaFused8x1 = MmaCfg<8, 1, 64, 3, true, 3, 2>;

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
__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_stream16(uint8_t* p, uint4 v) {
  __stcs(reinterpret_cast<uint4*>(p), v);  // evict-first: the staging image is not re-read soon
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
  if (g.chunk_buf) return __ldg(g.chunk_buf + gc);
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

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
k_hash_mma(const uint8_t* __restrict__ arena, GridDev g, uint64_t* __restrict__ chunk_dig,
           const uint8_t* __restrict__ btab, const uint64_t* __restrict__ spec_off,
           uint8_t* __restrict__ staging, int dbg) {
  constexpr int CW = C::CW, ST = C::ST, NA = C::NA, NDB = C::NDB, GP = C::GP, PPW = C::PPW;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // warp index through a shuffle: the compiler then treats it as warp-uniform
  // (TMEM addresses and ring offsets stay in uniform registers)
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  uint8_t* bring = smem + C::SM_DATA;
  uint64_t* dsm = reinterpret_cast<uint64_t*>(bring + C::SM_B);
  uint8_t* zero = reinterpret_cast<uint8_t*>(dsm + GP);
  uint32_t* ctab_all = reinterpret_cast<uint32_t*>(zero + C::SM_ZERO);
  uint64_t* bars = reinterpret_cast<uint64_t*>(zero + C::SM_ZERO + C::SM_CTAB);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + C::NBARS);
  const uint32_t bar_full = smem_u32(bars);              // [CW][ST]
  const uint32_t bar_afull = bar_full + 8 * CW * ST;     // [NA]
  const uint32_t bar_afree = bar_afull + 8 * NA;         // [NA]
  const uint32_t bar_dfull = bar_afree + 8 * NA;         // [NDB]
  const uint32_t bar_dfree = bar_dfull + 8 * NDB;        // [NDB]
  const uint32_t bar_bfull = bar_dfree + 8 * NDB;        // [kBR]

  const uint32_t ppc_shift = g.chunk_shift - 12;
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  const uint64_t slot_base = g.c_begin << ppc_shift;
  const uint64_t nslots = (c_end - g.c_begin) << ppc_shift;
  const uint64_t ngroups = (nslots + GP - 1) / GP;
  if (blockIdx.x >= ngroups) return;
  // my groups: the grid's balanced schedule (mma_schedule), else round robin
  // (recomputed from the kernel parameter at each use: no registers held;
  // hash-only variant only — the fused one stays at its register budget)
  const uint32_t* gs = C::FUSED ? nullptr : g.gsched;
  const uint64_t ngl = gs ? __ldg(gs + blockIdx.x + 1) - __ldg(gs + blockIdx.x)
                          : (ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x;
  auto group_of = [&g](uint32_t i) -> uint64_t {
    return !C::FUSED && g.gsched ? __ldg(g.gsched + gridDim.x + 1 + __ldg(g.gsched + blockIdx.x) + i)
                                 : blockIdx.x + uint64_t(i) * gridDim.x;
  };

  if (threadIdx.x < C::SM_ZERO / 16) reinterpret_cast<uint4*>(zero)[threadIdx.x] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < CW * ST; ++i) mbar_init(bar_full + 8 * i, 1);
    for (int i = 0; i < NA; ++i) {
      mbar_init(bar_afull + 8 * i, CW * 32);
      mbar_init(bar_afree + 8 * i, 1);
    }
    for (int i = 0; i < NDB; ++i) {
      mbar_init(bar_dfull + 8 * i, 1);
      mbar_init(bar_dfree + 8 * i, CW * 32);
    }
    for (int i = 0; i < kBR; ++i) mbar_init(bar_bfull + 8 * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == CW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)), "n"(C::TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == CW) {
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
      const uint32_t ab = static_cast<uint32_t>(gb % NA), db = static_cast<uint32_t>(i % NDB);
      if (b == 0 && i >= NDB)
        mbar_wait(bar_dfree + 8 * db, static_cast<uint32_t>((i / NDB - 1) & 1));
      mbar_wait(bar_afull + 8 * ab, static_cast<uint32_t>((gb / NA) & 1));
      // A buffer gb % NA was refilled only after batch gb - NA's MMAs
      // completed, so that batch's B slot is free: refill it kBR ahead
      if (gb >= NA && gb - NA + kBR < nb) load_b(gb - NA + kBR);
      mbar_wait(bar_bfull + 8 * (gb % kBR), static_cast<uint32_t>((gb / kBR) & 1));
      tc_fence_after();
      if (leader) {
        const uint64_t bdesc = sw128_desc(bring_u + static_cast<uint32_t>(gb % kBR) * kBBytes);
        const uint32_t dcol = tbase + C::DCOL + db * C::DBUF, acol = tbase + ab * C::ABUF;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int ps = 0; ps < C::SETS; ++ps)
            if (!(dbg & 2))
              tc_mma_i8(dcol + ps * 16, acol + ps * C::ASET + 8 * kk, bdesc + uint64_t(2 * kk),
                        idesc, (b > 0 || kk > 0) ? 1u : 0u);
        tc_commit(bar_afree + 8 * ab);
        if (b == kBatches - 1) tc_commit(bar_dfull + 8 * db);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------- compute warps
    // warp w: tasks TPW*w .. TPW*w + TPW-1 of each group; chain pair p of a
    // thread = pages (task 2p, task 2p+1) at its lane; TMEM pair set
    // (w / 4) * PAIRS + p in lanes 32 (w % 4) + lane
    constexpr int TPW = C::TPW, PAIRS = C::PAIRS, SLAB = C::SLAB, BOXW = C::BOXW;
    static_assert(BOXW == 64, "the arena-wide maps have 64-byte boxes");
    const CUtensorMap* maps = static_cast<const CUtensorMap*>(g.tmaps64);
    const uint32_t ring = smem_u32(smem + warp * ST * C::WSTAGE);
    const uint32_t fbar = bar_full + 8 * warp * ST;
    const uint32_t tl = static_cast<uint32_t>(32 * (warp & 3)) << 16;
    const uint32_t trow = tbase + tl + static_cast<uint32_t>(warp >> 2) * PAIRS * C::ASET;
    const uint32_t drow = tbase + tl + C::DCOL + static_cast<uint32_t>(warp >> 2) * PAIRS * 16;
    const uint32_t nst = static_cast<uint32_t>(ngl) * C::STAGES;  // data stages of this warp
    const uint64_t* htab = reinterpret_cast<const uint64_t*>(btab + kBTab);

    // producer state of the group being loaded
    uint32_t p_reg = 0, p_chk = 0, p_map[TPW], p_row[TPW], p_len[TPW];
    // tasks that are not 32 contiguous full pages load one TMA box per chunk
    // (the arena-wide chunk-box maps), replayed from the warp's issue plan
    const CUtensorMap* cmaps = static_cast<const CUtensorMap*>(g.tmaps64c);
    const bool cbox = BOXW == 64 && C::NBOX == 1 && cmaps != nullptr;
    // per-group TMA issue plan of a warp whose tasks are not all regular: up to
    // TPW * 4 boxes {map pointer, row, stage offset}, issued by lane 0 each stage
    // (entry 0 of the table: {count, tx bytes}; boxes from entry 1)
    uint32_t* plan = ctab_all + warp * (TPW * 16 + 4);
    const uint8_t* p_src[TPW];
    uint32_t reg_bits[2] = {0, 0};   // per group parity: bit t = task t loaded by TMA 2D (swizzled)
    uint32_t full_bits[2] = {0, 0};  // per group parity: bit t = task t is 32 full pages
    uint32_t ist = 0, cst = 0;

    auto page_info = [&](uint32_t i, int t, const uint8_t*& src, uint32_t& len, uint32_t& b,
                         uint32_t& row, uint64_t& gcout) {
      const uint64_t gi = group_of(i);
      const uint64_t rel = gi * GP + PPW * warp + 32 * t + lane;
      src = nullptr;
      len = 0;
      b = 0xffffffffu;
      row = 0;
      gcout = ~0ull;
      if (rel < nslots) {
        const uint64_t slot = slot_base + rel;
        const uint64_t gc = slot >> ppc_shift;
        uint64_t ca;
        uint32_t clen;
        chunk_loc(g, gc, ca, clen);
        const uint64_t in_chunk = (slot & ((1u << ppc_shift) - 1)) << 12;
        if (in_chunk < clen) {
          const uint64_t rem = clen - in_chunk;
          len = static_cast<uint32_t>(rem < 4096 ? rem : 4096);
          src = arena + ca + in_chunk;
          gcout = gc;
        }
      }
    };

    auto issue = [&](uint32_t p) {
      const uint32_t st = ist;
      ist = ist + 1 == ST ? 0 : ist + 1;
      if (p >= nst) return;
      const uint32_t i = p / C::STAGES;
      const uint32_t s = p % C::STAGES;
      if (s == 0) {
        p_reg = 0;
        p_chk = 0;
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          uint32_t b, row;
          uint64_t gc;
          page_info(i, t, p_src[t], p_len[t], b, row, gc);
          // arena-wide maps: a page at arena offset a is row a >> 12 of the
          // map of its 256-B alignment class (a >> 8) & 15
          const uint64_t ao = p_len[t] ? static_cast<uint64_t>(p_src[t] - arena) : 0;
          const uint64_t a0 = __shfl_sync(kFull, ao, 0);
          if (__all_sync(kFull, p_len[t] == 4096 && ao == a0 + uint64_t(lane) * 4096))
            p_reg |= 1u << t;
          p_map[t] = static_cast<uint32_t>(a0 >> 8) & 15u;
          p_row[t] = static_cast<uint32_t>(a0 >> 12);
          if (cbox && !((p_reg >> t) & 1)) p_chk |= 1u << t;  // one box per chunk
        }
        reg_bits[i & 1] = p_reg | p_chk;
        full_bits[i & 1] = p_reg;
        // issue plan (uniform): one box per regular task, one per valid chunk
        // of a chunk-box task; per-page bulk copies otherwise (generic path)
        uint32_t p_nplan = 1, p_tx = 0;
        if (p_reg != (1u << TPW) - 1 && (p_reg | p_chk) == (1u << TPW) - 1) {
#pragma unroll
          for (int t = 0; t < TPW; ++t) {
            const uint64_t ao = p_len[t] ? static_cast<uint64_t>(p_src[t] - arena) : 0;
            if ((p_reg >> t) & 1) {
              if (lane == 0) {
                const uint64_t mp = reinterpret_cast<uint64_t>(maps + p_map[t]);
                plan[p_nplan * 4] = static_cast<uint32_t>(mp);
                plan[p_nplan * 4 + 1] = static_cast<uint32_t>(mp >> 32);
                plan[p_nplan * 4 + 2] = p_row[t];
                plan[p_nplan * 4 + 3] = t * C::TASKB;
              }
              ++p_nplan;
              p_tx += C::TASKB;
            } else {
              const uint32_t halves = 32u >> ppc_shift;
#pragma unroll
              for (uint32_t hh = 0; hh < 4; ++hh) {
                if (hh < halves) {
                  const int src = static_cast<int>(hh << ppc_shift);
                  const uint64_t ah = __shfl_sync(kFull, ao, src);
                  const uint32_t vh = __shfl_sync(kFull, p_len[t] > 0 ? 1u : 0u, src);
                  if (vh) {
                    if (lane == 0) {
                      const uint64_t mp =
                          reinterpret_cast<uint64_t>(cmaps + (static_cast<uint32_t>(ah >> 8) & 15u));
                      plan[p_nplan * 4] = static_cast<uint32_t>(mp);
                      plan[p_nplan * 4 + 1] = static_cast<uint32_t>(mp >> 32);
                      plan[p_nplan * 4 + 2] = static_cast<uint32_t>(ah >> 12);
                      plan[p_nplan * 4 + 3] = t * C::TASKB + (hh << ppc_shift) * BOXW;
                    }
                    ++p_nplan;
                    p_tx += BOXW << ppc_shift;
                  }
                }
              }
            }
          }
          if (lane == 0) {
            plan[0] = p_nplan - 1;
            plan[1] = p_tx;
          }
        }
      }
      const uint32_t bar = fbar + 8 * st;
      const uint32_t dst = ring + st * C::WSTAGE;
      if (p_reg == (1u << TPW) - 1) {
        // regular group: one elected lane, NBOX TMA boxes per task
        if (lane == 0) {
          mbar_arrive_tx(bar, C::WSTAGE);
#pragma unroll
          for (int t = 0; t < TPW; ++t)
#pragma unroll
            for (int x = 0; x < C::NBOX; ++x)
              tma_load_2d(dst + t * C::TASKB + x * C::SUB, maps + p_map[t],
                          static_cast<int>(s * SLAB + x * BOXW), static_cast<int>(p_row[t]), bar);
        }
        return;
      }
      if ((p_reg | p_chk) == (1u << TPW) - 1) {
        // mixed regular / chunk-box group: the plan, one elected lane
        if (lane == 0) {
          const uint32_t np = plan[0];
          mbar_arrive_tx(bar, plan[1]);
          for (uint32_t e = 1; e <= np; ++e) {
            const uint4 pe = *reinterpret_cast<const uint4*>(plan + e * 4);
            const void* mp = reinterpret_cast<const void*>((uint64_t(pe.y) << 32) | pe.x);
            tma_load_2d(dst + pe.w, mp, static_cast<int>(s * SLAB), static_cast<int>(pe.z), bar);
          }
        }
        return;
      }
      uint32_t tx = 0;
      uint32_t vmask[TPW];
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        vmask[t] = __ballot_sync(kFull, s * SLAB < p_len[t]);
        tx += (p_reg >> t) & 1 ? uint32_t(C::TASKB) : __popc(vmask[t]) * SLAB;
      }
      if (lane == 0) mbar_arrive_tx(bar, tx);
      __syncwarp();
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        if ((p_reg >> t) & 1) {
          if (lane == 0)
#pragma unroll
            for (int x = 0; x < C::NBOX; ++x)
              tma_load_2d(dst + t * C::TASKB + x * C::SUB, maps + p_map[t],
                          static_cast<int>(s * SLAB + x * BOXW), static_cast<int>(p_row[t]), bar);
        } else if ((vmask[t] >> lane) & 1) {
#pragma unroll
          for (int x = 0; x < C::NBOX; ++x)
            bulk_load(dst + t * C::TASKB + x * C::SUB + lane * BOXW, p_src[t] + s * SLAB + x * BOXW,
                      BOXW, bar);
        }
      }
    };

#pragma unroll
    for (int p = 0; p < ST - 1; ++p) issue(p);

    uint32_t c_len[TPW];
    uint8_t* c_dst[TPW];  // FUSED: staging address of this lane's page, or null
    uint32_t L[PAIRS];
    bool c_full = false;  // every page of the group is a full page of a TMA-loaded task
    const uint32_t zbase = smem_u32(zero);
    // box row j: 16-B unit x stored at x ^ (j & 7) (SWIZZLE_128B) or
    // x ^ ((j >> 1) & 3) (SWIZZLE_64B)
    const uint32_t swz = static_cast<uint32_t>(BOXW == 128 ? (lane & 7) : ((lane >> 1) & 3)) << 4;
    uint32_t ph_full = 0;  // parity of the data ring's current wrap
    for (uint32_t p = 0; p < nst; ++p) {
      issue(p + ST - 1);
      const uint32_t st = cst;
      cst = cst + 1 == ST ? 0 : cst + 1;
      const uint32_t i = p / C::STAGES;
      const uint32_t s = p % C::STAGES;
      if (s == 0) {
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          const uint8_t* src;
          uint32_t b, row;
          uint64_t gc;
          page_info(i, t, src, c_len[t], b, row, gc);
          c_dst[t] = nullptr;
          if (C::FUSED && gc != ~0ull) {
            const uint64_t so = __ldg(spec_off + gc);
            if (so != ~0ull) {
              const uint64_t gi = group_of(i);
              const uint64_t slot = slot_base + gi * GP + PPW * warp + 32 * t + lane;
              c_dst[t] = staging + so + ((slot & ((1u << ppc_shift) - 1)) << 12);
            }
          }
        }
        c_full = full_bits[i & 1] == (1u << TPW) - 1;
#pragma unroll
        for (int q = 0; q < PAIRS; ++q) L[q] = 0x00250025u;  // l_0 = 0x25 in both lanes
      }
      mbar_wait(fbar + 8 * st, ph_full);
      if (st == ST - 1) ph_full ^= 1u;
      // per page: row address with its swizzle bits (unit x at addr ^ (x << 4),
      // next box + SUB); pages without bytes in this stage read the zero slab
      // (their chain continues over zeros, which adds nothing to the sum)
      const uint32_t sbase = ring + st * C::WSTAGE + lane * BOXW;
      uint32_t pa[TPW], pb[TPW];
      if (c_full) {
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          pa[t] = (sbase + t * C::TASKB) | swz;
          pb[t] = C::SUB;
        }
      } else {
        const uint32_t rb = reg_bits[i & 1];
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          const bool v = s * SLAB < c_len[t];
          pa[t] = v ? (sbase + t * C::TASKB) | ((rb >> t) & 1 ? swz : 0u) : zbase;
          pb[t] = v ? C::SUB : 0u;
        }
      }
#pragma unroll
      for (int h = 0; h < C::BPS; ++h) {
        const uint32_t gb = C::BPS * p + h;
        const uint32_t ab = gb % NA;
        if (gb >= NA) mbar_wait(bar_afree + 8 * ab, (gb / NA - 1) & 1);
        tc_fence_after();
        const uint32_t acol = trow + ab * C::ABUF;
#pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
          const uint32_t unit = 2 * h + uu;
          const uint32_t ux = (unit % C::UPB) << 4, uo = unit / C::UPB;
          // all loads, then the chains (independent: the compiler interleaves
          // them), then the TMEM stores (volatile asm: nothing moves across)
          uint4 v[TPW];
#pragma unroll
          for (int t = 0; t < TPW; ++t) v[t] = ld_shared16((pa[t] ^ ux) + uo * pb[t]);
          uint32_t upk[PAIRS][8], lpk[PAIRS][8];
#pragma unroll
          for (int q = 0; q < PAIRS; ++q) {
            if (dbg & 1) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                upk[q][j] = v[2 * q].x + j;
                lpk[q][j] = v[2 * q + 1].y + j;
              }
            } else {
              chain16(L[q], v[2 * q], v[2 * q + 1], upk[q], lpk[q]);
            }
          }
#pragma unroll
          for (int q = 0; q < PAIRS; ++q) {
            tc_st8(acol + q * C::ASET + 8 * uu, upk[q]);
            tc_st8(acol + q * C::ASET + 16 + 8 * uu, lpk[q]);
          }
        }
        tc_wait_st();
        tc_fence_before();
        mbar_arrive(bar_afull + 8 * ab);
      }
      if constexpr (C::FUSED) {
        // speculative compaction: every page of a predicted-staged chunk writes
        // this stage's slab to staging, UNITS lanes per page (coalesced
        // SLAB-byte segments), read back from the shared-memory stage before
        // the slot is refilled
        constexpr int PPI = 32 / C::UNITS;
        const uint32_t x = lane % C::UNITS, jj = lane / C::UNITS;
        const uint32_t rb = reg_bits[i & 1];
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          const uint32_t vm = __ballot_sync(kFull, c_dst[t] != nullptr && s * SLAB < c_len[t]);
          if (vm == 0) continue;
          const uint32_t tb = ring + st * C::WSTAGE + t * C::TASKB;
#pragma unroll
          for (int k = 0; k < 32 / PPI; ++k) {
            const uint32_t j = k * PPI + jj;
            uint8_t* d = reinterpret_cast<uint8_t*>(
                __shfl_sync(kFull, reinterpret_cast<uint64_t>(c_dst[t]), j));
            if ((vm >> j) & 1) {
              const uint32_t sw = (rb >> t) & 1 ? ((j >> 1) & 3) : 0u;  // SWIZZLE_64B row j
              st_stream16(d + s * SLAB + x * 16, ld_shared16(tb + j * BOXW + ((x ^ sw) << 4)));
            }
          }
        }
      }
      __syncwarp();  // the stage slot is refilled by this warp's next issue
      if (s == C::STAGES - 1) {
        // ---- epilogue of group i: accumulators -> page digests -> chunk digests
        const uint32_t db = i % NDB;
        mbar_wait(bar_dfull + 8 * db, (i / NDB) & 1);
        tc_fence_after();
        // d[16 q + 8 pg + j] = limb j of page (pair q, lane pg)
        uint32_t d[16 * PAIRS];
        if constexpr (PAIRS == 2) {
          uint32_t (&dd)[32] = reinterpret_cast<uint32_t (&)[32]>(d);
          tc_ld32(drow + db * C::DBUF, dd);
        } else {
          uint32_t (&dd)[16] = reinterpret_cast<uint32_t (&)[16]>(d);
          tc_ld16(drow + db * C::DBUF, dd);
        }
        tc_fence_before();
        mbar_arrive(bar_dfree + 8 * db);
        const uint64_t k0 = __ldg(htab + 34);
        uint32_t vm[TPW];
#pragma unroll
        for (int t = 0; t < TPW; ++t) {
          const int q = t >> 1, pg = t & 1;
          uint64_t S = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) S += static_cast<uint64_t>(d[16 * q + 8 * pg + j]) << (8 * j);
          const uint64_t ln = (L[q] >> (16 * pg)) & 0xffu;
          const uint32_t n = c_len[t];
          uint64_t hv = 0;
          if (n > 0) {
            const uint32_t m = n >> 8;
            hv = __ldg(htab + m) + __ldg(htab + 17 + m) * (S + ln - k0);
          }
          dsm[warp * PPW + 32 * t + lane] = hv;
          vm[t] = __ballot_sync(kFull, n > 0);
        }
        __syncwarp();
        const uint64_t gi = group_of(i);
        const uint64_t slot0 = slot_base + gi * GP + PPW * warp;
        const uint32_t ppc = 1u << ppc_shift;
        for (uint32_t c = lane; c < (uint32_t(PPW) >> ppc_shift); c += 32) {
          const uint32_t p0 = c << ppc_shift;
          const uint32_t t0 = p0 >> 5;
          uint32_t vq = vm[0];
#pragma unroll
          for (int t = 1; t < TPW; ++t)
            if (t0 == uint32_t(t)) vq = vm[t];
          if (!((vq >> (p0 & 31)) & 1)) continue;
          uint64_t hv;
          if (ppc_shift == 0) {
            hv = dsm[warp * PPW + p0];
          } else {
            // a chunk's pages lie in one task (ppc <= 32): valid pages are a prefix
            hv = kFnvOffset;
            for (uint32_t j = 0; j < ppc; ++j) {
              if (!((vq >> ((p0 + j) & 31)) & 1)) break;
              hv = fnv_u64(hv, dsm[warp * PPW + p0 + j]);
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
  if (warp == CW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::TCOLS)
                 : "memory");
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
  static std::mutex m;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(m);
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

// Chain warps per SM of the hash-only kernel. The 8-bit chains are issue-latency
// bound (ncu: tensor pipe 8 % active, 2.25 warps per scheduler with 8 warps x 2 chain
// pairs), so more warps with fewer pairs each win: 16 x 1 pair (same 1024-page groups,
// 94 registers) on the same box: C3 switch 0.877 -> 0.813 ms, 1 GiB 4.72 -> 5.02 TB/s,
// 4 GiB 5.59 -> 6.00 TB/s; 12 x 2 pairs (1536-page groups, 2 stages) ties at 4 GiB but
// loses below ~3.5 GiB to wave quantization. SNAP_MMA_CW=8|12|16 forces one (A/B).
// Grids of at most one 512-page group per SM (<= ~296 MiB) run 8 chain warps x 1
// pair (81): twice the groups of the 1024-page geometries, so every SM gets work
// (hash-only, same box: 16 MiB 190 -> 221 GB/s, 64 MiB 755 -> 878, 256 MiB 2850 ->
// 3312 vs the TMA FNV kernel; from 384 MiB on 16 x 1 wins: 3684 vs 2603).
uint32_t mma_cw_for(uint64_t slots, int sms) {
  static const int force = getenv("SNAP_MMA_CW") ? atoi(getenv("SNAP_MMA_CW")) : 0;
  if (force == 8 || force == 12 || force == 16 || force == 81) return uint32_t(force);
  return slots <= uint64_t(sms > 0 ? sms : 148) * uint64_t(MmaHash8x1::GP) ? 81u : 16u;
}

uint32_t mma_schedule(const uint64_t* addr, const uint64_t* bytes, uint32_t n,
                      uint32_t page_shift, uint32_t chunk_shift, int sms,
                      std::vector<uint32_t>& out, uint32_t cw) {
  out.clear();
  if (page_shift != 12 || chunk_shift < 12 || chunk_shift > 17 || n == 0 || sms <= 0) return 0;
  static_assert(MmaHash::GP == MmaFusedLight::GP, "one schedule for both 8-warp variants");
  const uint64_t GP = cw == 12 ? uint64_t(MmaHash12::GP)
                    : cw == 16 ? uint64_t(MmaHash16::GP)
                    : cw == 81 ? uint64_t(MmaHash8x1::GP) : uint64_t(MmaHash::GP);
  const uint64_t cb = 1ull << chunk_shift;
  std::vector<uint64_t> caddr;  // chunk address, ~0 for a partial chunk
  for (uint32_t b = 0; b < n; ++b)
    for (uint64_t o = 0; o < bytes[b]; o += cb) caddr.push_back(o + cb <= bytes[b] ? addr[b] + o : ~0ull);
  const uint64_t nch = caddr.size();
  const uint32_t ppc_shift = chunk_shift - 12;
  const uint64_t nslots = nch << ppc_shift;
  const uint64_t ngroups = (nslots + GP - 1) / GP;
  if (ngroups == 0 || ngroups >= (1ull << 32)) return 0;
  const uint32_t bins = uint32_t(ngroups < uint64_t(sms) ? ngroups : uint64_t(sms));
  // a task (32 page slots) is regular iff its chunks are full and contiguous
  const uint64_t cpt = 32 >> ppc_shift;  // chunks per task
  std::vector<uint8_t> heavy(ngroups, 0);
  for (uint64_t gi = 0; gi < ngroups; ++gi)
    for (uint64_t t = 0; t < GP / 32 && !heavy[gi]; ++t) {
      const uint64_t c0 = ((gi * GP) >> ppc_shift) + t * cpt;
      bool reg = c0 + cpt <= nch;
      for (uint64_t k = 0; reg && k < cpt; ++k)
        reg = caddr[c0 + k] != ~0ull && caddr[c0 + k] == caddr[c0] + k * cb;
      heavy[gi] = !reg;
    }
  // longest processing time first: heavy groups (cost 150), then regular (100),
  // each to the least-loaded CTA (SNAP_MMA_HEAVY overrides the heavy cost)
  static const uint64_t heavy_cost = getenv("SNAP_MMA_HEAVY") ? strtoull(getenv("SNAP_MMA_HEAVY"), nullptr, 10) : 150;
  std::vector<std::vector<uint32_t>> per(bins);
  std::vector<uint64_t> load(bins, 0);
  auto cmp = [&](uint32_t a, uint32_t b2) { return load[a] != load[b2] ? load[a] > load[b2] : a > b2; };
  std::vector<uint32_t> h(bins);
  for (uint32_t b = 0; b < bins; ++b) h[b] = b;
  std::make_heap(h.begin(), h.end(), cmp);
  for (int pass = 0; pass < 2; ++pass)
    for (uint64_t gi = 0; gi < ngroups; ++gi) {
      if (heavy[gi] != (pass == 0)) continue;
      std::pop_heap(h.begin(), h.end(), cmp);
      const uint32_t b = h.back();
      per[b].push_back(uint32_t(gi));
      load[b] += pass == 0 ? heavy_cost : 100;
      std::push_heap(h.begin(), h.end(), cmp);
    }
  out.resize(bins + 1 + ngroups);
  out[0] = 0;
  uint64_t k = bins + 1;
  for (uint32_t b = 0; b < bins; ++b) {
    std::sort(per[b].begin(), per[b].end());
    out[b + 1] = out[b] + uint32_t(per[b].size());
    for (uint32_t x : per[b]) out[k++] = x;
  }
  return bins;
}

bool hash_mma_ok(const GridDev& g) {
  return g.tmaps64 != nullptr && g.page_shift == 12 && g.chunk_shift >= 12 &&
         g.chunk_shift <= 17;
}

namespace {
template <class C>
int launch_mma(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig,
               const uint64_t* spec_off, uint8_t* staging, cudaStream_t s) {
  static uint64_t attr = 0;
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_hash_mma<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
  });
  const uint64_t c_end = g.c_end ? g.c_end : g.nchunks;
  if (c_end <= g.c_begin) return 0;
  const uint8_t* bt = device_btab();
  if (!bt) return -1;
  const uint64_t ngroups = (((c_end - g.c_begin) << (g.chunk_shift - 12)) + C::GP - 1) / C::GP;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t blocks = ngroups < uint64_t(sms) ? ngroups : uint64_t(sms);
#ifdef SNAP_MMA_DEBUG_MODES
  // timing-only modes (1: no chain, 2: no MMA; digests are wrong), build with
  // make EXTRA=-DSNAP_MMA_DEBUG_MODES and set SNAP_MMA_DEBUG
  static const int dbg = getenv("SNAP_MMA_DEBUG") ? atoi(getenv("SNAP_MMA_DEBUG")) : 0;
#else
  const int dbg = 0;
#endif
  // the balanced schedule covers the whole grid on exactly `blocks` CTAs
  // (SNAP_MMA_SCHED=0: round robin, for A/B measurements)
  static const bool sched_on = !(getenv("SNAP_MMA_SCHED") && getenv("SNAP_MMA_SCHED")[0] == '0');
  GridDev gg = g;
  if (C::FUSED || !sched_on || !(g.c_begin == 0 && c_end == g.nchunks && g.gs_bins == blocks)) gg.gsched = nullptr;
  k_hash_mma<C><<<unsigned(blocks), C::THREADS, C::SMEM, s>>>(arena, gg, chunk_dig, bt, spec_off,
                                                               staging, dbg);
  return 1;
}
}  // namespace

int launch_hash_mma(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig, cudaStream_t s) {
  if (g.mma_cw == 12) return launch_mma<MmaHash12>(arena, g, chunk_dig, nullptr, nullptr, s);
  if (g.mma_cw == 16) return launch_mma<MmaHash16>(arena, g, chunk_dig, nullptr, nullptr, s);
  if (g.mma_cw == 81) return launch_mma<MmaHash8x1>(arena, g, chunk_dig, nullptr, nullptr, s);
  return launch_mma<MmaHash>(arena, g, chunk_dig, nullptr, nullptr, s);
}

int launch_hash_mma_fused(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig,
                          const uint64_t* spec_off, uint8_t* staging, cudaStream_t s) {
  // fused: 16 chain warps x 1 pair, 3 stages (same-box A/B: full C2 on one GPU 4.28 ->
  // 4.10 ms; rank 0's layout at N = 2 / 4 / 8: K1 0.871 / 0.777 / 0.750 -> 0.858 /
  // 0.741 / 0.703 ms; a 12 x 2 geometry with 2 stages was slower, 4.59 ms).
  // SNAP_MMA_FUSED_CW=8 forces the round-1 geometry.
  static const int fcw = getenv("SNAP_MMA_FUSED_CW") ? atoi(getenv("SNAP_MMA_FUSED_CW")) : 16;
  if (fcw == 8) return launch_mma<MmaFusedLight>(arena, g, chunk_dig, spec_off, staging, s);
  if (fcw == 81) return launch_mma<MmaFused8x1>(arena, g, chunk_dig, spec_off, staging, s);
  return launch_mma<MmaFused16>(arena, g, chunk_dig, spec_off, staging, s);
}

}  // namespace snap
