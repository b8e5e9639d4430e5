// snap_internal.h — shared declarations of the sm_100a kernels and the ctx.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <mutex>
#include <utility>
#include <string>
#include <vector>

#include "snap.h"

namespace snap {

// Programmatic dependent launch: the kernel may be scheduled while the previous
// kernel of the stream drains; it must call griddep_wait() before touching
// anything that kernel wrote (K2 / K3 follow K1 and each other on one stream).
template <class... P, class... A>
inline cudaError_t launch_pdl(void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

// Per-(kernel, device) one-time setup, e.g. cudaFuncSetAttribute (which only
// applies to the current device): runs f() the first time this device is seen
// for `done`. Thread-safe; a process may drive several GPUs (one ctx each).
template <class F>
void once_per_device(uint64_t& done, F&& f) {
  static std::mutex m;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> lock(m);
  if (done & bit) return;
  f();
  done |= bit;
}

constexpr uint64_t kFnvOffset = 14695981039346656037ull;  // sim.hpp:57
constexpr uint32_t kFnvPrimeLo = 0x1b3u;                   // prime = 2^40 + 0x1b3 (sim.hpp:58)

// Device-resident buffer table for one installed grid.
struct TableDev {
  unsigned long long* keys = nullptr;  // kEmptyKey = unused
  unsigned long long* vals = nullptr;  // min chunk index
  uint64_t mask = 0;
};
constexpr unsigned long long kEmptyKey = 0xffffffffffffffffull;

struct GridDev {
  const uint64_t* addr = nullptr;    // [nbufs]
  const uint64_t* bytes = nullptr;   // [nbufs]
  const uint64_t* cstart = nullptr;  // [nbufs + 1] chunk prefix
  uint32_t nbufs = 0;
  uint64_t nchunks = 0;
  uint32_t page_shift = 12;
  uint32_t chunk_shift = 16;
  // [nchunks] buffer index of every chunk (built with the grid): one load
  // instead of a binary search over cstart at every task start (~log2(nbufs)
  // dependent L2 round trips); nullptr: the search
  const uint32_t* chunk_buf = nullptr;
  // [nchunks] arena offset and byte length of every chunk (with chunk_buf): a
  // task's page descriptors in one round of independent loads
  const uint64_t* chunk_addr = nullptr;
  const uint32_t* chunk_len = nullptr;
  // K1 hashes chunks [c_begin, c_end) (c_end == 0: all); lets the host-buffer
  // snapshot hash each slab as soon as its H2D copy lands
  uint64_t c_begin = 0;
  uint64_t c_end = 0;
  // per-buffer CUtensorMap array in device memory (4 KiB pages), or nullptr:
  // boxes of 32 pages x 128 B (SWIZZLE_128B, k_hash_tma)
  const void* tmaps = nullptr;
  // arena-wide maps (16 alignment classes, encode_arena_maps) with 64-byte
  // boxes (SWIZZLE_64B) of 32 pages (task loads) and of one chunk (pages per
  // chunk 8..32: tasks spanning buffers or buffer tails), for k_hash_mma
  const void* tmaps64 = nullptr;
  const void* tmaps64c = nullptr;
  // Single-GPU snapshot: the K2 insert pass fused into K1 — the lane that
  // finishes a chunk digest inserts it into `dd` (first occurrence by
  // atomicMin, skipped when `kn` holds it and kn_use) and records the slot in
  // dd_slot[chunk]. dd.keys == nullptr: off.
  TableDev dd{};
  TableDev kn{};
  uint64_t* dd_slot = nullptr;
  int kn_use = 0;
  // Multi-rank digest exchange fused into K1: every finished chunk digest is
  // also stored into each rank's gathered vector over NVLink (xdig[q] = rank
  // q's CUDA-IPC-mapped window, entry xoff + chunk). xdig == nullptr: off.
  uint64_t* const* xdig = nullptr;
  uint32_t xn = 0;
  uint64_t xoff = 0;
  // fused K1: predicted staged bytes of this launch's layout (kernel choice)
  uint64_t spec_bytes = 0;
  // k_hash_mma group schedule of the whole grid (mma_schedule), or nullptr
  // (round robin): gsched[0..gs_bins] = per-CTA start, then the group order
  const uint32_t* gsched = nullptr;
  uint32_t gs_bins = 0;
  // hash-only k_hash_mma geometry chosen at install time: 8 chain warps (1024-page
  // groups) or, for grids of >= 4 groups of 1536 pages per SM, 12 (mma_cw_for)
  uint32_t mma_cw = 8;
  // Fused verify-scatter (K4 + K1 in one pass, k_hash only): reverse != 0
  // reads chunk g from image + src_off[g] (launch_hash's staging / spec_off
  // arguments), writes it to its grid address and hashes the bytes it moved;
  // with expect != nullptr every chunk digest is compared and mismatches are
  // counted in *nbad (BlobStore::get verification, ckpt.cpp:23-29).
  int reverse = 0;
  const uint64_t* expect = nullptr;
  unsigned long long* nbad = nullptr;
  unsigned int* bad_flag = nullptr;  // mapped host word, 1 on any mismatch
};

// Host: balanced k_hash_mma group schedule for a grid of n buffers over `sms`
// CTAs (groups holding a task that is not 32 contiguous full pages run slower;
// longest-processing-time assignment with those weighted 1.5x — C3 A/B over
// weights 1.12 / 1.3 / 1.5 / 2: 1.5 and 2 best, 0.873 -> 0.860 ms per switch;
// 3 over-weights them: C3 -10 %, CTAs with one heavy group get 9 groups). out = [bins + 1] starts, then
// the group indices of CTA 0, CTA 1, ...; returns bins (0: no schedule).
uint32_t mma_schedule(const uint64_t* addr, const uint64_t* bytes, uint32_t n,
                      uint32_t page_shift, uint32_t chunk_shift, int sms,
                      std::vector<uint32_t>& out, uint32_t cw = 8);
// chain warps of the hash-only tensor-core K1 for a grid of `slots` page slots
uint32_t mma_cw_for(uint64_t slots, int sms);

// The decoupled look-back scans (k_select.cu) keep a tile's chunk count in 26
// bits of the status word: a selection / shard scan covers < 2^26 entries.
constexpr uint64_t kMaxScanEntries = 1ull << 26;

// Open-addressing digest table (dedup + known set), power-of-two capacity.

// Launchers (each returns the number of kernels launched).
// K1; with spec_off != nullptr also the fused speculative K3 (TMA bulk stores
// of every chunk whose spec_off[chunk] != ~0 to staging + spec_off[chunk]).
// whether the K1 launch_hash would pick for (g, spec_off) does the K2 insert in its
// epilogue (the FNV-chain k_hash family) rather than in a separate range kernel
bool k1_epilogue_insert(const GridDev& g, const uint64_t* spec_off);
int launch_hash(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig,
                const uint64_t* spec_off, uint8_t* staging, cudaStream_t s);
// K1 hash-only through TMA tensor loads (needs grid tensor maps, 4 KiB pages).
bool hash_tma_ok(const GridDev& g);
bool hash_tma_selected();  // SNAP_HASH_VARIANT=10: tensor maps are built for the grid
int launch_hash_tma(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig, cudaStream_t s);
// fused K1 with TMA tensor loads (CfgE geometry; needs the per-buffer maps)
int launch_hash_tma_fused(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig,
                          const uint64_t* spec_off, uint8_t* staging, cudaStream_t s);
// K1 hash-only on the tensor cores (k_hash_mma.cu: 8-bit FNV chain on the CUDA
// cores + the linear part as a tcgen05 int8 MMA); needs the grid tensor maps.
bool hash_mma_ok(const GridDev& g);
int launch_hash_mma(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig, cudaStream_t s);
// the same with the speculative K3 stores fused (spec_off / staging as launch_hash),
// for grids where few chunks are staged (multi-GPU striping)
int launch_hash_mma_fused(const uint8_t* arena, const GridDev& g, uint64_t* chunk_dig,
                          const uint64_t* spec_off, uint8_t* staging, cudaStream_t s);
// K1 kernel policy override (SNAP_HASH_VARIANT semantics; -1 = default policy)
void set_hash_variant(int v);
// name of the K1 kernel the last launch_hash call chose (process-wide)
const char* last_k1_name();
// host: one 128-byte CUtensorMap per buffer into host_maps (box of 32 pages x
// box_bytes, box_bytes 128 -> SWIZZLE_128B, 64 -> SWIZZLE_64B); 0 on success
// 16 arena-wide maps (one per 256-B alignment class of a page start), see k_hash_tma.cu
int encode_arena_maps(const uint8_t* arena, uint64_t arena_bytes, int box_bytes, int box_rows,
                      void* host_maps);
// box_rows rows per box; arena_bytes != 0: a partial last page counts as a row
// (when it fits the arena), for chunk-sized boxes at buffer tails
int encode_tensor_maps(const uint8_t* arena, const uint64_t* addr, const uint64_t* bytes,
                       uint32_t nbufs, void* host_maps, int box_bytes = 128, int box_rows = 32,
                       uint64_t arena_bytes = 0);
// Cross-GPU barrier after a fused-exchange K1: signal every peer (flag slot
// `rank` of its window := epoch, release.sys) and wait for every peer's
// signal in this rank's window (acquire.sys); traps after ~30 s.
int launch_peer_barrier(uint64_t* const* xflag, const uint64_t* myflag, uint32_t rank, uint32_t n,
                        uint64_t epoch, cudaStream_t s);
// The reference's whole-buffer digest, value-equal (k_whole.cu): per-segment
// state tables (64 KiB segments x 256 entry low bytes) then one serial combine
// per buffer. seg_start[b] = first segment of buffer b (nb + 1 entries), F =
// nseg * 256 u64 scratch, out[b] = digest_of_words(buffer b).
uint64_t whole_segments(uint64_t bytes);
int launch_whole_digest(const uint8_t* arena, const uint64_t* addr, const uint64_t* bytes,
                        const uint64_t* seg_start, uint32_t nb, uint64_t nseg, uint64_t* F,
                        uint64_t* out, cudaStream_t s);
int launch_buf_fold(const GridDev& g, const uint64_t* chunk_dig, uint64_t* buf_dig, cudaStream_t s);
int launch_fill_mix64(uint64_t* dst, uint64_t nwords, uint64_t seed, uint64_t base, cudaStream_t s);
int launch_xor_words(uint8_t* arena, const uint64_t* addrs, uint64_t n, uint64_t value,
                     cudaStream_t s);

int launch_table_clear(TableDev t, cudaStream_t s);
int launch_table_insert_min(TableDev t, const uint64_t* keys, uint64_t n, uint64_t index_base,
                            cudaStream_t s);
// K2: insert (slot + known flag per chunk), then the selection scan:
// sel/owner/offsets + compact index list; `scan_state` sized by scan_state_words(n).
uint64_t scan_state_words(uint64_t n);
int launch_dedup_insert(TableDev dedup, TableDev known, bool use_known, const uint64_t* dig,
                        const uint32_t* lens, uint64_t n, uint64_t* slot, cudaStream_t s);
// scan_state must be zero on entry (left zero by launch_resolve_dups' clean-up);
// spec_next (nullable) receives the staging layout (offset of selected chunks,
// ~0 otherwise) — the next speculative layout of the fused K1.
// spec_cur (nullable): the fused K1's speculative layout — the scan also does
// the K3 fix-up (copies selected chunks whose offset differs from arena to staging).
int launch_select(TableDev dedup, const uint64_t* slot, const uint32_t* lens, uint64_t n,
                  uint64_t* scan_state, uint8_t* sel, uint64_t* owner, uint64_t* offsets,
                  uint32_t* sel_list, uint64_t* totals, uint64_t* spec_next, cudaStream_t s,
                  const uint64_t* spec_cur = nullptr, const uint8_t* arena = nullptr,
                  const GridDev* grid = nullptr, uint8_t* staging = nullptr);
// The same selection for n <= 8192 chunks in one launch of <= 8 CTAs (insert +
// scan + fix-up + duplicate resolution + table clean-up, software grid
// barriers), identical outputs; the dedup table must be empty on entry and is
// left empty; `scratch` = >= 9 words of (zero) scan state, left zero.
bool select_small_ok(uint64_t n);
// n <= 4096: the whole selection in one 8-CTA cluster (DSMEM first-occurrence table)
bool select_cluster_ok(uint64_t n);
int launch_select_cluster(TableDev known, bool use_known, const uint64_t* dig,
                          const uint32_t* lens, uint64_t n, uint8_t* sel, uint64_t* owner,
                          uint64_t* offsets, uint32_t* sel_list, uint64_t* totals,
                          uint64_t* spec_next, cudaStream_t s, const uint64_t* spec_cur,
                          const uint8_t* arena, const GridDev* grid, uint8_t* staging);
int launch_select_small(TableDev dedup, TableDev known, bool use_known, const uint64_t* dig,
                        const uint32_t* lens, uint64_t n, uint8_t* sel, uint64_t* owner,
                        uint64_t* offsets, uint32_t* sel_list, uint64_t* totals,
                        uint64_t* spec_next, cudaStream_t s, uint64_t* scratch,
                        const uint64_t* spec_cur = nullptr, const uint8_t* arena = nullptr,
                        const GridDev* grid = nullptr, uint8_t* staging = nullptr);
// Shard scan of writer q over the global writer vector (write_list for q ==
// this rank: local chunk list + offsets).
int launch_shard_scan(const int32_t* writer, const uint32_t* glens, uint32_t nranks, uint64_t maxn,
                      int32_t q, bool write_list, uint64_t* scan_state, uint64_t* shard_off,
                      uint32_t* my_list, uint64_t* my_off, uint64_t* totals, cudaStream_t s);
// K3 fix-up fused into the multi-rank selection (staging == nullptr: off):
// spec_next[0..nlocal) reset by k_select_stripe, then written and the
// mismatched chunks copied by this rank's shard scan.
struct FixUp {
  const uint64_t* spec_cur = nullptr;
  uint64_t* spec_next = nullptr;
  uint64_t nlocal = 0;
  const uint8_t* arena = nullptr;
  GridDev grid{};
  uint8_t* staging = nullptr;
};
// Multi-rank step: owner / sel / writer per global chunk from the filled dedup
// table (k_select_stripe), then rank `me`'s shard scan, which also empties the
// table; the global staging offsets are left to launch_select (on demand).
int launch_select_stripe(TableDev dedup, const uint64_t* slot, const uint64_t* gdig,
                         const uint32_t* glens, uint32_t nranks, uint64_t maxn, int32_t me,
                         uint8_t* sel, uint64_t* owner, int32_t* writer, uint64_t* scan_state,
                         uint64_t* shard_off, uint32_t* my_list, uint64_t* my_off,
                         uint64_t* totals, cudaStream_t s, const FixUp& fix = FixUp{});
// host pages: first-occurrence / known-set / previous-page-set classification
// (flags bit 1 fresh, bit 2 inc; counts[0..1] += fresh, inc; counts zeroed by the caller)
int launch_page_classify(TableDev pages, TableDev known, bool use_known, TableDev prev,
                         bool use_prev, const uint64_t* dig, uint64_t n, uint64_t* slot,
                         uint8_t* flags, unsigned long long* counts, cudaStream_t s);
// Also resets `clear` (the dedup table just consumed) and clear_words of
// scan state to their empty values for the next selection (nullable).
int launch_resolve_dups(const uint8_t* sel, const uint64_t* owner, uint64_t* offsets, uint64_t n,
                        TableDev clear, uint64_t* scan_state, uint64_t clear_words,
                        cudaStream_t s);

// K3 / K4 chunk copies.
// offsets_by_list: dst offset of list entry k is offsets[k] (shard lists) instead
// of offsets[sel_list[k]] (single-GPU image). spec_cur (nullable): chunks the
// fused hash pass already wrote at the right offset are skipped; spec_next
// (nullable) receives the actual layout (next prediction). moved (nullable)
// receives the list index of every chunk actually copied (count in *nmoved,
// zeroed by the caller).
int launch_gather(const uint8_t* arena, const GridDev& g, const uint32_t* lens,
                  const uint32_t* sel_list, const uint64_t* totals, const uint64_t* offsets,
                  bool offsets_by_list, const uint64_t* spec_cur, uint64_t* spec_next,
                  uint8_t* staging, uint64_t max_sel, cudaStream_t s, uint32_t* moved = nullptr,
                  unsigned int* nmoved = nullptr);
int launch_scatter(uint8_t* arena, const GridDev& g, const uint32_t* lens, const uint8_t* image,
                   const uint64_t* src_off, cudaStream_t s);
// K4 from striped shards (peer staging pointers): chunk g of global row `row`.
int launch_scatter_shards(uint8_t* arena, const GridDev& g, const uint32_t* lens, uint64_t row,
                          const uint64_t* owner, const int32_t* writer, const uint64_t* shard_off,
                          const uint8_t* const* shards, unsigned long long* missing,
                          cudaStream_t s);
int launch_compare(const uint64_t* a, const uint64_t* b, uint64_t n, unsigned long long* nbad,
                   cudaStream_t s);

// K3 with an image source: chunk sel_list[k] from image + src_off[chunk] to
// dst + offsets[chunk] (offsets[k] when offsets_by_list).
int launch_gather_from(const uint8_t* image, const uint64_t* src_off, const uint32_t* lens,
                       const uint32_t* sel_list, const uint64_t* totals, const uint64_t* offsets,
                       uint8_t* dst, uint64_t max_sel, cudaStream_t s, bool offsets_by_list = false);
// Splice chunk cache (fixed HBM slot array + digest -> slot index): slot
// assignment of the selected chunks from the free stack (+ index insert), the
// reclamation pass, and the swap-in pass (cache.vals = slot index).
int launch_cache_assign(TableDev cache, const uint64_t* dig, const uint32_t* sel_list,
                        const uint64_t* totals, const uint32_t* lens, const uint32_t* free_stack,
                        uint64_t free_n, uint32_t slot_shift, uint64_t* list_off,
                        uint32_t* slot_len, uint64_t max_n, cudaStream_t s);
int launch_cache_gc(TableDev old, TableDev live, TableDev fresh, uint32_t* free_stack,
                    uint64_t free_n, const uint32_t* slot_len, unsigned long long* cnt,
                    cudaStream_t s);
// copies counters[0..2] (re-arming them to zero) and totals[0..1] (or zeros) to
// the mapped host words host[0..4]
int launch_splice_report(unsigned long long* counters, const uint64_t* totals,
                         unsigned long long* host, cudaStream_t s);
int launch_splice_in(uint8_t* arena, const GridDev& to, const uint32_t* lens, const uint64_t* want,
                     const int64_t* match, const uint64_t* dig_from, TableDev cache,
                     const uint8_t* cache_base, uint32_t slot_shift, unsigned long long* counters,
                     cudaStream_t s);
// dst[r] <- src[r], bytes[r] (multiple of 16) for r < nr; device pointer arrays.
int launch_copy_ranges(uint8_t* const* dst, const uint8_t* const* src, const uint64_t* bytes,
                       uint32_t nr, uint64_t max_bytes, cudaStream_t s);

// Fixed-order allreduce over peer memory (k_allreduce.cu): GPU `me` sums its
// slice of every source in list order and stores it into every dst; with
// use_flags, device flag barriers (system-scope release/acquire on the peers'
// flag lines) before the reads and after the stores.
struct ArArgs {
  const uint8_t* const* src = nullptr;  // [R] peer-mapped sources, sum order
  uint8_t* const* dst = nullptr;        // [N] every GPU's destination
  uint64_t* const* flags = nullptr;     // [N] every GPU's flag lines
  uint64_t* myflag = nullptr;
  uint32_t R = 0, N = 1, me = 0;
  int dtype = 0;
  uint64_t elems = 0;
  uint64_t epoch = 0;
  int use_flags = 0;
  unsigned int* cta_count = nullptr;    // zero; the last CTA resets it
};
int launch_ordered_allreduce(const ArArgs& a, cudaStream_t s);

// K5.
int launch_grad_sum(int dtype, uint8_t* arena, const uint64_t* src_addrs_dev, uint32_t nsrc,
                    uint64_t dst_addr, uint64_t elems, int accumulate, cudaStream_t s);

}  // namespace snap
