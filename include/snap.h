/*
 * snap.h — C ABI of the B200-native snapshot / dedup / restore / splice hot
 * path (arXiv 2202.07848 "Singularity", reference = fleetsim C++ simulator).
 *
 * The reference has no FFI: its hot path is in-process C++ (SURVEY.md §8b).
 * Each entry point below names the reference interface it replaces
 * (path:line relative to the reference's proj/). A maintainer swaps the
 * reference's std::vector "device" for this library by binding these symbols
 * (INTEGRATION.md shows the adapter). Plain pointers and sizes only.
 *
 * Conventions
 *  - One snap_ctx per (job, GPU), the analogue of proxy::ProxyServer
 *    (proxy.hpp:32-122): it owns the device arena (one cudaMalloc reservation,
 *    SPEC.md:232), the chunk grid, digest vectors, the dedup table, the staging
 *    image and (optionally) an NCCL communicator.
 *  - All device work is issued on the ctx's own CUDA stream, in call order.
 *    Calls that return host data synchronise that stream once per call.
 *  - A ctx is used by one host thread at a time (the reference's proxy
 *    serializes all device access); different ctxs are independent.
 *    With a communicator attached, snap_snapshot / snap_select /
 *    snap_snapshot_host / snap_known_commit AND every call that installs a grid
 *    (snap_set_buffers, snap_load) are collective: every rank makes the same
 *    sequence of them (the grid's chunk counts and lengths are exchanged when
 *    it is installed, so a snapshot always issues the same NCCL sequence).
 *    snap_comm_init / snap_comm_destroy are collective over the new / current
 *    communicator.
 *  - Return codes (common.hpp:31-49 error conventions):
 *      SNAP_OK        success
 *      SNAP_EINVAL    bad argument / geometry          (ConfigError)
 *      SNAP_ENOMEM    out of device/host memory         (alloc -> nullopt)
 *      SNAP_EFAULT    modeled fault, e.g. digest verification failed,
 *                     missing content                   (SimFault)
 *      SNAP_ECUDA     CUDA / NCCL runtime error
 *      SNAP_EINTERNAL invariant broken                  (InternalError)
 *    snap_last_error(ctx) returns the message of the last failure.
 *  - Addresses are byte offsets inside the ctx arena (vdev::MemRange::addr,
 *    vdev.hpp:49-53). Buffers are 256-byte aligned and sized
 *    (BidiAllocator::kAlign, alloc.hpp:28; alloc.cpp:64).
 *  - There is NO CPU fallback: every compute entry point runs sm_100a kernels
 *    and fails with SNAP_ECUDA when no B200 is present.
 */
#ifndef SNAP_H
#define SNAP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNAP_OK 0
#define SNAP_EINVAL (-1)
#define SNAP_ENOMEM (-2)
#define SNAP_EFAULT (-3)
#define SNAP_ECUDA (-4)
#define SNAP_EINTERNAL (-5)

typedef struct snap_ctx snap_ctx;

/* A tracked allocation: splice::RankBuf (splice.hpp:26-34) and
 * ckpt::WorkerSnapshot::DevRec (ckpt.hpp:64-71). Canonical order of a buffer
 * list is the order build_manifest walks it: rank ascending, slot ascending
 * (ckpt.cpp:104,147). */
typedef struct {
  uint32_t rank;
  int32_t slot;
  uint64_t addr;
  uint64_t bytes;
  int32_t cat; /* vdev::BufCat (vdev.hpp:17): 0 Param 1 OptState 2 Grad 3 Activation 4 Scratch */
  uint32_t flags; /* SNAP_BUF_* layout hints (never affect results, only speed) */
} snap_buf;

/* Hint: the buffer holds identical bytes at the same address on every DP
 * rank (default for cat Param/OptState, test_workload.cpp:210-218). Only used
 * to predict the staging layout of the fused hash+compaction pass. */
#define SNAP_BUF_REPLICATED 1u
#define SNAP_BUF_PRIVATE 2u
/* RankBuf::pending_result (splice.hpp:33): a gradient whose collective result
 * is pending; skipped by splice switches (consumed by K5 accumulation). */
#define SNAP_BUF_PENDING 4u

/* Chunk grid: page digest = digest_of_words(page) (sim.hpp:67-70 on the
 * reference's 4 KiB page unit, ckpt.hpp:15); chunk digest = digest_of_words
 * over its page digests, or the direct FNV-1a of the chunk when
 * page_bytes == chunk_bytes; buffer digest = digest_of_words over its chunk
 * digests (the ledger key that replaces Gpu::digest, vdev.cpp:118). */
typedef struct {
  uint32_t page_bytes;  /* power of two, >= 256; default 4096 */
  uint32_t chunk_bytes; /* power of two, multiple of page_bytes, <= 32 pages */
} snap_geom;

/* ---------------------------------------------------------------- context */

/* ProxyServer ctor (proxy.cpp:7-14) + Gpu(id, mem_bytes) (vdev.cpp:67-70):
 * reserves `arena_bytes` of HBM on `device` (zero-filled). */
int snap_open(int device, uint64_t arena_bytes, snap_ctx** out);
int snap_close(snap_ctx* ctx);
const char* snap_last_error(const snap_ctx* ctx);
const char* snap_strerror(int code);
int snap_arena(snap_ctx* ctx, void** dev_base, uint64_t* bytes);
/* Number of kernels this ctx has launched so far (evidence counter). */
uint64_t snap_launch_count(const snap_ctx* ctx);
int snap_sync(snap_ctx* ctx);

/* splice::DeviceLayout::carve (splice.cpp:7-19): host arithmetic only.
 * out = {rank_region_end, scratch_base, scratch_bytes}. */
int snap_layout_carve(uint64_t mem_bytes, uint64_t max_buffer_bytes, double slack_fraction,
                      uint64_t out[3]);

/* ------------------------------------------- device-proxy memory tracker */

/* mem::BidiAllocator (alloc.hpp:17-62, alloc.cpp:62-155): stable requests
 * top-down, transient bottom-up over [low, high), 256-byte rounding, free
 * lists with coalescing. Host metadata only; one tracker per rank over the
 * ctx rank region (proxy.cpp:100-108).
 * snap_alloc_alloc: SNAP_OK, SNAP_ENOMEM (cursors would cross = nullopt),
 * SNAP_EFAULT (zero size). snap_alloc_free: SNAP_EFAULT for an unknown
 * address (SimFault, alloc.cpp:88). Snapshot = u64 words, exact state
 * (BidiAllocator::snapshot/restore, alloc.cpp:116-140). */
int snap_alloc_create(uint64_t low, uint64_t high, void** out);
int snap_alloc_destroy(void* a);
int snap_alloc_alloc(void* a, uint64_t bytes, int stable, uint64_t* addr);
int snap_alloc_free(void* a, uint64_t addr);
uint64_t snap_alloc_stable_digest(void* a);
int snap_alloc_cursors(void* a, uint64_t* transient_cursor, uint64_t* stable_cursor,
                       uint64_t* live_bytes);
int snap_alloc_snapshot(void* a, uint64_t* words, uint64_t cap, uint64_t* n);
int snap_alloc_restore(void* a, const uint64_t* words, uint64_t n);

/* Pinned host memory for staging images / host-side inputs (page-locked so
 * H2D/D2H run at PCIe DMA speed). */
int snap_host_alloc(uint64_t bytes, void** out);
int snap_host_free(void* p);

/* Gpu::write_words / Gpu::words (vdev.cpp:106-124): host <-> arena copies. */
int snap_write(snap_ctx* ctx, uint64_t addr, const void* src, uint64_t bytes);
int snap_read(snap_ctx* ctx, uint64_t addr, void* dst, uint64_t bytes);
/* Device-side synthetic content: words[i] = mix64(seed ^ (base + i))
 * (sim.hpp:37-41), i counted in u64 words from `addr`. */
int snap_fill_mix64(snap_ctx* ctx, uint64_t addr, uint64_t bytes, uint64_t seed, uint64_t base);
/* XOR `value` into the u64 word at each addrs[i] (dirty-chunk mutation). */
int snap_xor_words(snap_ctx* ctx, const uint64_t* addrs, uint64_t n, uint64_t value);

/* ------------------------------------------------------- K1: hash (digest) */

/* Installs the buffer list (a consistent cut of the ledger, ckpt.cpp:147) and
 * its chunk grid; returns the number of chunks. */
int snap_set_buffers(snap_ctx* ctx, const snap_buf* bufs, uint64_t n, const snap_geom* geom,
                     uint64_t* n_chunks);
/* K1: digests every chunk of every installed buffer (replaces
 * GpuLedger::refresh_digests, splice.cpp:150-159, and the hashing inside
 * BlobStore::put, ckpt.cpp:17). Async on the ctx stream. */
int snap_hash(snap_ctx* ctx);
/* Copies digest vectors to the host (any pointer may be NULL).
 * buf_digests triggers the per-buffer fold kernel. */
int snap_get_digests(snap_ctx* ctx, uint64_t* chunk_digests, uint32_t* chunk_lens,
                     uint64_t* buf_digests);
/* Gpu::digest over a list of ranges (vdev.cpp:118), hierarchical digest per
 * range; synchronous convenience used by the ledger adapters. */
int snap_digest_ranges(snap_ctx* ctx, const snap_buf* bufs, uint64_t n, const snap_geom* geom,
                       uint64_t* out_buf_digests);

/* Gpu::digest (vdev.cpp:118) VALUE-EQUAL to the reference: digest_of_words
 * over every byte of each range (one 64-bit FNV-1a chain per range), the
 * opt-in compatibility path of SURVEY §8(c) — the ledger and snapshot keys use
 * the parallel chunk-Merkle digest above. The serial chain is split by the
 * chain's affinity in the state above its low byte: per 64 KiB segment, 256
 * chains (one per entry low byte) run in parallel, then one table lookup per
 * segment combines them. Synchronous. */
int snap_digest_whole(snap_ctx* ctx, const snap_buf* bufs, uint64_t n, uint64_t* out);

/* ----------------------------------------- K2: dedup + dirty (selection) */

/* Known-digest set = the BlobStore's key set (ckpt.hpp:39): chunks whose
 * digest is known are not staged again (BlobStore::put fresh test,
 * ckpt.cpp:18-20). */
int snap_known_clear(snap_ctx* ctx);
int snap_known_add(snap_ctx* ctx, const uint64_t* digests, uint64_t n);
/* Adds every digest of the current grid to the known set (after a snapshot
 * has been persisted: the next one is incremental). */
int snap_known_commit(snap_ctx* ctx);
/* K2 (single GPU): first occurrence in canonical order and not known
 * (build_manifest unique_device set, ckpt.cpp:97,157-166), staging offsets by
 * a deterministic decoupled look-back scan. Async. */
int snap_select(snap_ctx* ctx);
/* Copies the selection to the host (any pointer may be NULL).
 * sel[g] in {0,1}; owner[g] = first-occurrence chunk index or UINT64_MAX
 * when known; offsets[g] = staging byte offset of the chunk's bytes
 * (UINT64_MAX when known). */
int snap_get_selection(snap_ctx* ctx, uint8_t* sel, uint64_t* owner, uint64_t* offsets,
                       uint64_t* staged_bytes, uint64_t* staged_chunks);

/* --------------------------------------------------- K3: stream compaction */

/* K3: gathers the selected chunks into the ctx staging image, canonical
 * order (replaces the content_of + BlobStore::put copies, ckpt.cpp:161-163,
 * and host_cache_put, splice.cpp:79-82,266). Async. */
int snap_compact(snap_ctx* ctx);
/* One call = K1 + K2 + K3 (+ K2 exchange when a communicator is attached):
 * the device section of build_manifest (ckpt.cpp:147-167). Async. */
int snap_snapshot(snap_ctx* ctx);
/* End-to-end from HOST memory, the call a checkpoint driver makes
 * (CheckpointFlow -> build_manifest -> persist, ckpt.cpp:543-617): copies
 * `bytes` from host_src into the arena at `addr`, runs snap_snapshot over the
 * installed buffers, and copies the staging image (this rank's shard when a
 * communicator is attached) and the chunk digests back to the host. */
int snap_snapshot_host(snap_ctx* ctx, const void* host_src, uint64_t addr, uint64_t bytes,
                       void* host_staging, uint64_t staging_cap, uint64_t* staged_bytes,
                       uint64_t* host_digests);
int snap_staging(snap_ctx* ctx, void** dev_ptr, uint64_t* bytes);
int snap_read_staging(snap_ctx* ctx, uint64_t off, void* dst, uint64_t bytes);

/* ------------------------------------------------ K4: scatter-restore */

/* K4: restore_job materialization (ckpt.cpp:517-528): chunk g of the
 * installed grid is written at its recorded address from
 * image + src_off[g] (host array, n_chunks entries). `image` is a device
 * pointer (staging of this or a peer ctx, or any device buffer). With
 * verify != 0 the restored chunks are re-hashed against expect_digests
 * (BlobStore::get digest verification, ckpt.cpp:26-27) and SNAP_EFAULT is
 * returned on any mismatch. */
int snap_restore(snap_ctx* ctx, const void* image, uint64_t image_bytes, const uint64_t* src_off,
                 const uint64_t* expect_digests, int verify);
/* Inverse of the last snap_snapshot from this ctx's own staging image. */
int snap_restore_self(snap_ctx* ctx, int verify);

/* --------------------------------------- K5: spliced gradient reduction */

#define SNAP_U64 0
#define SNAP_F32 1
#define SNAP_BF16 2
/* K5: dst[i] = sum_r src_r[i] over `nsrc` arena ranges, fixed ascending order
 * (u64 modular: collectives.cpp:140-141; f32: ((s0+s1)+s2)+..., IEEE RN;
 * bf16: the same left-to-right sum in fp32 of the bf16 values, rounded once to
 * bf16, RN-even). With accumulate != 0, dst is the first addend. Async. */
int snap_grad_sum(snap_ctx* ctx, int dtype, const uint64_t* src_addrs, uint32_t nsrc,
                  uint64_t dst_addr, uint64_t elems, int accumulate);

/* ------------------------------------------------- replica splicing */

/* Context switch between time-sliced ranks sharing this GPU
 * (GpuLedger::plan_switch + execute_switch, splice.cpp:167-306, called by
 * JobRuntime::switch_to, job.cpp:146-198). The reference's host cache becomes a
 * digest-indexed chunk cache in HBM: a fixed array of chunk slots whose chunks
 * no rank records any more are reclaimed when a swap-out could run out of
 * slots (the reference's std::map only grows, splice.hpp:128). */
typedef struct {
  uint64_t hashed_bytes;   /* live bytes of the outgoing rank digested (K1) */
  uint64_t swap_out_bytes; /* bytes newly saved to the chunk cache (K3) */
  uint64_t swap_in_bytes;  /* bytes restored from the chunk cache (K4) */
  uint64_t resident_bytes; /* incoming bytes already in place (same range, same digest) */
  uint64_t cache_bytes;    /* bytes of the chunks the cache holds after the switch */
  uint64_t install_bytes;  /* queued collective results installed (switch_report, job.cpp:165-171) */
  uint64_t cache_free_bytes; /* free slot capacity after the switch */
  uint64_t reclaimed_bytes;  /* bytes reclaimed by the cache so far (cumulative) */
} snap_switch_stats;
/* cache_bytes of HBM in 64 KiB slots (snap_splice_init) or slot_bytes slots
 * (power of two >= 256; a rank's chunk_bytes must not exceed it). */
int snap_splice_init(snap_ctx* ctx, uint64_t cache_bytes);
int snap_splice_init_slots(snap_ctx* ctx, uint64_t cache_bytes, uint32_t slot_bytes);
int snap_splice_set_rank(snap_ctx* ctx, int rank, const snap_buf* bufs, uint64_t n,
                         const snap_geom* geom);
int snap_splice_switch(snap_ctx* ctx, int from, int to, snap_switch_stats* stats);
int snap_splice_recorded(snap_ctx* ctx, int rank, uint64_t* digests, uint64_t* n);
/* Collective-result install for the sliced ranks of this GPU
 * (JobRuntime::on_coll_complete, job.cpp:206-222 -> GpuLedger::install_result,
 * splice.cpp:142-148): the result at arena [src_addr, +bytes) is written into
 * rank ranks[i]'s buffer at dst_addrs[i]. The active rank (the `to` of the last
 * switch; rank < 0 or a ctx without splicing: immediately) gets it now; the
 * others queue it (ProxyServer::install_queue, proxy.hpp:75-79; one library
 * copy of the result shared by the queued entries) and the next
 * snap_splice_switch to that rank applies it after its swap-ins
 * (switch_to, job.cpp:164-171), reported as install_bytes. 16-byte aligned. */
int snap_splice_install(snap_ctx* ctx, const int* ranks, const uint64_t* dst_addrs, uint32_t n,
                        uint64_t src_addr, uint64_t bytes);
/* Queued installs of `rank`: number and bytes. */
int snap_splice_pending(snap_ctx* ctx, int rank, uint64_t* count, uint64_t* bytes);

/* ------------------------------------------------ multi-GPU (NCCL/NVLink) */

int snap_comm_unique_id(void* id128);
int snap_comm_init(snap_ctx* ctx, int nranks, int rank, const void* id128);
/* Collective over the current communicator's ranks (call before re-forming a
 * smaller/larger device-level world on resize, collectives.cpp:37-59). */
int snap_comm_destroy(snap_ctx* ctx);
/* With a communicator attached, snap_select allgathers every rank's digest
 * vector (padded to the largest rank, rank-major) and selects over the global
 * canonical order; selection vectors then have n_global = nranks * max_per_rank
 * entries. Physical copies of replicated chunks are striped over their holders
 * (ranks with the same digest at the same local chunk index):
 * writer = holders[local_index % |holders|]; each rank stages only its shard. */
int snap_global_info(snap_ctx* ctx, uint64_t* n_global, uint64_t* max_per_rank);
int snap_get_global_digests(snap_ctx* ctx, uint64_t* gdig, uint32_t* glens);
/* writer[g] (-1 when not staged) and shard_off[g] (offset inside the writer's
 * shard, UINT64_MAX when not staged) over the global vector; my_bytes /
 * my_chunks = size of this rank's shard. Any pointer may be NULL. */
int snap_get_shard(snap_ctx* ctx, int32_t* writer, uint64_t* shard_off, uint64_t* my_bytes,
                   uint64_t* my_chunks);

/* Resize / reshard (Scheduler::resize -> restore_job, sched.cpp:385-427,
 * ckpt.cpp:407-538): every rank exports its staging shard as a 64-byte CUDA
 * IPC handle, the handles are exchanged out of band (all ranks, rank order),
 * and a target GPU then rebuilds rank `src_rank`'s device state (the
 * installed grid must be that rank's layout) straight from the shards —
 * peer shards are read over NVLink by the same kernel that scatters the
 * chunks to their recorded addresses. verify != 0 re-hashes (K1) against the
 * snapshot's digests (BlobStore::get verification, ckpt.cpp:26-27). */
int snap_ipc_export(snap_ctx* ctx, void* handle64);
int snap_ipc_import(snap_ctx* ctx, int nranks, const void* handles);
int snap_restore_shards(snap_ctx* ctx, int src_rank, int verify);

/* Device-level allreduce of a gradient range (after K5 local sum,
 * collectives.cpp:147-154 local closer) through NCCL (its own reduction
 * order; exact for u64). Async. */
int snap_allreduce(snap_ctx* ctx, int dtype, uint64_t addr, uint64_t elems);
/* Fixed-order device-level allreduce (the CollectiveEngine sum,
 * collectives.cpp:137-154, with the north star's fixed-order fp32 mode),
 * collective: every GPU passes the gradients of its sliced ranks (nlocal <= 16
 * arena ranges, each with a globally unique order key, e.g. its dp rank) and
 * the destination range of its own result. The sum over every source of every
 * GPU is taken in ascending key order, ((g_k0 + g_k1) + g_k2) + ... (u64 mod
 * 2^64; f32 IEEE RN; bf16 in fp32, rounded once) — bit-identical on every GPU
 * and to a CPU left-to-right sum. One fused kernel per GPU reads its 1/N slice
 * of every source (peer arenas over NVLink, CUDA IPC) and stores the summed
 * slice into every GPU's destination: reduce-scatter + all-gather in one pass
 * over peer memory. The destination may be one of the sources. Passing one
 * K5 partial sum per GPU (key = GPU index) gives the hierarchical order. */
int snap_allreduce_ordered(snap_ctx* ctx, int dtype, const uint32_t* keys, const uint64_t* src_addrs,
                           uint32_t nlocal, uint64_t dst_addr, uint64_t elems);
/* In-process communicator: `nranks` ctxs driven by threads of one process
 * (e.g. N ranks emulated on one GPU, the reference's whole-fleet-in-one-process
 * model) join the group named `key`; every collective entry point then works
 * as with NCCL (collectives through host memory, IPC handles of this process
 * resolved to the exporting ctx's buffers). Blocks until all ranks joined.
 * Released by snap_comm_destroy / snap_close. */
int snap_comm_init_local(snap_ctx* ctx, int nranks, int rank, const char* key);

/* ------------------------------------- squash-window validation (§8f-3) */

/* One entry of a rank's mutation set: ValidationRecord::mutations
 * (splice.hpp:50-53), addr -> (bytes, digest after the window). */
typedef struct {
  uint64_t addr;
  uint64_t bytes;
  uint64_t digest;
} snap_mutation;

/* WorkerExec::do_window_open, validation branch (worker.cpp:355-362): K1
 * digests every live, non-pending buffer of `rank` (SNAP_BUF_PENDING skipped)
 * and keeps addr -> (bytes, digest) as the rank's open snapshot. Uses the
 * ctx's auxiliary grid: the installed snapshot grid is left untouched. */
int snap_window_open(snap_ctx* ctx, int rank, const snap_buf* bufs, uint64_t n);
/* do_window_close, validation branch (worker.cpp:411-421): re-digests the
 * rank's live, non-pending buffers; the mutation set = every buffer whose
 * address is new or whose digest or size changed, in address order.
 * *n_out = its size; `out` (capacity `cap`) may be NULL to query the size. */
int snap_window_close(snap_ctx* ctx, int rank, const snap_buf* bufs, uint64_t n,
                      snap_mutation* out, uint64_t cap, uint64_t* n_out);
/* One rank's ValidationRecord: its mutation set (address order) and the
 * in-window D2H copies as (bytes, digest) pairs in issue order
 * (worker.cpp:664-669; digests from snap_digest_ranges). */
typedef struct {
  int32_t rank;
  const snap_mutation* mutations;
  uint64_t n_mutations;
  const uint64_t* d2h; /* 2 * n_d2h words: bytes, digest */
  uint64_t n_d2h;
} snap_window_record;
/* splice::validate_window (splice.cpp:21-61): records compared against the
 * lowest rank's in rank order; returns 1 = pass, 0 = fail (reason written to
 * `reason`, same text as the reference), <0 = error. Host only. */
int snap_validate_window(const snap_window_record* recs, uint64_t n, char* reason,
                         uint64_t cap);

/* --------------------------------------------- host-page snapshot (§8f-4) */

typedef struct {
  uint64_t pages;        /* 4 KiB pages of the rank (WorkerSnapshot::pages size) */
  uint64_t s_cr;         /* pages * 4096 (Manifest::s_cr contribution) */
  uint64_t s_cr_inc;     /* bytes of pages absent from the previous page set */
  uint64_t upload_bytes; /* bytes of fresh pages: first occurrence, not in the known set */
} snap_pages_stats;
#define SNAP_PAGE_FRESH 1u /* flags[p] bit: BlobStore::put would store it (ckpt.cpp:18-20) */
#define SNAP_PAGE_INC 2u   /* flags[p] bit: not in the previous checkpoint's page set */

/* build_manifest host section (ckpt.cpp:59-68, 116-130) for one rank: the
 * host buffers (bufs[i], words[i] u64 words each, in slot order) are
 * concatenated and zero-padded to 4 KiB pages (paged_host_words); the page
 * digests digest_of_words(page) are computed on the GPU (H2D + K1 with
 * page == chunk == 4 KiB), and each page is classified against the ctx's known
 * set (the store index) and against prev_pages (the rank's page list in the
 * previous manifest, may be NULL). page_digests (capacity cap) and flags
 * (SNAP_PAGE_*) may be NULL; stats->pages is always set. The installed grid is
 * not touched. Add the fresh digests to the known set (snap_known_add) once
 * the pages are persisted. */
int snap_host_pages(snap_ctx* ctx, const void* const* bufs, const uint64_t* words, uint64_t nbufs,
                    const uint64_t* prev_pages, uint64_t n_prev, uint64_t* page_digests,
                    uint64_t cap, uint8_t* flags, snap_pages_stats* stats);

/* ------------------------------------- on-disk format (persist / load) */

/* BlobStore::blob_rel_path (ckpt.cpp:35-40): "blobs/<2hex>/<16hex>" of the
 * digest, NUL-terminated into out (cap >= 32). Host only, no context. */
int snap_blob_rel_path(uint64_t digest, char* out, uint64_t cap);

typedef struct {
  uint64_t blobs;         /* blobs this rank staged (its files to write / files read) */
  uint64_t written;       /* files created by this call */
  uint64_t present;       /* already in the directory: content-addressed, skipped */
  uint64_t bytes;         /* bytes written (upload_bytes) or read */
  uint64_t layout_chunks; /* chunks of the rank's layout */
  uint64_t layout_blobs;  /* distinct blobs the layout references */
  uint64_t layout_bytes;  /* their bytes (total_blob_bytes) */
  uint64_t layout_bufs;   /* buffer records of the layout (installed by snap_load) */
} snap_persist_stats;

/* BlobStore::persist (ckpt.cpp:42-52) for the last snapshot plus the
 * manifest's device section (ckpt.cpp:194-262): every chunk this rank staged
 * (its shard when a communicator is attached) becomes
 * <dir>/blobs/<2hex>/<16hex> holding the chunk's bytes (tmp + rename; blobs
 * already present are skipped, like a non-fresh BlobStore::put). The rank's
 * layout (buffer records + chunk digests) goes to <dir>/layout.<rank>.snapl
 * (read by snap_load) and <dir>/manifest.dev.<rank>.json. Blob names are the
 * chunk digests of the installed geometry; with page_bytes == chunk_bytes the
 * name is digest_of_words(content) and the files are byte-identical to what
 * the reference's BlobStore writes for those chunks. host_image (optional) is
 * this rank's staging image already on the host (snap_snapshot_host output);
 * otherwise the device staging is streamed out through pinned slabs.
 * nthreads <= 0: one writer thread per core, at most 16. */
int snap_persist(snap_ctx* ctx, const char* dir, const void* host_image, uint64_t host_bytes,
                 int nthreads, snap_persist_stats* stats);
/* snap_persist with an explicit layout id (time-sliced ranks share one GPU and
 * one ctx: each rank's cut is persisted as layout.<its rank>). snap_persist
 * uses the communicator rank (0 without one). */
int snap_persist_rank(snap_ctx* ctx, const char* dir, int layout_rank, const void* host_image,
                      uint64_t host_bytes, int nthreads, snap_persist_stats* stats);
/* restore_job materialization from a directory (ckpt.cpp:504-533): installs
 * rank `rank`'s layout, streams every referenced blob through pinned slabs to
 * the device and scatters the chunks to their recorded addresses (K4).
 * verify != 0 re-hashes the restored grid (BlobStore::get verification,
 * ckpt.cpp:26-27): SNAP_EFAULT on a corrupt, truncated or missing blob. */
int snap_load(snap_ctx* ctx, const char* dir, int rank, int verify, int nthreads,
              snap_persist_stats* stats);
/* The rest of restore_job's materialization for a GPU (ckpt.cpp:517-528): a
 * co-resident (time-sliced, currently inactive) rank's persisted layout
 * becomes splice rank `splice_rank`'s buffer map, and every chunk whose digest
 * the HBM chunk cache does not hold yet is streamed in from the blob files
 * (the reference copies it into its host cache). A later snap_splice_switch to
 * that rank restores it from the cache, or finds it resident. Needs
 * snap_splice_init; SNAP_EFAULT on a missing or truncated blob. */
int snap_splice_load(snap_ctx* ctx, const char* dir, int layout_rank, int splice_rank,
                     int nthreads, snap_persist_stats* stats);

/* ---------------------------------------------------------- timing */

int snap_timer_start(snap_ctx* ctx);
int snap_timer_stop(snap_ctx* ctx, float* ms);
/* Per-kernel-class CUDA events on the ctx stream (live roofline evidence):
 * kind 0 hash, 1 select, 2 compact, 3 restore, 4 grad, 5 exchange, 6 splice switch. */
#define SNAP_PROF_HASH 0
#define SNAP_PROF_SELECT 1
#define SNAP_PROF_COMPACT 2
#define SNAP_PROF_RESTORE 3
#define SNAP_PROF_GRAD 4
#define SNAP_PROF_EXCHANGE 5
#define SNAP_PROF_SWITCH 6 /* a whole snap_splice_switch: first launch .. last kernel */
int snap_prof_enable(snap_ctx* ctx, int on);
int snap_prof_read(snap_ctx* ctx, int kind, float* total_ms, uint64_t* count);

/* K1 kernel policy for this process (tuning / A-B measurement; no reference
 * counterpart). -1 = default per-launch choice; 9 = cp.async kernel, 10 = TMA
 * tensor loads, 11 = tensor-core FNV (8-bit chain on the CUDA cores + linear
 * part as a tcgen05 int8 MMA); the other values force measured alternatives.
 * Every variant yields identical digests. Applies to grids installed after
 * the call (the TMA-based kernels need tensor maps built at install time). */
int snap_set_k1_variant(int variant);
/* Name of the K1 kernel the most recent hash launch of this process used
 * (measurement labels; static string). */
const char* snap_last_k1_kernel(void);

#ifdef __cplusplus
}
#endif
#endif /* SNAP_H */
