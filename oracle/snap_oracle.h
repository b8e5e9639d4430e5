/*
 * snap_oracle.h — CPU restatement of the reference's snapshot/restore/splice
 * hot path. TEST INFRASTRUCTURE ONLY: imported by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline leg.
 * The product (paper_2202_07848_b200/libsnap.so) never links or calls it.
 *
 * Parity pinning: every digest function here is checked against
 *   (1) the reference's own known-answer tests (test_simcore.cpp:107-117),
 *   (2) the golden vectors in SURVEY.md Appendix B, and
 *   (3) the reference library itself, compiled from /root/reference by
 *       oracle/Makefile into oracle/_ref/ (tests/test_oracle.py).
 */
#ifndef SNAP_ORACLE_H
#define SNAP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* sim::digest_of (proj/include/fleetsim/sim.hpp:55-65): 64-bit FNV-1a. */
uint64_t or_fnv1a(const void* bytes, uint64_t n, uint64_t h);
/* sim::digest_of_words (sim.hpp:67-70). */
uint64_t or_digest_of_words(const uint64_t* words, uint64_t n);
/* sim::mix64 (sim.hpp:37-41). */
uint64_t or_mix64(uint64_t x);
/* words[i] = mix64(seed ^ (base + i)) — the synthetic content of SURVEY §8(d). */
void or_fill_mix64(uint64_t* dst, uint64_t nwords, uint64_t seed, uint64_t base);

/* One tracked allocation: RankBuf/DevRec (splice.hpp:26-34, ckpt.hpp:64-71). */
typedef struct {
  uint32_t rank;
  int32_t slot;
  uint64_t addr;  /* byte offset in the rank's device arena */
  uint64_t bytes; /* multiple of 256 (alloc.cpp:64 rounding) */
  int32_t cat;
  uint32_t flags;
} or_buf;

/* Number of chunks of the grid (SURVEY §8c "CPU restatement"). */
uint64_t or_num_chunks(const or_buf* bufs, uint64_t n, uint32_t chunk_bytes);

/* Per-chunk digests over the chunk grid.
 * page digest  = digest_of_words(page bytes)
 * chunk digest = page_bytes == chunk_bytes ? digest_of_words(chunk bytes)
 *                                          : digest_of_words(page digests)
 * buffer digest = digest_of_words(chunk digests of the buffer)
 * arenas[rank] is the host copy of that rank's device memory.
 * chunk_lens (nullable) receives each chunk's byte length. */
int or_hash(const uint8_t* const* arenas, const or_buf* bufs, uint64_t n, uint32_t page_bytes,
            uint32_t chunk_bytes, uint64_t* chunk_digests, uint32_t* chunk_lens,
            uint64_t* buf_digests, int nthreads);

/* Selection = cross-rank/spatial dedup + dirty test (ckpt.cpp:97,157-166,18-20):
 * sel[g] = first occurrence of d[g] in canonical order && d[g] not in known[].
 * owner[g] = index of the first occurrence (UINT64_MAX if d[g] is known).
 * offsets[g] = staging byte offset of chunk g if sel[g] (else of its owner, or
 * UINT64_MAX when known). Returns total staged bytes. */
uint64_t or_select(const uint64_t* d, const uint32_t* lens, uint64_t n, const uint64_t* known,
                   uint64_t nknown, uint8_t* sel, uint64_t* owner, uint64_t* offsets);

/* Physical writer of each selected chunk for a world of `world` ranks whose
 * canonical chunk vectors are d_r (rank-major concatenation, n_per_rank[r]
 * each): holders = ranks whose chunk at the same local index has the same
 * digest; writer = holders[local_index % |holders|]. writer[g] = -1 when not
 * selected. shard_off[g] = byte offset in the writer's staging shard. */
void or_stripe(const uint64_t* d, const uint32_t* lens, const uint64_t* n_per_rank, uint32_t world,
               const uint8_t* sel, int32_t* writer, uint64_t* shard_off, uint64_t* shard_bytes);

/* Stream compaction into the staging image (canonical order). */
void or_compact(const uint8_t* const* arenas, const or_buf* bufs, uint64_t n, uint32_t chunk_bytes,
                const uint8_t* sel, const uint64_t* offsets, uint8_t* staging);

/* Inverse scatter-restore (ckpt.cpp:517-528): chunk g of the layout is written
 * at its recorded address from image + src_off[g]. */
void or_restore(uint8_t* const* arenas, const or_buf* bufs, uint64_t n, uint32_t chunk_bytes,
                const uint8_t* image, const uint64_t* src_off);

/* Spliced-replica gradient sum (collectives.cpp:137-144, worker.cpp:290-297):
 * u64 modular and fp32 fixed (ascending dp) order. */
void or_grad_sum_u64(const uint64_t* const* grads, uint32_t nranks, uint64_t n, uint64_t* out);
void or_grad_sum_f32(const float* const* grads, uint32_t nranks, uint64_t n, float* out);
void or_grad_sum_bf16(const uint16_t* const* grads, uint32_t nranks, uint64_t n, uint16_t* out);

#ifdef __cplusplus
}
#endif
#endif
