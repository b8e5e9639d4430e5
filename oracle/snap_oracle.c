/*
 * snap_oracle.c — CPU restatement of the reference's hot path (TEST
 * INFRASTRUCTURE ONLY; see snap_oracle.h). Each function cites the reference
 * lines it restates. Plain C, optional OpenMP across independent chunks.
 */
#include "snap_oracle.h"

#include <stdlib.h>
#include <string.h>

#define FNV_OFFSET 14695981039346656037ull /* sim.hpp:57 */
#define FNV_PRIME 1099511628211ull         /* sim.hpp:58 */

/* sim.hpp:58-65 — h = offset; for each byte: h ^= b; h *= prime. */
uint64_t or_fnv1a(const void* bytes, uint64_t n, uint64_t h) {
  const uint8_t* p = (const uint8_t*)bytes;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= FNV_PRIME;
  }
  return h;
}

/* sim.hpp:67-70 — the little-endian bytes of the words. */
uint64_t or_digest_of_words(const uint64_t* words, uint64_t n) {
  return or_fnv1a(words, n * 8, FNV_OFFSET);
}

/* sim.hpp:37-41 */
uint64_t or_mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

void or_fill_mix64(uint64_t* dst, uint64_t nwords, uint64_t seed, uint64_t base) {
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < nwords; ++i) dst[i] = or_mix64(seed ^ (base + i));
}

static uint64_t nchunks_of(uint64_t bytes, uint32_t chunk_bytes) {
  return (bytes + chunk_bytes - 1) / chunk_bytes;
}

uint64_t or_num_chunks(const or_buf* bufs, uint64_t n, uint32_t chunk_bytes) {
  uint64_t t = 0;
  for (uint64_t b = 0; b < n; ++b) t += nchunks_of(bufs[b].bytes, chunk_bytes);
  return t;
}

/* Digest of one chunk: direct FNV when page == chunk, else FNV
 * over the page digests (each page digest = digest_of_words(page), i.e. the
 * value BlobStore::put returns for that page, ckpt.cpp:16-17,122-130). */
static uint64_t chunk_digest(const uint8_t* p, uint64_t len, uint32_t page_bytes,
                             uint32_t chunk_bytes) {
  if (page_bytes == chunk_bytes) return or_fnv1a(p, len, FNV_OFFSET);
  uint64_t pd[1024];
  uint64_t np = (len + page_bytes - 1) / page_bytes;
  for (uint64_t q = 0; q < np; ++q) {
    uint64_t off = q * page_bytes;
    uint64_t pl = len - off < page_bytes ? len - off : page_bytes;
    pd[q] = or_fnv1a(p + off, pl, FNV_OFFSET);
  }
  return or_digest_of_words(pd, np);
}

int or_hash(const uint8_t* const* arenas, const or_buf* bufs, uint64_t n, uint32_t page_bytes,
            uint32_t chunk_bytes, uint64_t* chunk_digests, uint32_t* chunk_lens,
            uint64_t* buf_digests, int nthreads) {
  if (page_bytes == 0 || chunk_bytes % page_bytes || chunk_bytes / page_bytes > 1024) return -1;
  uint64_t* start = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
  start[0] = 0;
  for (uint64_t b = 0; b < n; ++b) start[b + 1] = start[b] + nchunks_of(bufs[b].bytes, chunk_bytes);
  uint64_t total = start[n];
  /* flatten (buffer, chunk) for a chunk-parallel loop */
  uint64_t* owner_buf = (uint64_t*)malloc((total ? total : 1) * sizeof(uint64_t));
  for (uint64_t b = 0; b < n; ++b)
    for (uint64_t g = start[b]; g < start[b + 1]; ++g) owner_buf[g] = b;
  (void)nthreads;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : 1)
  for (uint64_t g = 0; g < total; ++g) {
    uint64_t b = owner_buf[g];
    uint64_t k = g - start[b];
    uint64_t off = k * chunk_bytes;
    uint64_t len = bufs[b].bytes - off < chunk_bytes ? bufs[b].bytes - off : chunk_bytes;
    const uint8_t* p = arenas[bufs[b].rank] + bufs[b].addr + off;
    chunk_digests[g] = chunk_digest(p, len, page_bytes, chunk_bytes);
    if (chunk_lens) chunk_lens[g] = (uint32_t)len;
  }
  if (buf_digests)
    for (uint64_t b = 0; b < n; ++b)
      buf_digests[b] = or_digest_of_words(chunk_digests + start[b], start[b + 1] - start[b]);
  free(owner_buf);
  free(start);
  return 0;
}

/* ---- a tiny open-addressing map digest -> first index ------------------- */
typedef struct {
  uint64_t* key;
  uint64_t* val;
  uint8_t* used;
  uint64_t mask;
} omap;

static void omap_init(omap* m, uint64_t n) {
  uint64_t cap = 16;
  while (cap < 2 * n + 16) cap <<= 1;
  m->key = (uint64_t*)malloc(cap * 8);
  m->val = (uint64_t*)malloc(cap * 8);
  m->used = (uint8_t*)calloc(cap, 1);
  m->mask = cap - 1;
}
static void omap_free(omap* m) {
  free(m->key);
  free(m->val);
  free(m->used);
}
/* returns pointer to the value slot; *fresh = 1 if inserted */
static uint64_t* omap_slot(omap* m, uint64_t k, int* fresh) {
  uint64_t i = or_mix64(k) & m->mask;
  for (;;) {
    if (!m->used[i]) {
      m->used[i] = 1;
      m->key[i] = k;
      *fresh = 1;
      return &m->val[i];
    }
    if (m->key[i] == k) {
      *fresh = 0;
      return &m->val[i];
    }
    i = (i + 1) & m->mask;
  }
}
static int omap_has(const omap* m, uint64_t k) {
  uint64_t i = or_mix64(k) & m->mask;
  for (;;) {
    if (!m->used[i]) return 0;
    if (m->key[i] == k) return 1;
    i = (i + 1) & m->mask;
  }
}

/* build_manifest device loop (ckpt.cpp:147-167): ranks ascending, slots
 * ascending; the first occurrence of a digest is the one stored (S_G), and
 * BlobStore::put counts only store-fresh bytes (ckpt.cpp:18-20,162-164). */
uint64_t or_select(const uint64_t* d, const uint32_t* lens, uint64_t n, const uint64_t* known,
                   uint64_t nknown, uint8_t* sel, uint64_t* owner, uint64_t* offsets) {
  omap kn, first;
  omap_init(&kn, nknown);
  omap_init(&first, n);
  int fresh;
  for (uint64_t i = 0; i < nknown; ++i) omap_slot(&kn, known[i], &fresh);
  uint64_t off = 0;
  for (uint64_t g = 0; g < n; ++g) {
    if (omap_has(&kn, d[g])) {
      sel[g] = 0;
      owner[g] = UINT64_MAX;
      offsets[g] = UINT64_MAX;
      continue;
    }
    uint64_t* v = omap_slot(&first, d[g], &fresh);
    if (fresh) {
      *v = g;
      sel[g] = 1;
      owner[g] = g;
      offsets[g] = off;
      off += lens[g];
    } else {
      sel[g] = 0;
      owner[g] = *v;
      offsets[g] = offsets[*v];
    }
  }
  omap_free(&kn);
  omap_free(&first);
  return off;
}

void or_stripe(const uint64_t* d, const uint32_t* lens, const uint64_t* n_per_rank, uint32_t world,
               const uint8_t* sel, int32_t* writer, uint64_t* shard_off, uint64_t* shard_bytes) {
  uint64_t* base = (uint64_t*)malloc((world + 1) * 8);
  base[0] = 0;
  for (uint32_t r = 0; r < world; ++r) base[r + 1] = base[r] + n_per_rank[r];
  for (uint32_t r = 0; r < world; ++r) shard_bytes[r] = 0;
  for (uint32_t r = 0; r < world; ++r) {
    for (uint64_t i = 0; i < n_per_rank[r]; ++i) {
      uint64_t g = base[r] + i;
      if (!sel[g]) {
        writer[g] = -1;
        shard_off[g] = UINT64_MAX;
        continue;
      }
      uint32_t holders[1024];
      uint32_t nh = 0;
      for (uint32_t q = 0; q < world; ++q)
        if (i < n_per_rank[q] && d[base[q] + i] == d[g] && lens[base[q] + i] == lens[g])
          holders[nh++] = q;
      uint32_t w = holders[i % nh];
      writer[g] = (int32_t)w;
      shard_off[g] = shard_bytes[w];
      shard_bytes[w] += lens[g];
    }
  }
  free(base);
}

void or_compact(const uint8_t* const* arenas, const or_buf* bufs, uint64_t n, uint32_t chunk_bytes,
                const uint8_t* sel, const uint64_t* offsets, uint8_t* staging) {
  uint64_t g = 0;
  for (uint64_t b = 0; b < n; ++b) {
    uint64_t nc = nchunks_of(bufs[b].bytes, chunk_bytes);
    for (uint64_t k = 0; k < nc; ++k, ++g) {
      if (!sel[g]) continue;
      uint64_t off = k * chunk_bytes;
      uint64_t len = bufs[b].bytes - off < chunk_bytes ? bufs[b].bytes - off : chunk_bytes;
      memcpy(staging + offsets[g], arenas[bufs[b].rank] + bufs[b].addr + off, len);
    }
  }
}

/* restore_job materialization (ckpt.cpp:517-528): bytes land at the same
 * addresses they were dumped from. */
void or_restore(uint8_t* const* arenas, const or_buf* bufs, uint64_t n, uint32_t chunk_bytes,
                const uint8_t* image, const uint64_t* src_off) {
  uint64_t g = 0;
  for (uint64_t b = 0; b < n; ++b) {
    uint64_t nc = nchunks_of(bufs[b].bytes, chunk_bytes);
    for (uint64_t k = 0; k < nc; ++k, ++g) {
      uint64_t off = k * chunk_bytes;
      uint64_t len = bufs[b].bytes - off < chunk_bytes ? bufs[b].bytes - off : chunk_bytes;
      memcpy(arenas[bufs[b].rank] + bufs[b].addr + off, image + src_off[g], len);
    }
  }
}

/* collectives.cpp:140-141: p.sum[i] += contrib[i] (u64, wraps mod 2^64). */
void or_grad_sum_u64(const uint64_t* const* grads, uint32_t nranks, uint64_t n, uint64_t* out) {
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t s = 0;
    for (uint32_t r = 0; r < nranks; ++r) s += grads[r][i];
    out[i] = s;
  }
}

/* fp32 fixed order: ascending dp index (job.cpp:45-50 resident order),
 * ((g0 + g1) + g2) + ... with IEEE round-to-nearest per add. */
void or_grad_sum_f32(const float* const* grads, uint32_t nranks, uint64_t n, float* out) {
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < n; ++i) {
    volatile float s = grads[0][i];
    for (uint32_t r = 1; r < nranks; ++r) s = s + grads[r][i];
    out[i] = s;
  }
}

/* bf16 gradients (C5): the same ascending-order chain in fp32 over the bf16
 * values, rounded once to bf16 (round to nearest, ties to even; NaN stays a
 * quiet NaN). */
static float or_bf16_to_f32(uint16_t h) {
  union { uint32_t u; float f; } x;
  x.u = (uint32_t)h << 16;
  return x.f;
}
static uint16_t or_f32_to_bf16(float f) {
  union { uint32_t u; float f; } x;
  x.f = f;
  if ((x.u & 0x7f800000u) == 0x7f800000u && (x.u & 0x007fffffu)) return (uint16_t)((x.u >> 16) | 0x40);
  x.u += 0x7fffu + ((x.u >> 16) & 1u);
  return (uint16_t)(x.u >> 16);
}
void or_grad_sum_bf16(const uint16_t* const* grads, uint32_t nranks, uint64_t n, uint16_t* out) {
#pragma omp parallel for schedule(static)
  for (uint64_t i = 0; i < n; ++i) {
    volatile float s = or_bf16_to_f32(grads[0][i]);
    for (uint32_t r = 1; r < nranks; ++r) s = s + or_bf16_to_f32(grads[r][i]);
    out[i] = or_f32_to_bf16(s);
  }
}
