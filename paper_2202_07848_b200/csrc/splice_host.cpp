// splice_host.cpp — replica splicing context switch (GpuLedger::plan_switch /
// execute_switch, splice.cpp:167-306, driven by JobRuntime::switch_to,
// job.cpp:146-198), B200-native:
//  * the reference's host cache (std::map<digest, words>, splice.hpp:128) is a
//    digest-indexed CHUNK cache in spare HBM (180 GB per GPU holds several
//    replicas' state), so swap-out/in are D2D copies at HBM speed instead of
//    PCIe transfers, and dedup is per 64 KiB chunk instead of per buffer;
//  * swap-out = K1 hash of the outgoing rank's live, non-pending buffers +
//    K2 selection against the cache index + K3 gather of the new chunks;
//  * swap-in = one pass over the incoming rank's chunks: resident when the
//    fresh digest of the same address range equals the incoming rank's
//    recorded digest (the stale-digest defect of SURVEY App. A-1 is fixed by
//    construction: the comparison uses the digests just computed), else a
//    copy from the cache by digest; a missing digest is a SimFault.
// One host sync per switch (cache cursor + the switch report of job.cpp:181-195).
#include "ctx.h"

struct RankGrid {
  std::vector<snap_buf> bufs;
  std::vector<uint64_t> cstart;
  std::vector<uint32_t> lens;
  std::vector<uint64_t> chunk_addr;
  uint64_t nchunks = 0, bytes = 0;
  DevMem d_addr, d_bytes, d_cstart, d_lens, d_rec, d_tmaps;
  GridDev grid;
  bool recorded = false;
};

struct SpliceState {
  uint64_t cap = 0, cursor = 0, entries = 0;
  DevMem cache, ck, cv, counters, seed_off;
  uint64_t cmask = 0;
  std::map<int, RankGrid> ranks;
  std::map<std::pair<int, int>, DevMem> match;
  int active = -1;
};

void splice_release(snap_ctx* ctx) {
  SpliceState* S = ctx->splice;
  if (!S) return;
  for (auto& [r, g] : S->ranks)
    for (DevMem* m : {&g.d_addr, &g.d_bytes, &g.d_cstart, &g.d_lens, &g.d_rec, &g.d_tmaps})
      release(*m);
  for (auto& [k, m] : S->match) release(m);
  for (DevMem* m : {&S->cache, &S->ck, &S->cv, &S->counters, &S->seed_off}) release(*m);
  delete S;
  ctx->splice = nullptr;
}

extern "C" {

int snap_splice_init(snap_ctx* ctx, uint64_t cache_bytes) {
  if (!ctx || cache_bytes == 0) return SNAP_EINVAL;
  CK(cudaSetDevice(ctx->device));
  splice_release(ctx);
  ctx->splice = new SpliceState();
  SpliceState* S = ctx->splice;
  S->cap = (cache_bytes + 255) / 256 * 256;
  uint8_t* c;
  RC(ensure(ctx, S->cache, S->cap, &c));
  const uint64_t tcap = table_cap(std::max<uint64_t>(S->cap / 4096, 1024));
  unsigned long long *k, *v, *cnt;
  RC(ensure(ctx, S->ck, tcap + 1, &k));
  RC(ensure(ctx, S->cv, tcap + 1, &v));
  RC(ensure(ctx, S->counters, 4, &cnt));
  S->cmask = tcap - 1;
  CKL(snap::launch_table_clear(TableDev{k, v, S->cmask}, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

// The rank's live buffers (its RankBuf map, splice.hpp:26-34) in slot order;
// buffers flagged SNAP_BUF_PENDING (pending_result: consumed by the local
// gradient accumulation, splice.cpp:175) are neither hashed nor swapped.
int snap_splice_set_rank(snap_ctx* ctx, int rank, const snap_buf* bufs, uint64_t n,
                         const snap_geom* geom) {
  if (!ctx || !ctx->splice || rank < 0 || (!bufs && n)) return SNAP_EINVAL;
  snap_geom g = geom ? *geom : snap_geom{4096, 65536};
  if (!pow2(g.page_bytes) || !pow2(g.chunk_bytes) || g.page_bytes < 256 ||
      g.chunk_bytes < g.page_bytes || g.chunk_bytes / g.page_bytes > 32)
    return fail(ctx, SNAP_EINVAL, "splice: bad geometry");
  CK(cudaSetDevice(ctx->device));
  SpliceState* S = ctx->splice;
  RankGrid& R = S->ranks[rank];
  R.bufs.clear();
  for (uint64_t i = 0; i < n; ++i)
    if (!(bufs[i].flags & SNAP_BUF_PENDING)) R.bufs.push_back(bufs[i]);
  const uint64_t nb = R.bufs.size();
  std::vector<uint64_t> addr(nb), bytes(nb);
  R.cstart.assign(nb + 1, 0);
  R.lens.clear();
  R.chunk_addr.clear();
  R.bytes = 0;
  for (uint64_t b = 0; b < nb; ++b) {
    const snap_buf& x = R.bufs[b];
    if (x.bytes == 0 || x.addr % 256 || x.bytes % 256)
      return fail(ctx, SNAP_EINVAL, "splice: buffers must be non-zero 256-byte multiples");
    RC(check_range(ctx, x.addr, x.bytes));
    addr[b] = x.addr;
    bytes[b] = x.bytes;
    const uint64_t nc = (x.bytes + g.chunk_bytes - 1) / g.chunk_bytes;
    R.cstart[b + 1] = R.cstart[b] + nc;
    for (uint64_t k = 0; k < nc; ++k) {
      R.lens.push_back(uint32_t(std::min<uint64_t>(g.chunk_bytes, x.bytes - k * g.chunk_bytes)));
      R.chunk_addr.push_back(x.addr + k * g.chunk_bytes);
    }
    R.bytes += x.bytes;
  }
  R.nchunks = R.cstart[nb];
  uint64_t *da, *db, *dc, *dr;
  uint32_t* dl;
  RC(ensure(ctx, R.d_addr, nb, &da));
  RC(ensure(ctx, R.d_bytes, nb, &db));
  RC(ensure(ctx, R.d_cstart, nb + 1, &dc));
  RC(ensure(ctx, R.d_lens, R.nchunks, &dl));
  RC(ensure(ctx, R.d_rec, R.nchunks, &dr));
  CK(cudaMemcpyAsync(da, addr.data(), nb * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(db, bytes.data(), nb * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dc, R.cstart.data(), (nb + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dl, R.lens.data(), R.nchunks * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  R.grid = GridDev{da, db, dc, uint32_t(nb), R.nchunks, log2u(g.page_bytes), log2u(g.chunk_bytes)};
  build_tmaps(ctx, R.d_tmaps, addr.data(), bytes.data(), uint32_t(nb), R.grid);
  R.recorded = false;
  for (auto it = S->match.begin(); it != S->match.end();) {
    if (it->first.first == rank || it->first.second == rank) {
      release(it->second);
      it = S->match.erase(it);
    } else {
      ++it;
    }
  }
  return SNAP_OK;
}

// JobRuntime::switch_to(from -> to): from/to may be -1 (first activation /
// drained GPU). A rank that was never switched out has no recorded content:
// switching to it installs nothing (its buffers are created by its own run).
int snap_splice_switch(snap_ctx* ctx, int from, int to, snap_switch_stats* st) {
  if (!ctx || !ctx->splice) return SNAP_EINVAL;
  SpliceState* S = ctx->splice;
  if ((from >= 0 && !S->ranks.count(from)) || (to >= 0 && !S->ranks.count(to)))
    return fail(ctx, SNAP_EINVAL, "splice: unknown rank");
  CK(cudaSetDevice(ctx->device));
  TableDev cache{P<unsigned long long>(S->ck), P<unsigned long long>(S->cv), S->cmask};
  snap_switch_stats out{};
  RankGrid* F = from >= 0 ? &S->ranks[from] : nullptr;
  RankGrid* T = to >= 0 ? &S->ranks[to] : nullptr;
  if (F) {
    if (S->cursor + F->bytes > S->cap)
      return fail(ctx, SNAP_ENOMEM, "splice: chunk cache full (" + std::to_string(S->cursor) +
                                        " of " + std::to_string(S->cap) + " bytes used)");
    // swap-out: refresh digests (K1), select against the cache (K2), gather (K3)
    CKL(snap::launch_hash(ctx->arena, F->grid, P<uint64_t>(F->d_rec), nullptr, nullptr,
                          ctx->stream));
    F->recorded = true;
    RC(select_with_known(ctx, P<uint64_t>(F->d_rec), P<uint32_t>(F->d_lens), F->nchunks, cache,
                         S->entries > 0));
    ctx->selected = false;  // the ctx selection vectors now hold this plan
    CKL(snap::launch_gather(ctx->arena, F->grid, P<uint32_t>(F->d_lens), P<uint32_t>(ctx->sel_list),
                            P<uint64_t>(ctx->totals), P<uint64_t>(ctx->offsets), false, nullptr,
                            nullptr, P<uint8_t>(S->cache) + S->cursor, F->nchunks, ctx->stream));
    CKL(snap::launch_cache_insert(cache, P<uint64_t>(F->d_rec), P<uint32_t>(ctx->sel_list),
                                  P<uint64_t>(ctx->totals), P<uint64_t>(ctx->offsets), S->cursor,
                                  F->nchunks, ctx->stream));
    out.hashed_bytes = F->bytes;
  }
  unsigned long long cnt[3] = {0, 0, 0};
  if (T && T->recorded) {
    const int64_t* match = nullptr;
    if (F) {
      auto key = std::make_pair(from, to);
      if (!S->match.count(key)) {
        std::map<uint64_t, std::pair<int64_t, uint32_t>> at;  // chunk addr -> (index, len)
        for (uint64_t g = 0; g < F->nchunks; ++g) at[F->chunk_addr[g]] = {int64_t(g), F->lens[g]};
        std::vector<int64_t> m(T->nchunks, -1);
        for (uint64_t g = 0; g < T->nchunks; ++g) {
          auto it = at.find(T->chunk_addr[g]);
          if (it != at.end() && it->second.second == T->lens[g]) m[g] = it->second.first;
        }
        int64_t* dm;
        RC(ensure(ctx, S->match[key], T->nchunks, &dm));
        CK(cudaMemcpyAsync(dm, m.data(), T->nchunks * 8, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
      }
      match = P<int64_t>(S->match[key]);
    }
    CKL(snap::launch_splice_in(ctx->arena, T->grid, P<uint32_t>(T->d_lens), P<uint64_t>(T->d_rec),
                               match, F ? P<uint64_t>(F->d_rec) : nullptr, cache,
                               P<uint8_t>(S->cache), P<unsigned long long>(S->counters),
                               ctx->stream));
    CK(cudaMemcpyAsync(cnt, S->counters.p, 24, cudaMemcpyDeviceToHost, ctx->stream));
  }
  uint64_t tot[2] = {0, 0};
  if (F) CK(cudaMemcpyAsync(tot, ctx->totals.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  S->cursor += tot[1];
  S->entries += tot[0];
  S->active = to;
  out.swap_out_bytes = tot[1];
  out.swap_in_bytes = cnt[0];
  out.resident_bytes = cnt[1];
  out.cache_bytes = S->cursor;
  if (st) *st = out;
  if (cnt[2])
    return fail(ctx, SNAP_EFAULT, "splice: content for " + std::to_string(cnt[2]) +
                                      " chunk digest(s) lost (not resident, not cached)");
  return SNAP_OK;
}

}  // extern "C"

// restore_job's cache seeding for a co-resident rank (ckpt.cpp:526-528): the
// rank's recorded digests become `dig`, and every chunk whose digest the chunk
// cache does not hold yet is copied in from image + src_off (device image,
// host offsets, one per chunk of the rank's splice grid).
int splice_seed(snap_ctx* ctx, int rank, const uint8_t* image, const uint64_t* src_off,
                const uint64_t* dig) {
  SpliceState* S = ctx->splice;
  if (!S || !S->ranks.count(rank)) return fail(ctx, SNAP_EINVAL, "splice: unknown rank");
  RankGrid& R = S->ranks[rank];
  if (S->cursor + R.bytes > S->cap)
    return fail(ctx, SNAP_ENOMEM, "splice: chunk cache full (" + std::to_string(S->cursor) +
                                      " of " + std::to_string(S->cap) + " bytes used)");
  CK(cudaSetDevice(ctx->device));
  TableDev cache{P<unsigned long long>(S->ck), P<unsigned long long>(S->cv), S->cmask};
  uint64_t* so;
  RC(ensure(ctx, S->seed_off, R.nchunks, &so));
  if (R.nchunks) {
    CK(cudaMemcpyAsync(P<uint64_t>(R.d_rec), dig, R.nchunks * 8, cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(so, src_off, R.nchunks * 8, cudaMemcpyHostToDevice, ctx->stream));
  }
  RC(select_with_known(ctx, P<uint64_t>(R.d_rec), P<uint32_t>(R.d_lens), R.nchunks, cache,
                       S->entries > 0));
  ctx->selected = false;
  CKL(snap::launch_gather_from(image, so, P<uint32_t>(R.d_lens), P<uint32_t>(ctx->sel_list),
                               P<uint64_t>(ctx->totals), P<uint64_t>(ctx->offsets),
                               P<uint8_t>(S->cache) + S->cursor, R.nchunks, ctx->stream));
  CKL(snap::launch_cache_insert(cache, P<uint64_t>(R.d_rec), P<uint32_t>(ctx->sel_list),
                                P<uint64_t>(ctx->totals), P<uint64_t>(ctx->offsets), S->cursor,
                                R.nchunks, ctx->stream));
  uint64_t tot[2] = {0, 0};
  CK(cudaMemcpyAsync(tot, ctx->totals.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  S->cursor += tot[1];
  S->entries += tot[0];
  R.recorded = true;
  return SNAP_OK;
}

extern "C" {

int snap_splice_recorded(snap_ctx* ctx, int rank, uint64_t* digests, uint64_t* n) {
  if (!ctx || !ctx->splice || !ctx->splice->ranks.count(rank)) return SNAP_EINVAL;
  RankGrid& R = ctx->splice->ranks[rank];
  if (n) *n = R.nchunks;
  if (digests && R.recorded && R.nchunks) {
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpyAsync(digests, R.d_rec.p, R.nchunks * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return R.recorded ? SNAP_OK : fail(ctx, SNAP_EINVAL, "rank has no recorded content yet");
}

}  // extern "C"
