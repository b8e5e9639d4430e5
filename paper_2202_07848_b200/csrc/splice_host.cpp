// splice_host.cpp — replica splicing context switch (GpuLedger::plan_switch /
// execute_switch, splice.cpp:167-306, driven by JobRuntime::switch_to,
// job.cpp:146-198), B200-native:
//  * the reference's host cache (std::map<digest, words>, splice.hpp:128) is a
//    digest-indexed CHUNK cache in spare HBM (180 GB per GPU holds several
//    replicas' state), so swap-out/in are D2D copies at HBM speed instead of
//    PCIe transfers, and dedup is per 64 KiB chunk instead of per buffer;
//  * the cache is a fixed array of chunk-sized slots with a device free stack
//    and a digest -> slot index; when a swap-out could run out of slots, the
//    chunks no rank records any more are reclaimed (the reference's map only
//    grows, which a fixed HBM region cannot afford over many mini-batches);
//  * swap-out = K1 hash of the outgoing rank's live, non-pending buffers +
//    K2 selection against the cache index + slot assignment + K3 gather of
//    the new chunks;
//  * swap-in = one pass over the incoming rank's chunks: resident when the
//    fresh digest of the same address range equals the incoming rank's
//    recorded digest (the stale-digest defect of SURVEY App. A-1 is fixed by
//    construction: the comparison uses the digests just computed), else a
//    copy from the cache by digest; a missing digest is a SimFault;
//  * collective results for inactive ranks are queued and installed at their
//    next switch-in (JobRuntime::on_coll_complete / switch_to, job.cpp:164-171,
//    206-222, ProxyServer::install_queue, proxy.hpp:75-79).
// One host sync per switch (the switch report of job.cpp:181-195).
#include <memory>

#include "ctx.h"

struct RankGrid {
  std::vector<snap_buf> bufs;
  std::vector<uint64_t> cstart;
  std::vector<uint32_t> lens;
  std::vector<uint64_t> chunk_addr;
  uint64_t nchunks = 0, bytes = 0;
  uint32_t chunk_bytes = 0;
  DevMem d_addr, d_bytes, d_cstart, d_lens, d_rec, d_tmaps, d_chunk_buf, d_chunk_addr;
  GridDev grid;
  bool recorded = false;
};

// A collective result kept for the ranks that install it later
// (DeferredInstall::words, proxy.hpp:75-78): one device copy shared by every
// queued install of the same call.
struct ResultSlab {
  DevMem mem;
  ~ResultSlab() { release(mem); }
};
struct Install {
  uint64_t dst = 0, bytes = 0;
  std::shared_ptr<ResultSlab> src;
};

struct SpliceState {
  uint64_t slot_bytes = 65536, nslots = 0, free_n = 0, live_bytes = 0, entries = 0;
  uint32_t slot_shift = 16;
  uint64_t gc_runs = 0, gc_freed_bytes = 0;
  DevMem cache, ck, cv, ck2, cv2, lk, lv, free_stack, slot_len, list_off, counters, seed_off;
  DevMem inst_ptrs;  // device arrays of the install copies
  // swap-in counters (zero between switches) and their mapped host report:
  // [swap-in bytes, resident bytes, lost, selected chunks, selected bytes]
  DevMem sin_cnt;
  unsigned long long* h_rep = nullptr;
  unsigned long long* d_rep = nullptr;
  uint64_t cmask = 0, lmask = 0;
  std::map<int, RankGrid> ranks;
  std::map<std::pair<int, int>, DevMem> match;
  std::map<int, std::vector<Install>> queue;
  int active = -1;
};

void splice_release(snap_ctx* ctx) {
  SpliceState* S = ctx->splice;
  if (!S) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto& [r, g] : S->ranks)
    for (DevMem* m : {&g.d_addr, &g.d_bytes, &g.d_cstart, &g.d_lens, &g.d_rec, &g.d_tmaps,
                      &g.d_chunk_buf, &g.d_chunk_addr})
      release(*m);
  for (auto& [k, m] : S->match) release(m);
  for (DevMem* m : {&S->cache, &S->ck, &S->cv, &S->ck2, &S->cv2, &S->lk, &S->lv, &S->free_stack,
                    &S->slot_len, &S->list_off, &S->counters, &S->seed_off, &S->inst_ptrs,
                    &S->sin_cnt})
    release(*m);
  if (S->h_rep) cudaFreeHost(S->h_rep);
  delete S;
  ctx->splice = nullptr;
}

namespace {

TableDev cache_index(SpliceState* S) {
  return TableDev{P<unsigned long long>(S->ck), P<unsigned long long>(S->cv), S->cmask};
}

// Reclaims the slots of cached chunks that no rank records any more: live set
// = every recorded rank's digest vector (the outgoing rank's already
// refreshed), index rebuilt with the live entries, dead slots pushed back.
int cache_gc(snap_ctx* ctx) {
  SpliceState* S = ctx->splice;
  uint64_t nrec = 0;
  for (auto& [r, g] : S->ranks)
    if (g.recorded) nrec += g.nchunks;
  const uint64_t lcap = table_cap(std::max<uint64_t>(nrec, 1));
  unsigned long long *lk, *lv, *k2, *v2, *cnt;
  RC(ensure(ctx, S->lk, lcap + 1, &lk));
  RC(ensure(ctx, S->lv, lcap + 1, &lv));
  RC(ensure(ctx, S->ck2, S->cmask + 2, &k2));
  RC(ensure(ctx, S->cv2, S->cmask + 2, &v2));
  RC(ensure(ctx, S->counters, 4, &cnt));
  TableDev live{lk, lv, lcap - 1};
  CKL(snap::launch_table_clear(live, ctx->stream));
  for (auto& [r, g] : S->ranks)
    if (g.recorded) CKL(snap::launch_table_insert_min(live, P<uint64_t>(g.d_rec), g.nchunks, 0, ctx->stream));
  TableDev fresh{k2, v2, S->cmask};
  CKL(snap::launch_table_clear(fresh, ctx->stream));
  CKL(snap::launch_cache_gc(cache_index(S), live, fresh, P<uint32_t>(S->free_stack), S->free_n,
                            P<uint32_t>(S->slot_len), cnt, ctx->stream));
  unsigned long long c[3] = {0, 0, 0};
  CK(cudaMemcpyAsync(c, cnt, 24, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  std::swap(S->ck, S->ck2);
  std::swap(S->cv, S->cv2);
  S->free_n += c[0];
  S->live_bytes -= c[1];
  S->entries = c[2];
  S->gc_runs += 1;
  S->gc_freed_bytes += c[1];
  return SNAP_OK;
}

// Stores the chunks the last selection over `dig` picked (ctx->sel_list /
// ctx->totals) into free cache slots: from the arena grid `from` (swap-out) or
// from image + src_off (seeding). When the worst case (every chunk new) does
// not fit the free slots, the actual count is read back (one sync) and the
// cache is reclaimed only if the new chunks really do not fit. Reclaiming
// after the selection is safe: every digest the selection just looked up is
// recorded by the rank being stored, so none of them is dead.
int cache_put(snap_ctx* ctx, const uint64_t* dig, const uint32_t* lens, uint64_t n,
              const GridDev* from, const uint8_t* image, const uint64_t* src_off) {
  SpliceState* S = ctx->splice;
  uint64_t tot[2] = {0, 0};
  if (S->free_n < n) {
    CK(cudaMemcpyAsync(tot, ctx->totals.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (tot[0] > S->free_n) RC(cache_gc(ctx));
    if (tot[0] > S->free_n)
      return fail(ctx, SNAP_ENOMEM, "splice: chunk cache full (" + std::to_string(S->nslots - S->free_n) +
                                        " of " + std::to_string(S->nslots) + " slots hold chunks "
                                        "recorded by some rank; " + std::to_string(tot[0]) +
                                        " new chunks)");
  }
  uint64_t* loff;
  RC(ensure(ctx, S->list_off, std::max<uint64_t>(n, 1), &loff));
  CKL(snap::launch_cache_assign(cache_index(S), dig, P<uint32_t>(ctx->sel_list),
                                P<uint64_t>(ctx->totals), lens, P<uint32_t>(S->free_stack),
                                S->free_n, S->slot_shift, loff, P<uint32_t>(S->slot_len), n,
                                ctx->stream));
  if (from) {
    CKL(snap::launch_gather(ctx->arena, *from, lens, P<uint32_t>(ctx->sel_list),
                            P<uint64_t>(ctx->totals), loff, true, nullptr, nullptr,
                            P<uint8_t>(S->cache), std::min(n, S->free_n), ctx->stream));
  } else {
    CKL(snap::launch_gather_from(image, src_off, lens, P<uint32_t>(ctx->sel_list),
                                 P<uint64_t>(ctx->totals), loff, P<uint8_t>(S->cache),
                                 std::min(n, S->free_n), ctx->stream, true));
  }
  return SNAP_OK;
}

// Applies the rank's queued result installs (switch_to, job.cpp:164-171):
// one kernel for all of them; returns their bytes.
int apply_installs(snap_ctx* ctx, int rank, uint64_t* bytes_out) {
  SpliceState* S = ctx->splice;
  *bytes_out = 0;
  auto it = S->queue.find(rank);
  if (it == S->queue.end() || it->second.empty()) return SNAP_OK;
  const auto& q = it->second;
  const uint32_t nr = uint32_t(q.size());
  std::vector<uint64_t> host(3 * nr);
  uint64_t mx = 0;
  for (uint32_t i = 0; i < nr; ++i) {
    host[i] = reinterpret_cast<uint64_t>(ctx->arena + q[i].dst);
    host[nr + i] = reinterpret_cast<uint64_t>(q[i].src->mem.p);
    host[2 * nr + i] = q[i].bytes;
    mx = std::max(mx, q[i].bytes);
    *bytes_out += q[i].bytes;
  }
  uint64_t* d;
  RC(ensure(ctx, S->inst_ptrs, 3 * nr, &d));
  CK(cudaMemcpyAsync(d, host.data(), 3 * nr * 8, cudaMemcpyHostToDevice, ctx->stream));
  CKL(snap::launch_copy_ranges(reinterpret_cast<uint8_t* const*>(d),
                               reinterpret_cast<const uint8_t* const*>(d + nr), d + 2 * nr, nr, mx,
                               ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // host array + result slabs die here
  S->queue.erase(it);
  return SNAP_OK;
}

}  // namespace

extern "C" {

int snap_splice_init_slots(snap_ctx* ctx, uint64_t cache_bytes, uint32_t slot_bytes) {
  if (!ctx || cache_bytes == 0 || !pow2(slot_bytes) || slot_bytes < 256)
    return fail(ctx, SNAP_EINVAL, "splice_init: cache_bytes > 0, slot_bytes a power of two >= 256");
  CK(cudaSetDevice(ctx->device));
  splice_release(ctx);
  ctx->splice = new SpliceState();
  SpliceState* S = ctx->splice;
  S->slot_bytes = slot_bytes;
  S->slot_shift = log2u(slot_bytes);
  S->nslots = std::max<uint64_t>(cache_bytes / slot_bytes, 1);
  if (S->nslots >= (1ull << 32)) return fail(ctx, SNAP_EINVAL, "splice_init: too many slots");
  uint8_t* c;
  RC(ensure(ctx, S->cache, S->nslots * slot_bytes, &c));
  // index capacity >= 2 x slots: an index of cached chunks never fills
  const uint64_t tcap = table_cap(S->nslots);
  unsigned long long *k, *v, *cnt;
  RC(ensure(ctx, S->ck, tcap + 1, &k));
  RC(ensure(ctx, S->cv, tcap + 1, &v));
  RC(ensure(ctx, S->counters, 4, &cnt));
  unsigned long long* sin;
  RC(ensure(ctx, S->sin_cnt, 4, &sin));
  CK(cudaMemsetAsync(sin, 0, 32, ctx->stream));
  {
    void* hp = nullptr;
    CK(cudaHostAlloc(&hp, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    S->h_rep = static_cast<unsigned long long*>(hp);
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&S->d_rep), hp, 0));
  }
  S->cmask = tcap - 1;
  CKL(snap::launch_table_clear(TableDev{k, v, S->cmask}, ctx->stream));
  // the reclamation's second index, allocated now: no cudaMalloc inside a switch
  unsigned long long *k2, *v2;
  RC(ensure(ctx, S->ck2, tcap + 1, &k2));
  RC(ensure(ctx, S->cv2, tcap + 1, &v2));
  uint32_t *fs, *sl;
  RC(ensure(ctx, S->free_stack, S->nslots, &fs));
  RC(ensure(ctx, S->slot_len, S->nslots, &sl));
  std::vector<uint32_t> init(S->nslots);
  for (uint64_t j = 0; j < S->nslots; ++j) init[j] = uint32_t(S->nslots - 1 - j);  // slot 0 on top
  CK(cudaMemcpyAsync(fs, init.data(), S->nslots * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  S->free_n = S->nslots;
  return SNAP_OK;
}

int snap_splice_init(snap_ctx* ctx, uint64_t cache_bytes) {
  return snap_splice_init_slots(ctx, cache_bytes, 65536);
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
  SpliceState* S = ctx->splice;
  if (g.chunk_bytes > S->slot_bytes)
    return fail(ctx, SNAP_EINVAL, "splice: chunk_bytes larger than the cache slot");
  CK(cudaSetDevice(ctx->device));
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
  R.chunk_bytes = g.chunk_bytes;
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
  if (R.nchunks >= snap::kMaxScanEntries)
    return fail(ctx, SNAP_EINVAL, "splice: a rank holds at most 2^26 - 1 chunks");
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
  std::vector<uint32_t> cbuf;
  std::vector<uint64_t> caddr;
  const uint32_t* dcb = nullptr;
  const uint64_t* dca = nullptr;
  RC(upload_chunk_buf(ctx, R.d_chunk_buf, R.d_chunk_addr, R.cstart, addr.data(),
                      log2u(g.chunk_bytes), cbuf, caddr, &dcb, &dca));
  CK(cudaStreamSynchronize(ctx->stream));
  R.grid = GridDev{da, db, dc, uint32_t(nb), R.nchunks, log2u(g.page_bytes), log2u(g.chunk_bytes),
                   dcb, dca, dca ? dl : nullptr};
  build_tmaps(ctx, R.d_tmaps, addr.data(), bytes.data(), uint32_t(nb), R.grid);
  R.recorded = false;
  // the reclamation's live-digest table covers every rank's chunks: sized here, not in a switch
  uint64_t total = 0;
  for (auto& [q, gq] : S->ranks) total += gq.nchunks;
  const uint64_t lcap = table_cap(std::max<uint64_t>(total, 1));
  unsigned long long *lk, *lv;
  RC(ensure(ctx, S->lk, lcap + 1, &lk));
  RC(ensure(ctx, S->lv, lcap + 1, &lv));
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
  snap_switch_stats out{};
  RankGrid* F = from >= 0 ? &S->ranks[from] : nullptr;
  RankGrid* T = to >= 0 ? &S->ranks[to] : nullptr;
  // SNAP_PROF_SWITCH: the switch's GPU span, first launch to the report kernel
  auto* span = new ProfScope(ctx, kProfSwitch);
  struct SpanEnd {
    ProfScope*& p;
    ~SpanEnd() { delete p; }
  } span_end{span};
  if (F) {
    // swap-out: refresh digests (K1), select against the cache (K2), slots +
    // gather (K3); reclaim first when the new chunks might not fit
    CKL(snap::launch_hash(ctx->arena, F->grid, P<uint64_t>(F->d_rec), nullptr, nullptr,
                          ctx->stream));
    F->recorded = true;
    RC(select_with_known(ctx, P<uint64_t>(F->d_rec), P<uint32_t>(F->d_lens), F->nchunks,
                         cache_index(S), S->entries > 0));
    ctx->selected = false;  // the ctx selection vectors now hold this plan
    RC(cache_put(ctx, P<uint64_t>(F->d_rec), P<uint32_t>(F->d_lens), F->nchunks, &F->grid,
                 nullptr, nullptr));
    out.hashed_bytes = F->bytes;
  }
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
                               match, F ? P<uint64_t>(F->d_rec) : nullptr, cache_index(S),
                               P<uint8_t>(S->cache), S->slot_shift,
                               P<unsigned long long>(S->sin_cnt), ctx->stream));
  }
  CKL(snap::launch_splice_report(P<unsigned long long>(S->sin_cnt),
                                 F ? P<uint64_t>(ctx->totals) : nullptr, S->d_rep, ctx->stream));
  delete span;  // end event before the host waits
  span = nullptr;
  CK(cudaStreamSynchronize(ctx->stream));
  const volatile unsigned long long* rep = S->h_rep;
  const unsigned long long cnt[3] = {rep[0], rep[1], rep[2]};
  const uint64_t tot[2] = {rep[3], rep[4]};
  S->free_n -= tot[0];
  S->live_bytes += tot[1];
  S->entries += tot[0];
  S->active = to;
  // deferred collective results of the incoming rank (after the swap-ins,
  // like the reference: execute_switch, then install_result per queued entry)
  uint64_t inst = 0;
  if (to >= 0) RC(apply_installs(ctx, to, &inst));
  out.swap_out_bytes = tot[1];
  out.swap_in_bytes = cnt[0];
  out.resident_bytes = cnt[1];
  out.cache_bytes = S->live_bytes;
  out.install_bytes = inst;
  out.cache_free_bytes = S->free_n * S->slot_bytes;
  out.reclaimed_bytes = S->gc_freed_bytes;
  if (st) *st = out;
  if (cnt[2])
    return fail(ctx, SNAP_EFAULT, "splice: content for " + std::to_string(cnt[2]) +
                                      " chunk digest(s) lost (not resident, not cached)");
  return SNAP_OK;
}

// JobRuntime::on_coll_complete (job.cpp:206-222): the result at arena
// [src_addr, +bytes) goes into rank ranks[i]'s buffer at dst_addrs[i]. The
// active rank (and every rank of a ctx without splicing) gets it now; the
// others queue it (one library copy of the result shared by the queue,
// DeferredInstall::words, proxy.hpp:75-78) until their next switch-in.
int snap_splice_install(snap_ctx* ctx, const int* ranks, const uint64_t* dst_addrs, uint32_t n,
                        uint64_t src_addr, uint64_t bytes) {
  if (!ctx || (n && (!ranks || !dst_addrs)) || bytes % 16 || src_addr % 16)
    return fail(ctx, SNAP_EINVAL, "install: 16-byte aligned ranges");
  RC(check_range(ctx, src_addr, bytes));
  for (uint32_t i = 0; i < n; ++i) {
    RC(check_range(ctx, dst_addrs[i], bytes));
    if (dst_addrs[i] % 16) return fail(ctx, SNAP_EINVAL, "install: 16-byte aligned ranges");
  }
  CK(cudaSetDevice(ctx->device));
  SpliceState* S = ctx->splice;
  std::vector<uint64_t> now;
  std::shared_ptr<ResultSlab> slab;
  for (uint32_t i = 0; i < n; ++i) {
    const bool active = !S || ranks[i] < 0 || ranks[i] == S->active;
    if (active) {
      now.push_back(dst_addrs[i]);
      continue;
    }
    if (!slab) {
      slab = std::make_shared<ResultSlab>();
      uint8_t* p;
      RC(ensure(ctx, slab->mem, bytes, &p));
      now.push_back(~0ull);  // marker: copy the result into the slab
    }
    S->queue[ranks[i]].push_back(Install{dst_addrs[i], bytes, slab});
  }
  if (now.empty() || bytes == 0) return SNAP_OK;
  const uint32_t nr = uint32_t(now.size());
  std::vector<uint64_t> host(3 * nr);
  for (uint32_t i = 0; i < nr; ++i) {
    host[i] = now[i] == ~0ull ? reinterpret_cast<uint64_t>(slab->mem.p)
                              : reinterpret_cast<uint64_t>(ctx->arena + now[i]);
    host[nr + i] = reinterpret_cast<uint64_t>(ctx->arena + src_addr);
    host[2 * nr + i] = bytes;
  }
  struct Scratch {  // pointer arrays of a ctx without splicing, freed on every path
    DevMem m;
    ~Scratch() { release(m); }
  } tmp;
  uint64_t* d;
  RC(ensure(ctx, S ? S->inst_ptrs : tmp.m, 3 * nr, &d));
  CK(cudaMemcpyAsync(d, host.data(), 3 * nr * 8, cudaMemcpyHostToDevice, ctx->stream));
  CKL(snap::launch_copy_ranges(reinterpret_cast<uint8_t* const*>(d),
                               reinterpret_cast<const uint8_t* const*>(d + nr), d + 2 * nr, nr,
                               bytes, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

// Pending installs of a rank: count and bytes (the switch report's
// install_bytes before it happens).
int snap_splice_pending(snap_ctx* ctx, int rank, uint64_t* count, uint64_t* bytes) {
  if (!ctx || !ctx->splice) return SNAP_EINVAL;
  uint64_t c = 0, b = 0;
  auto it = ctx->splice->queue.find(rank);
  if (it != ctx->splice->queue.end())
    for (const Install& q : it->second) c += 1, b += q.bytes;
  if (count) *count = c;
  if (bytes) *bytes = b;
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
  CK(cudaSetDevice(ctx->device));
  uint64_t* so;
  RC(ensure(ctx, S->seed_off, R.nchunks, &so));
  if (R.nchunks) {
    CK(cudaMemcpyAsync(P<uint64_t>(R.d_rec), dig, R.nchunks * 8, cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(so, src_off, R.nchunks * 8, cudaMemcpyHostToDevice, ctx->stream));
  }
  R.recorded = true;  // its digests are live from now on
  RC(select_with_known(ctx, P<uint64_t>(R.d_rec), P<uint32_t>(R.d_lens), R.nchunks,
                       cache_index(S), S->entries > 0));
  ctx->selected = false;
  RC(cache_put(ctx, P<uint64_t>(R.d_rec), P<uint32_t>(R.d_lens), R.nchunks, nullptr, image, so));
  uint64_t tot[2] = {0, 0};
  CK(cudaMemcpyAsync(tot, ctx->totals.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  S->free_n -= tot[0];
  S->live_bytes += tot[1];
  S->entries += tot[0];
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
