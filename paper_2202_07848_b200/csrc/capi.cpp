// capi.cpp — the C ABI (include/snap.h): one snap_ctx per (job, GPU), the
// B200 analogue of proxy::ProxyServer (proxy.hpp:32-122) + vdev::Gpu memory
// (vdev.hpp:65-122). Host code only; every byte of device work is one of the
// sm_100a kernels in k_*.cu, issued on the ctx stream (NCCL collectives on the
// same stream for the cross-rank exchange).
#include <cstdlib>

#include "ctx.h"

void splice_release(snap_ctx* ctx);
void window_release(snap_ctx* ctx);

namespace {

int ensure_known(snap_ctx* ctx, uint64_t extra) {
  // grows (and rebuilds) the known-set table to keep load <= 1/2
  const uint64_t need = ctx->kn_count + extra;
  uint64_t* list;
  RC(ensure_keep(ctx, ctx->kn_list, need, ctx->kn_count * 8, &list));
  if (ctx->kn_mask && 2 * need <= ctx->kn_mask + 1) return SNAP_OK;
  const uint64_t cap = table_cap(need);
  unsigned long long *k, *v;
  RC(ensure(ctx, ctx->kn_keys, cap + 1, &k));
  RC(ensure(ctx, ctx->kn_vals, cap + 1, &v));
  ctx->kn_mask = cap - 1;
  TableDev t{k, v, ctx->kn_mask};
  CKL(snap::launch_table_clear(t, ctx->stream));
  CKL(snap::launch_table_insert_min(t, P<uint64_t>(ctx->kn_list), ctx->kn_count, 0, ctx->stream));
  return SNAP_OK;
}

int known_insert_dev(snap_ctx* ctx, const uint64_t* dev_digests, uint64_t n) {
  if (n == 0) return SNAP_OK;
  RC(ensure_known(ctx, n));
  uint64_t* list = P<uint64_t>(ctx->kn_list);
  CK(cudaMemcpyAsync(list + ctx->kn_count, dev_digests, n * 8, cudaMemcpyDeviceToDevice,
                     ctx->stream));
  TableDev t{P<unsigned long long>(ctx->kn_keys), P<unsigned long long>(ctx->kn_vals), ctx->kn_mask};
  CKL(snap::launch_table_insert_min(t, list + ctx->kn_count, n, 0, ctx->stream));
  ctx->kn_count += n;
  return SNAP_OK;
}

}  // namespace

// Dedup table + scan state for a selection over n entries: allocated, and
// cleared only when they are not known to be empty (the resolve pass of the
// previous selection leaves them empty).
int prepare_dedup(snap_ctx* ctx, uint64_t n, TableDev* out, uint64_t** slot, uint64_t** scan) {
  const uint64_t cap = table_cap(n);
  const uint64_t words = snap::scan_state_words(n) + 1;
  unsigned long long *k, *v;
  const void* k_old = ctx->dd_keys.p;
  const void* v_old = ctx->dd_vals.p;
  const void* s_old = ctx->scan.p;
  RC(ensure(ctx, ctx->dd_keys, cap + 1, &k));
  RC(ensure(ctx, ctx->dd_vals, cap + 1, &v));
  RC(ensure(ctx, ctx->dd_slot, n, slot));
  RC(ensure(ctx, ctx->scan, words, scan));
  if (k != k_old || v != v_old) ctx->dd_clean_mask = 0, ctx->dd_clean = false;
  if (*scan != s_old) ctx->scan_clean_words = 0;
  ctx->dd_mask = cap - 1;
  *out = TableDev{k, v, ctx->dd_mask};
  if (!ctx->dd_clean || ctx->dd_mask > ctx->dd_clean_mask) {
    CKL(snap::launch_table_clear(*out, ctx->stream));
    ctx->dd_clean_mask = ctx->dd_mask;
  }
  if (!ctx->dd_clean || words > ctx->scan_clean_words) {
    CK(cudaMemsetAsync(*scan, 0, words * 8, ctx->stream));
    ctx->scan_clean_words = words;
  }
  ctx->dd_clean = false;  // about to be filled
  return SNAP_OK;
}

// Selection over a canonical vector against an explicit known table (the
// splice chunk cache uses its own index as the known set). `inserted`: the K2
// insert already ran inside K1 (hash_fused) into the prepared table.
int select_with_known(snap_ctx* ctx, const uint64_t* dig, const uint32_t* lens, uint64_t n,
                      TableDev kn, bool use_known, bool inserted, uint64_t* spec_next,
                      const uint64_t* fix_spec, uint8_t* fix_staging) {
  if (n >= snap::kMaxScanEntries)
    return fail(ctx, SNAP_EINVAL, "select: a selection covers at most 2^26 - 1 chunks");
  uint64_t *slot, *scan, *owner, *offsets, *totals;
  uint8_t* sel;
  uint32_t* list;
  TableDev dd;
  if (inserted) {
    dd = TableDev{P<unsigned long long>(ctx->dd_keys), P<unsigned long long>(ctx->dd_vals),
                  ctx->dd_mask};
    slot = P<uint64_t>(ctx->dd_slot);
    scan = P<uint64_t>(ctx->scan);
  } else {
    RC(prepare_dedup(ctx, n, &dd, &slot, &scan));
  }
  RC(ensure(ctx, ctx->sel, n, &sel));
  RC(ensure(ctx, ctx->owner, n, &owner));
  RC(ensure(ctx, ctx->offsets, n, &offsets));
  RC(ensure(ctx, ctx->sel_list, n, &list));
  RC(ensure(ctx, ctx->totals, 4, &totals));
  static const bool small_off = [] {
    const char* e = std::getenv("SNAP_SELECT_SMALL");
    return e && e[0] == '0';
  }();
  static const bool cluster_off = [] {
    const char* e = std::getenv("SNAP_SELECT_CLUSTER");
    return e && e[0] == '0';
  }();
  if (!inserted && !small_off && !cluster_off && snap::select_cluster_ok(n)) {
    // the table and scan state prepare_dedup guarantees clean stay untouched
    CKL(snap::launch_select_cluster(kn, use_known, dig, lens, n, sel, owner, offsets, list,
                                    totals, spec_next, ctx->stream, fix_spec, ctx->arena,
                                    &ctx->grid, fix_staging));
    ctx->dd_clean = true;
    ctx->sel_n = n;
    ctx->global_offsets_pending = false;
    return SNAP_OK;
  }
  if (!inserted && !small_off && snap::select_small_ok(n)) {
    // scratch: the (zero) scan state, at least 9 words (prepare_dedup zeroed it)
    CKL(snap::launch_select_small(dd, kn, use_known, dig, lens, n, sel, owner, offsets, list,
                                  totals, spec_next, ctx->stream, scan, fix_spec, ctx->arena,
                                  &ctx->grid, fix_staging));
    ctx->dd_clean = true;
    ctx->sel_n = n;
    ctx->global_offsets_pending = false;
    return SNAP_OK;
  }
  if (!inserted) CKL(snap::launch_dedup_insert(dd, kn, use_known, dig, lens, n, slot, ctx->stream));
  CKL(snap::launch_select(dd, slot, lens, n, scan, sel, owner, offsets, list, totals, spec_next,
                          ctx->stream, fix_spec, ctx->arena, &ctx->grid, fix_staging));
  const uint64_t words = snap::scan_state_words(n) + 1;
  CKL(snap::launch_resolve_dups(sel, owner, offsets, n, dd, scan, words, ctx->stream));
  ctx->dd_clean = true;
  ctx->scan_clean_words = std::max(ctx->scan_clean_words, words);
  ctx->sel_n = n;
  ctx->global_offsets_pending = false;
  return SNAP_OK;
}

namespace {

// Selection over a canonical vector (local grid or allgathered global one).
int select_impl(snap_ctx* ctx, const uint64_t* dig, const uint32_t* lens, uint64_t n,
                bool inserted = false, uint64_t* spec_next = nullptr,
                const uint64_t* fix_spec = nullptr, uint8_t* fix_staging = nullptr) {
  TableDev kn{P<unsigned long long>(ctx->kn_keys), P<unsigned long long>(ctx->kn_vals), ctx->kn_mask};
  RC(select_with_known(ctx, dig, lens, n, kn, ctx->kn_count > 0, inserted, spec_next, fix_spec,
                       fix_staging));
  ctx->selected = true;
  return SNAP_OK;
}

// Exchange window layout (see ctx.h): flag lines, then two gathered vectors.
uint64_t xflag_bytes(const snap_ctx* ctx) { return uint64_t(ctx->nranks) * 128; }
uint64_t* gdig_region(const snap_ctx* ctx, uint64_t epoch) {
  return reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(ctx->d_gdig.p) + xflag_bytes(ctx)) +
         (epoch & 1) * uint64_t(ctx->nranks) * ctx->maxn;
}

void close_peer_staging(snap_ctx* ctx) {
  for (size_t r = 0; r < ctx->peer_staging.size(); ++r)
    if (int(r) != ctx->rank && r < ctx->peer_opened.size())
      ipc_close(ctx->peer_staging[r], ctx->peer_opened[r]);
  ctx->peer_staging.clear();
  ctx->peer_opened.clear();
}

void close_peer_windows(snap_ctx* ctx) {
  for (size_t q = 0; q < ctx->xpeer.size(); ++q)
    if (int(q) != ctx->rank && ctx->xpeer[q]) cudaIpcCloseMemHandle(ctx->xpeer[q]);
  ctx->xpeer.clear();
  ctx->xwin_ready = false;
  ctx->k1_fanout = false;
}

// (Re)allocates this rank's exchange window for the grid's maxn and maps every
// peer's window; collective (NCCL). Mode agreement: if any rank cannot map a
// peer, every rank keeps the NCCL allgather (xwin_ready stays false).
// Opt-in (SNAP_FUSED_EXCHANGE=1, same on every rank): measured on B200 at N = 2
// and 4, the NVLink stores + system fence add as much to K1 as the barrier saves
// over the NCCL allgather — the exchange step's cost is inter-GPU skew of K1
// completion, which any barrier absorbs (profiles/r01_summary.md).
int setup_exchange_window(snap_ctx* ctx) {
  const int R = ctx->nranks;
  close_peer_windows(ctx);
  static const bool fused = [] {
    const char* e = std::getenv("SNAP_FUSED_EXCHANGE");
    return e && e[0] == '1';
  }();
  const uint64_t need = xflag_bytes(ctx) + 2 * uint64_t(R) * ctx->maxn * 8;
  if (!fused || !ctx->comm) {  // allgather into the (unmapped) window
    if (need > ctx->d_gdig.cap) {
      release(ctx->d_gdig);
      uint8_t* w;
      RC(ensure(ctx, ctx->d_gdig, need, &w));
    }
    return SNAP_OK;
  }
  uint8_t* xh;
  RC(ensure(ctx, ctx->d_xh, 64 * uint64_t(R) + 16, &xh));
  int32_t* word = reinterpret_cast<int32_t*>(xh + 64 * uint64_t(R));
  auto agree = [&](int32_t v, CommOp op, int32_t* out) -> int {
    CK(cudaMemcpyAsync(word, &v, 4, cudaMemcpyHostToDevice, ctx->stream));
    RC(comm_allreduce(ctx, word, word, 1, kCommI32, op));
    CK(cudaMemcpyAsync(out, word, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return SNAP_OK;
  };
  // every importer has closed its mapping of the old windows once this
  // collective returns, so a window may be freed and reallocated after it
  int32_t any_grow = 0;
  RC(agree(need > ctx->d_gdig.cap ? 1 : 0, kCommMax, &any_grow));
  if (need > ctx->d_gdig.cap) {
    release(ctx->d_gdig);
    uint8_t* w;
    RC(ensure(ctx, ctx->d_gdig, need, &w));
  }
  CK(cudaMemsetAsync(ctx->d_gdig.p, 0, xflag_bytes(ctx), ctx->stream));  // epochs restart
  cudaIpcMemHandle_t h;
  const bool ipc = cudaIpcGetMemHandle(&h, ctx->d_gdig.p) == cudaSuccess;
  if (!ipc) {
    cudaGetLastError();
    std::memset(&h, 0, sizeof h);
  }
  CK(cudaMemcpyAsync(xh + 64 * ctx->rank, &h, 64, cudaMemcpyHostToDevice, ctx->stream));
  RC(comm_allgather(ctx, xh + 64 * ctx->rank, xh, 64, kCommU8));
  std::vector<uint8_t> all(64 * size_t(R));
  CK(cudaMemcpyAsync(all.data(), xh, all.size(), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->xpeer.assign(R, nullptr);
  bool ok = true;
  static const uint8_t zero[64] = {};
  for (int q = 0; q < R; ++q) {
    if (q == ctx->rank) {
      ctx->xpeer[q] = ctx->d_gdig.p;
      continue;
    }
    if (std::memcmp(all.data() + 64 * q, zero, 64) == 0) {
      ok = false;
      continue;
    }
    cudaIpcMemHandle_t ph;
    std::memcpy(&ph, all.data() + 64 * q, 64);
    if (cudaIpcOpenMemHandle(&ctx->xpeer[q], ph, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ctx->xpeer[q] = nullptr;
      ok = false;
    }
  }
  int32_t all_ok = 0;
  RC(agree(ok ? 1 : 0, kCommMin, &all_ok));
  if (!all_ok) {
    close_peer_windows(ctx);
    return SNAP_OK;
  }
  std::vector<uint64_t*> xd(R), xf(R);
  for (int q = 0; q < R; ++q) {
    xf[q] = static_cast<uint64_t*>(ctx->xpeer[q]);
    xd[q] = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(ctx->xpeer[q]) + xflag_bytes(ctx));
  }
  uint64_t **dxd, **dxf;
  RC(ensure(ctx, ctx->d_xdig, R, &dxd));
  RC(ensure(ctx, ctx->d_xflag, R, &dxf));
  CK(cudaMemcpyAsync(dxd, xd.data(), 8 * R, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dxf, xf.data(), 8 * R, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->xepoch = 0;
  ctx->xwin_ready = true;
  return SNAP_OK;
}

// K1 launches of a multi-rank ctx store their digests into every rank's
// gathered vector of the coming exchange (epoch xepoch + 1) when the windows
// are mapped; the exchange then reduces to the barrier.
void k1_fanout(snap_ctx* ctx, GridDev& g) {
  if (!ctx->attached() || !ctx->xwin_ready) return;
  g.xdig = P<uint64_t*>(ctx->d_xdig);
  g.xn = uint32_t(ctx->nranks);
  g.xoff = ((ctx->xepoch + 1) & 1) * uint64_t(ctx->nranks) * ctx->maxn +
           uint64_t(ctx->rank) * ctx->maxn;
  ctx->k1_fanout = true;
}

}  // namespace

// Per-grid part of the exchange, collective: every rank's chunk count (-> maxn)
// and chunk lengths are all-gathered and the exchange windows set up. Issued by
// snap_comm_init and by snap_set_buffers / snap_load with a communicator
// attached (those calls are collective then), never conditionally inside a
// snapshot: every rank's snapshot issues the same NCCL sequence no matter
// which rank re-installed its grid.
int grid_exchange(snap_ctx* ctx) {
  const int R = ctx->nranks;
  uint64_t* dc;
  RC(ensure(ctx, ctx->d_counts, 2 * R, &dc));
  CK(cudaMemcpyAsync(dc + R, &ctx->nchunks, 8, cudaMemcpyHostToDevice, ctx->stream));
  RC(comm_allgather(ctx, dc + R, dc, 1, kCommU64));
  ctx->counts.assign(R, 0);
  CK(cudaMemcpyAsync(ctx->counts.data(), dc, 8 * R, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->maxn = *std::max_element(ctx->counts.begin(), ctx->counts.end());
  if (uint64_t(R) * ctx->maxn >= snap::kMaxScanEntries)
    return fail(ctx, SNAP_EINVAL, "exchange: nranks x max chunks per rank exceeds 2^26 entries");
  ctx->k1_fanout = false;  // K1 ran before the windows existed for this grid
  RC(setup_exchange_window(ctx));
  const uint64_t maxn = ctx->maxn, n = uint64_t(R) * maxn;
  uint32_t* glens;
  RC(ensure(ctx, ctx->d_glens, n + maxn, &glens));
  uint32_t* slen = glens + n;
  CK(cudaMemsetAsync(slen, 0, maxn * 4, ctx->stream));
  if (ctx->nchunks)
    CK(cudaMemcpyAsync(slen, P<uint32_t>(ctx->d_lens), ctx->nchunks * 4, cudaMemcpyDeviceToDevice,
                       ctx->stream));
  RC(comm_allgather(ctx, slen, glens, maxn, kCommU32));
  ctx->glens_valid = true;
  return SNAP_OK;
}

namespace {

// The exchange step: per-rank digest vectors gathered (rank-major, padded to
// the largest rank) — by K1's own NVLink stores + a peer barrier, or by an
// NCCL allgather. The only bytes that cross NVLink: 8 B per 64 KiB chunk.
int exchange_impl(snap_ctx* ctx) {
  const int R = ctx->nranks;
  if (!ctx->glens_valid)
    return fail(ctx, SNAP_EINTERNAL, "exchange: grid not exchanged (snap_set_buffers / "
                                     "snap_comm_init are collective with a communicator)");
  const uint64_t maxn = ctx->maxn, n = uint64_t(R) * maxn;
  const uint64_t epoch = ctx->xepoch + 1;
  uint64_t* gdig = gdig_region(ctx, epoch);
  if (ctx->k1_fanout) {
    CKL(snap::launch_peer_barrier(P<uint64_t*>(ctx->d_xflag), static_cast<uint64_t*>(ctx->d_gdig.p),
                                  uint32_t(ctx->rank), uint32_t(R), epoch, ctx->stream));
  } else {
    // the digest vector is sent in place: d_dig holds >= maxn entries, the
    // padding entries' values are ignored (their gathered lengths are 0)
    uint64_t* sdig;
    RC(ensure_keep(ctx, ctx->d_dig, maxn, ctx->nchunks * 8, &sdig));
    RC(comm_allgather(ctx, sdig, gdig, maxn, kCommU64));
  }
  ctx->k1_fanout = false;
  ctx->xepoch = epoch;
  (void)n;
  ctx->exchanged = true;
  return SNAP_OK;
}

// The multi-rank step's selection: owners (dedup over the gathered vectors),
// stripe writers and this rank's shard scan — all the compaction needs. The
// global image's staging offsets (read only by snap_get_selection) are left
// to global_offsets(), which scans the owners this step recorded.
int select_stripe_impl(snap_ctx* ctx) {
  const uint64_t maxn = ctx->maxn, n = uint64_t(ctx->nranks) * maxn;
  TableDev kn{P<unsigned long long>(ctx->kn_keys), P<unsigned long long>(ctx->kn_vals), ctx->kn_mask};
  TableDev dd;
  uint64_t *slot, *scan, *owner, *shard_off, *my_off, *my_tot, *scan2;
  uint8_t* sel;
  int32_t* writer;
  uint32_t* my_list;
  RC(prepare_dedup(ctx, n, &dd, &slot, &scan));
  RC(ensure(ctx, ctx->sel, n, &sel));
  RC(ensure(ctx, ctx->owner, n, &owner));
  RC(ensure(ctx, ctx->d_writer, n, &writer));
  RC(ensure(ctx, ctx->d_shard_off, n, &shard_off));
  RC(ensure(ctx, ctx->d_my_list, maxn, &my_list));
  RC(ensure(ctx, ctx->d_my_off, maxn, &my_off));
  RC(ensure(ctx, ctx->d_my_totals, 4, &my_tot));
  RC(ensure(ctx, ctx->scan2, snap::scan_state_words(n) + 1, &scan2));
  const uint64_t* gdig = gdig_region(ctx, ctx->xepoch);
  const uint32_t* glens = P<uint32_t>(ctx->d_glens);
  CKL(snap::launch_dedup_insert(dd, kn, ctx->kn_count > 0, gdig, glens, n, slot, ctx->stream));
  // snap_snapshot with a whole-grid staging image: the shard scan also does
  // the K3 fix-up and writes the next speculative layout
  snap::FixUp fix;
  if (ctx->fixup_request && ctx->spec_used && ctx->staging.cap >= ctx->grid_bytes) {
    fix.spec_cur = P<uint64_t>(ctx->d_spec[ctx->spec_cur]);
    RC(ensure(ctx, ctx->d_spec[1 - ctx->spec_cur], ctx->nchunks, &fix.spec_next));
    fix.nlocal = ctx->nchunks;
    fix.arena = ctx->arena;
    fix.grid = ctx->grid;
    fix.staging = static_cast<uint8_t*>(ctx->staging.p);
  }
  CKL(snap::launch_select_stripe(dd, slot, gdig, glens, ctx->nranks, maxn, ctx->rank, sel, owner,
                                 writer, scan2, shard_off, my_list, my_off, my_tot, ctx->stream,
                                 fix));
  ctx->fixup_done = fix.staging != nullptr;
  ctx->spec_next_done = fix.staging != nullptr;
  ctx->dd_clean = true;  // the shard scan emptied the table
  ctx->sel_n = n;
  ctx->selected = true;
  ctx->shard_offsets_all = false;
  ctx->global_offsets_pending = true;
  return SNAP_OK;
}

// Global staging offsets of the last multi-rank step, from its owners.
int global_offsets(snap_ctx* ctx) {
  if (!ctx->global_offsets_pending) return SNAP_OK;
  const uint64_t n = ctx->sel_n;
  const uint64_t words = snap::scan_state_words(n) + 1;
  uint64_t *scan, *offsets, *totals;
  uint32_t* list;
  const void* s_old = ctx->scan.p;
  RC(ensure(ctx, ctx->scan, words, &scan));
  if (scan != s_old) ctx->scan_clean_words = 0;
  if (words > ctx->scan_clean_words) CK(cudaMemsetAsync(scan, 0, words * 8, ctx->stream));
  RC(ensure(ctx, ctx->offsets, n, &offsets));
  RC(ensure(ctx, ctx->sel_list, n, &list));
  RC(ensure(ctx, ctx->totals, 4, &totals));
  CKL(snap::launch_select(TableDev{}, nullptr, P<uint32_t>(ctx->d_glens), n, scan,
                          P<uint8_t>(ctx->sel), P<uint64_t>(ctx->owner), offsets, list, totals,
                          nullptr, ctx->stream));
  CKL(snap::launch_resolve_dups(P<uint8_t>(ctx->sel), P<uint64_t>(ctx->owner), offsets, n,
                                TableDev{}, scan, words, ctx->stream));
  ctx->scan_clean_words = std::max(ctx->scan_clean_words, words);
  ctx->global_offsets_pending = false;
  return SNAP_OK;
}

// Speculative staging layout before any digest is known:
// single GPU: every chunk staged, canonical order (identity prefix);
// multi-rank: chunks of buffers hinted replicated are predicted striped
// (writer = local_index % nranks), others written by their own rank; shard
// order follows the predicted global index (first holder's rank, local index).
// Staging capacity: a whole image on one GPU (every chunk may be staged); for a
// multi-rank shard the predicted shard size + margin. keep = preserve the
// speculative bytes already written when growing.
int staging_reserve(snap_ctx* ctx, uint64_t bytes, bool keep, uint8_t** out) {
  bytes = std::min<uint64_t>(std::max<uint64_t>(bytes, 256), std::max<uint64_t>(ctx->grid_bytes, 256));
  if (bytes <= ctx->staging.cap) {
    *out = static_cast<uint8_t*>(ctx->staging.p);
    return SNAP_OK;
  }
  if (ctx->d2h) CK(cudaStreamSynchronize(ctx->d2h));  // in-flight D2H reads of the old image
  return ensure_keep(ctx, ctx->staging, bytes, keep ? ctx->staging.cap : 0, out);
}

// Staging capacity: the worst case (every chunk of this rank staged) unless the
// grid is huge (C5: 80 GB per GPU), where a multi-rank shard is sized to the
// predicted layout and grown on demand — at the price of one host sync per
// snapshot to learn the actual shard size (compact_impl).
constexpr uint64_t kFullStagingMax = 16ull << 30;
uint64_t staging_target(const snap_ctx* ctx) {
  if (!ctx->attached() || ctx->nranks == 1 || ctx->spec_bytes == 0 ||
      ctx->grid_bytes <= kFullStagingMax)
    return ctx->grid_bytes;
  return ctx->spec_bytes + ctx->spec_bytes / 16 + (64ull << 20);
}

bool replicated_hint(const snap_buf& b) {
  if (b.flags & SNAP_BUF_REPLICATED) return true;
  if (b.flags & SNAP_BUF_PRIVATE) return false;
  return b.cat == 0 || b.cat == 1;  // Param / OptState: identical across DP replicas
}

// SNAP_SPEC_STRIPE=N (measurement aid, single GPU): every snapshot predicts the
// layout rank 0 of an N-rank job stages, so K1's fused stores can be timed at
// the write fraction of an N-GPU run on one GPU (tools/stripe_emu.py)
int spec_stripe_emu() {
  static const int v = getenv("SNAP_SPEC_STRIPE") ? atoi(getenv("SNAP_SPEC_STRIPE")) : 0;
  return v;
}

int init_spec(snap_ctx* ctx) {
  const uint64_t n = ctx->nchunks;
  std::vector<uint64_t> spec(n, ~0ull);
  const int emu = spec_stripe_emu();
  if ((!ctx->attached() || ctx->nranks == 1) && emu > 1) {
    // measurement aid: predict the layout rank 0 of an emu-rank job stages
    // (private chunks + every emu-th replicated chunk); the fix-up copies the rest
    std::vector<uint8_t> rep(n, 0);
    for (size_t b = 0; b < ctx->bufs.size(); ++b)
      for (uint64_t g = ctx->h_cstart[b]; g < ctx->h_cstart[b + 1]; ++g)
        rep[g] = replicated_hint(ctx->bufs[b]);
    uint64_t off = 0;
    for (uint64_t g = 0; g < n; ++g)
      if (!rep[g] || g % uint64_t(emu) == 0) {
        spec[g] = off;
        off += ctx->h_lens[g];
      }
  } else if (!ctx->attached() || ctx->nranks == 1) {
    // one GPU: every chunk staged in canonical order, except (several ranks in
    // one buffer list, e.g. C2 held by one GPU) the chunks of a buffer hinted
    // replicated whose slot the lowest rank also holds with the same size —
    // predicted to be that rank's duplicates
    std::vector<uint8_t> dup(n, 0);
    if (!ctx->bufs.empty()) {
      uint32_t r0 = ctx->bufs[0].rank;
      for (const snap_buf& b : ctx->bufs) r0 = std::min(r0, b.rank);
      std::map<int32_t, uint64_t> first;  // slot -> bytes in the lowest rank
      for (const snap_buf& b : ctx->bufs)
        if (b.rank == r0) first[b.slot] = b.bytes;
      for (size_t b = 0; b < ctx->bufs.size(); ++b) {
        const snap_buf& x = ctx->bufs[b];
        auto it = first.find(x.slot);
        if (x.rank != r0 && replicated_hint(x) && it != first.end() && it->second == x.bytes)
          for (uint64_t g = ctx->h_cstart[b]; g < ctx->h_cstart[b + 1]; ++g) dup[g] = 1;
      }
    }
    uint64_t off = 0;
    for (uint64_t g = 0; g < n; ++g) {
      if (dup[g]) continue;
      spec[g] = off;
      off += ctx->h_lens[g];
    }
  } else {
    std::vector<uint8_t> rep(n, 0);
    for (size_t b = 0; b < ctx->bufs.size(); ++b)
      for (uint64_t g = ctx->h_cstart[b]; g < ctx->h_cstart[b + 1]; ++g)
        rep[g] = replicated_hint(ctx->bufs[b]);
    const uint64_t N = ctx->nranks, me = ctx->rank;
    uint64_t off = 0;
    auto take = [&](uint64_t g) {
      spec[g] = off;
      off += ctx->h_lens[g];
    };
    if (me == 0) {
      for (uint64_t g = 0; g < n; ++g)
        if (!rep[g] || g % N == 0) take(g);
    } else {
      for (uint64_t g = 0; g < n; ++g)
        if (rep[g] && g % N == me) take(g);
      for (uint64_t g = 0; g < n; ++g)
        if (!rep[g]) take(g);
    }
  }
  uint64_t* d;
  RC(ensure(ctx, ctx->d_spec[ctx->spec_cur], n, &d));
  CK(cudaMemcpyAsync(d, spec.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->spec_ready = true;
  uint64_t top = 0;
  for (uint64_t g = 0; g < n; ++g)
    if (spec[g] != ~0ull) top = std::max<uint64_t>(top, spec[g] + ctx->h_lens[g]);
  ctx->spec_bytes = top;
  ctx->h_spec = std::move(spec);
  ctx->h_spec_valid = true;
  return SNAP_OK;
}

// K1 with the fused speculative compaction (full snapshots); incremental
// snapshots (known set non-empty) hash only and gather the few dirty chunks.
// Chunks [c0, c1) only (c1 == 0: all), so the host-buffer path can hash each
// slab as soon as it lands.
int hash_fused(snap_ctx* ctx, uint64_t c0 = 0, uint64_t c1 = 0) {
  GridDev g = ctx->grid;
  g.c_begin = c0;
  g.c_end = c1;
  const bool spec = ctx->kn_count == 0;
  uint8_t* st = nullptr;
  const uint64_t* so = nullptr;
  if (spec) {
    if (!ctx->spec_ready || spec_stripe_emu() > 1) RC(init_spec(ctx));
    RC(staging_reserve(ctx, staging_target(ctx), true, &st));
    g.spec_bytes = ctx->spec_bytes;
    so = P<uint64_t>(ctx->d_spec[ctx->spec_cur]);
  }
  static const int k1_insert_env = [] {
    const char* e = std::getenv("SNAP_K1_INSERT");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  // Single GPU, grids above the cluster selection's 4096 chunks, K1 kernels with
  // the insert epilogue (the FNV-chain k_hash family): K1 also does the K2 insert
  // of its chunks (the table is prepared once, before the first slice of the
  // grid). Same-box A/B on C2 N=1 with the final K1: 2933-2938 vs 2921-2926 GB/s
  // (the standalone insert kernel's 7.5 us after K1 goes; in round 1, before the
  // descriptor maps, the epilogue cost more than it saved). The tensor-core K1
  // would run the insert as a separate, non-PDL range kernel: slower than the
  // standalone insert (full C2 on one GPU 4.08 vs 4.11 ms), so not there.
  // SNAP_K1_INSERT=0 / 1 forces it off / on.
  if (c0 == 0)
    ctx->k1_insert_now =
        !ctx->attached() &&
        (k1_insert_env >= 0 ? k1_insert_env == 1
                            : !snap::select_cluster_ok(ctx->nchunks) && snap::k1_epilogue_insert(g, so));
  if (ctx->k1_insert_now) {
    if (c0 == 0) {
      uint64_t *slot, *scan;
      RC(prepare_dedup(ctx, ctx->nchunks, &g.dd, &slot, &scan));
    }
    g.dd = TableDev{P<unsigned long long>(ctx->dd_keys), P<unsigned long long>(ctx->dd_vals),
                    ctx->dd_mask};
    g.dd_slot = P<uint64_t>(ctx->dd_slot);
    g.kn = TableDev{P<unsigned long long>(ctx->kn_keys), P<unsigned long long>(ctx->kn_vals),
                    ctx->kn_mask};
    g.kn_use = ctx->kn_count > 0 ? 1 : 0;
    ctx->k1_inserted = true;
  }
  k1_fanout(ctx, g);
  CKL(snap::launch_hash(ctx->arena, g, P<uint64_t>(ctx->d_dig), so, st, ctx->stream));
  ctx->spec_used = spec;
  return SNAP_OK;
}

int compact_impl(snap_ctx* ctx, uint32_t* moved = nullptr, unsigned int* nmoved = nullptr) {
  uint8_t* st;
  const bool shard = ctx->attached() && ctx->exchanged;
  if (shard && staging_target(ctx) < ctx->grid_bytes) {
    // shard-sized staging: learn the actual shard size, grow (keeping the
    // speculative bytes) before the fix-up writes beyond the prediction
    uint64_t tot[2] = {0, 0};
    CK(cudaMemcpyAsync(tot, ctx->d_my_totals.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    RC(staging_reserve(ctx, tot[1], true, &st));
    ctx->spec_bytes = std::max<uint64_t>(tot[1], 1);
  } else {
    RC(staging_reserve(ctx, ctx->grid_bytes, true, &st));
  }
  const uint64_t* spec_cur = nullptr;
  uint64_t* spec_next = nullptr;
  if (ctx->spec_used) {
    spec_cur = P<uint64_t>(ctx->d_spec[ctx->spec_cur]);
    RC(ensure(ctx, ctx->d_spec[1 - ctx->spec_cur], ctx->nchunks, &spec_next));
    if (ctx->spec_next_done) {
      spec_next = nullptr;  // the selection scan already wrote the next layout
    } else {
      CK(cudaMemsetAsync(spec_next, 0xff, ctx->nchunks * 8, ctx->stream));
    }
  }
  ctx->spec_next_done = false;
  const bool fixed = ctx->fixup_done && ctx->spec_used && !moved;
  ctx->fixup_done = false;
  if (nmoved) CK(cudaMemsetAsync(nmoved, 0, 4, ctx->stream));
  if (fixed) {
    // the selection scan already copied the mismatched chunks
  } else if (ctx->attached() && ctx->exchanged) {
    CKL(snap::launch_gather(ctx->arena, ctx->grid, P<uint32_t>(ctx->d_lens),
                            P<uint32_t>(ctx->d_my_list), P<uint64_t>(ctx->d_my_totals),
                            P<uint64_t>(ctx->d_my_off), true, spec_cur, spec_next, st,
                            ctx->nchunks, ctx->stream, moved, nmoved));
  } else {
    CKL(snap::launch_gather(ctx->arena, ctx->grid, P<uint32_t>(ctx->d_lens),
                            P<uint32_t>(ctx->sel_list), P<uint64_t>(ctx->totals),
                            P<uint64_t>(ctx->offsets), false, spec_cur, spec_next, st,
                            ctx->nchunks, ctx->stream, moved, nmoved));
  }
  if (ctx->spec_used) {
    ctx->spec_cur = 1 - ctx->spec_cur;
    ctx->spec_used = false;  // the image is final; a second compact re-gathers
    ctx->h_spec_valid = false;
  }
  ctx->staging_valid = ctx->staging.cap;
  return SNAP_OK;
}

}  // namespace

extern "C" {

const char* snap_strerror(int code) {
  switch (code) {
    case SNAP_OK: return "ok";
    case SNAP_EINVAL: return "invalid argument";
    case SNAP_ENOMEM: return "out of memory";
    case SNAP_EFAULT: return "fault (content/digest)";
    case SNAP_ECUDA: return "CUDA/NCCL error";
    case SNAP_EINTERNAL: return "internal error";
  }
  return "unknown";
}

const char* snap_last_error(const snap_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

int snap_open(int device, uint64_t arena_bytes, snap_ctx** out) {
  if (!out || arena_bytes == 0 || arena_bytes % 256) return SNAP_EINVAL;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return SNAP_ECUDA;
  }
  if (device < 0 || device >= ndev) return SNAP_EINVAL;
  snap_ctx* ctx = new snap_ctx();
  ctx->device = device;
  auto bail = [&](int code) {
    snap_close(ctx);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(SNAP_ECUDA);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(SNAP_ECUDA);
  // + one page of padding: the tensor-core K1's arena-wide tensor maps may read
  // a partial last page as a whole 4 KiB row (bytes past a buffer are never hashed)
  e = cudaMalloc(&ctx->arena, arena_bytes + 4096);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return bail(e == cudaErrorMemoryAllocation ? SNAP_ENOMEM : SNAP_ECUDA);
  }
  ctx->arena_bytes = arena_bytes;
  if (cudaMemsetAsync(ctx->arena, 0, arena_bytes, ctx->stream) != cudaSuccess) return bail(SNAP_ECUDA);
  if (cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess)
    return bail(SNAP_ECUDA);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return bail(SNAP_ECUDA);
  *out = ctx;
  return SNAP_OK;
}

int snap_close(snap_ctx* ctx) {
  if (!ctx) return SNAP_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  close_peer_windows(ctx);
  ar_release(ctx);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  local_group_leave(ctx);
  splice_release(ctx);
  window_release(ctx);
  for (DevMem* m :
       {&ctx->d_addr, &ctx->d_bytes, &ctx->d_cstart, &ctx->d_lens, &ctx->d_dig, &ctx->d_bufdig, &ctx->d_chunk_buf, &ctx->d_chunk_addr,
        &ctx->dd_keys, &ctx->dd_vals, &ctx->dd_slot, &ctx->kn_keys, &ctx->kn_vals, &ctx->kn_list,
        &ctx->scan, &ctx->sel, &ctx->owner, &ctx->offsets, &ctx->sel_list, &ctx->totals,
        &ctx->staging, &ctx->d_counts, &ctx->d_gdig, &ctx->d_glens, &ctx->d_writer,
        &ctx->d_shard_off, &ctx->d_my_list, &ctx->d_my_off, &ctx->d_my_totals, &ctx->d_dig2,
        &ctx->d_expect, &ctx->d_nbad, &ctx->d_srcoff, &ctx->d_spec[0], &ctx->d_spec[1],
        &ctx->d_tmaps, &ctx->scan2, &ctx->d_xdig, &ctx->d_xflag, &ctx->d_xh, &ctx->d_arflag,
        &ctx->d_arh, &ctx->d_arrec, &ctx->d_arptr, &ctx->d_arcnt, &ctx->d_vbad})
    release(*m);
  for (cudaEvent_t e : ctx->prof.pool) cudaEventDestroy(e);
  if (ctx->arena) cudaFree(ctx->arena);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  close_peer_staging(ctx);
  release(ctx->d_peers);
  for (cudaEvent_t e : ctx->pipe_ev) cudaEventDestroy(e);
  release(ctx->d_moved);
  for (uint8_t* q : ctx->io_pin)
    if (q) cudaFreeHost(q);
  if (ctx->h_badflag) cudaFreeHost(ctx->h_badflag);
  if (ctx->rv_exec) cudaGraphExecDestroy(ctx->rv_exec);
  if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
  if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return SNAP_OK;
}

int snap_arena(snap_ctx* ctx, void** base, uint64_t* bytes) {
  if (!ctx) return SNAP_EINVAL;
  if (base) *base = ctx->arena;
  if (bytes) *bytes = ctx->arena_bytes;
  return SNAP_OK;
}

uint64_t snap_launch_count(const snap_ctx* ctx) { return ctx ? ctx->launches : 0; }

int snap_sync(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

// splice.cpp:7-19, same arithmetic and the same InternalError condition.
int snap_layout_carve(uint64_t mem_bytes, uint64_t max_buffer_bytes, double slack_fraction,
                      uint64_t out[3]) {
  const uint64_t align = 256;
  const uint64_t slack = static_cast<uint64_t>(mem_bytes * slack_fraction);
  uint64_t scratch = std::max<uint64_t>(max_buffer_bytes, 4096);
  scratch = (scratch + align - 1) / align * align;
  if (!(mem_bytes > slack + scratch + align)) return SNAP_EINTERNAL;
  out[2] = scratch;
  out[1] = (mem_bytes - slack - scratch) / align * align;
  out[0] = out[1];
  return SNAP_OK;
}

int snap_host_alloc(uint64_t bytes, void** out) {
  if (!out) return SNAP_EINVAL;
  *out = nullptr;
  cudaError_t e = cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? SNAP_ENOMEM : SNAP_ECUDA;
  }
  return SNAP_OK;
}

int snap_host_free(void* p) {
  if (p && cudaFreeHost(p) != cudaSuccess) {
    cudaGetLastError();
    return SNAP_ECUDA;
  }
  return SNAP_OK;
}

int snap_write(snap_ctx* ctx, uint64_t addr, const void* src, uint64_t bytes) {
  if (!ctx || (!src && bytes)) return SNAP_EINVAL;
  RC(check_range(ctx, addr, bytes));
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(ctx->arena + addr, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

int snap_read(snap_ctx* ctx, uint64_t addr, void* dst, uint64_t bytes) {
  if (!ctx || (!dst && bytes)) return SNAP_EINVAL;
  RC(check_range(ctx, addr, bytes));
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(dst, ctx->arena + addr, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

int snap_fill_mix64(snap_ctx* ctx, uint64_t addr, uint64_t bytes, uint64_t seed, uint64_t base) {
  if (!ctx || addr % 8 || bytes % 8) return fail(ctx, SNAP_EINVAL, "fill: unaligned range");
  RC(check_range(ctx, addr, bytes));
  CK(cudaSetDevice(ctx->device));
  CKL(snap::launch_fill_mix64(reinterpret_cast<uint64_t*>(ctx->arena + addr), bytes / 8, seed,
                              base, ctx->stream));
  return SNAP_OK;
}

int snap_xor_words(snap_ctx* ctx, const uint64_t* addrs, uint64_t n, uint64_t value) {
  if (!ctx || (!addrs && n)) return SNAP_EINVAL;
  for (uint64_t i = 0; i < n; ++i)
    if (addrs[i] % 8 || addrs[i] + 8 > ctx->arena_bytes)
      return fail(ctx, SNAP_EINVAL, "xor_words: bad address");
  if (n == 0) return SNAP_OK;
  CK(cudaSetDevice(ctx->device));
  uint64_t* d;
  RC(ensure(ctx, ctx->d_srcoff, n, &d));
  CK(cudaMemcpyAsync(d, addrs, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CKL(snap::launch_xor_words(ctx->arena, d, n, value, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

// ---------------------------------------------------------------- K1

int snap_set_buffers(snap_ctx* ctx, const snap_buf* bufs, uint64_t n, const snap_geom* geom,
                     uint64_t* n_chunks) {
  if (!ctx || (!bufs && n)) return SNAP_EINVAL;
  snap_geom g = geom ? *geom : snap_geom{4096, 65536};
  if (!pow2(g.page_bytes) || !pow2(g.chunk_bytes) || g.page_bytes < 256 ||
      g.chunk_bytes < g.page_bytes || g.chunk_bytes / g.page_bytes > 32)
    return fail(ctx, SNAP_EINVAL, "geometry: page/chunk must be powers of two, page >= 256, "
                                  "chunk a multiple of page with <= 32 pages");
  std::vector<uint64_t> addr(n), bytes(n), cstart(n + 1);
  std::vector<uint32_t> lens;
  cstart[0] = 0;
  uint64_t total = 0;
  for (uint64_t b = 0; b < n; ++b) {
    const snap_buf& x = bufs[b];
    if (x.bytes == 0 || x.addr % 256 || x.bytes % 256)
      return fail(ctx, SNAP_EINVAL, "buffer " + std::to_string(b) +
                                        ": address and size must be non-zero multiples of 256");
    RC(check_range(ctx, x.addr, x.bytes));
    addr[b] = x.addr;
    bytes[b] = x.bytes;
    const uint64_t nc = (x.bytes + g.chunk_bytes - 1) / g.chunk_bytes;
    cstart[b + 1] = cstart[b] + nc;
    for (uint64_t k = 0; k < nc; ++k)
      lens.push_back(static_cast<uint32_t>(std::min<uint64_t>(g.chunk_bytes, x.bytes - k * g.chunk_bytes)));
    total += x.bytes;
  }
  if (cstart[n] >= (1ull << 31)) return fail(ctx, SNAP_EINVAL, "too many chunks");
  CK(cudaSetDevice(ctx->device));
  uint64_t *da, *db, *dc, *dd;
  uint32_t* dl;
  RC(ensure(ctx, ctx->d_addr, n, &da));
  RC(ensure(ctx, ctx->d_bytes, n, &db));
  RC(ensure(ctx, ctx->d_cstart, n + 1, &dc));
  RC(ensure(ctx, ctx->d_lens, cstart[n], &dl));
  RC(ensure(ctx, ctx->d_dig, cstart[n], &dd));
  CK(cudaMemcpyAsync(da, addr.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(db, bytes.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dc, cstart.data(), (n + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dl, lens.data(), lens.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  std::vector<uint32_t> cbuf;
  std::vector<uint64_t> caddr;
  const uint32_t* dcb = nullptr;
  const uint64_t* dca = nullptr;
  RC(upload_chunk_buf(ctx, ctx->d_chunk_buf, ctx->d_chunk_addr, cstart, addr.data(),
                      log2u(g.chunk_bytes), cbuf, caddr, &dcb, &dca));
  CK(cudaStreamSynchronize(ctx->stream));  // host vectors die here
  ctx->bufs.assign(bufs, bufs + n);
  ctx->geom = g;
  ctx->nchunks = cstart[n];
  ctx->grid_bytes = total;
  ctx->h_cstart = std::move(cstart);
  ctx->h_lens = std::move(lens);
  ctx->grid = GridDev{da, db, dc, static_cast<uint32_t>(n), ctx->nchunks, log2u(g.page_bytes),
                      log2u(g.chunk_bytes), dcb, dca, dca ? dl : nullptr};
  build_tmaps(ctx, ctx->d_tmaps, addr.data(), bytes.data(), static_cast<uint32_t>(n), ctx->grid);
  ctx->hashed = false;
  ctx->selected = false;
  ctx->exchanged = false;
  ctx->glens_valid = false;
  ctx->spec_ready = false;
  ctx->spec_used = false;
  ctx->k1_inserted = false;
  ctx->spec_next_done = false;
  ctx->xwin_ready = false;  // maxn may change: the next exchange re-maps the windows
  ctx->k1_fanout = false;
  if (n_chunks) *n_chunks = ctx->nchunks;
  // with a communicator attached this call is collective: the new grid's
  // counts and lengths are exchanged here, never inside a snapshot
  if (ctx->attached()) RC(grid_exchange(ctx));
  return SNAP_OK;
}

int snap_hash(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  CK(cudaSetDevice(ctx->device));
  {
    ProfScope ps(ctx, kProfHash);
    GridDev g = ctx->grid;
    k1_fanout(ctx, g);  // collective K1: digests straight into every rank's gathered vector
    CKL(snap::launch_hash(ctx->arena, g, P<uint64_t>(ctx->d_dig), nullptr, nullptr, ctx->stream));
  }
  ctx->spec_used = false;
  ctx->k1_inserted = false;
  ctx->hashed = true;
  ctx->selected = false;
  ctx->exchanged = false;
  return SNAP_OK;
}

int snap_get_digests(snap_ctx* ctx, uint64_t* chunk_digests, uint32_t* chunk_lens,
                     uint64_t* buf_digests) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->hashed) return fail(ctx, SNAP_EINVAL, "get_digests before snap_hash");
  CK(cudaSetDevice(ctx->device));
  if (chunk_digests && ctx->nchunks)
    CK(cudaMemcpyAsync(chunk_digests, ctx->d_dig.p, ctx->nchunks * 8, cudaMemcpyDeviceToHost,
                       ctx->stream));
  if (buf_digests && !ctx->bufs.empty()) {
    uint64_t* bd;
    RC(ensure(ctx, ctx->d_bufdig, ctx->bufs.size(), &bd));
    CKL(snap::launch_buf_fold(ctx->grid, P<uint64_t>(ctx->d_dig), bd, ctx->stream));
    CK(cudaMemcpyAsync(buf_digests, bd, ctx->bufs.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (chunk_lens && ctx->nchunks) std::memcpy(chunk_lens, ctx->h_lens.data(), ctx->nchunks * 4);
  return SNAP_OK;
}

// Gpu::digest (vdev.cpp:118), value-equal: digest_of_words over each whole
// range (the compatibility path; the ledger keys use the chunk-Merkle digest).
int snap_digest_whole(snap_ctx* ctx, const snap_buf* bufs, uint64_t n, uint64_t* out) {
  if (!ctx || (n && (!bufs || !out))) return SNAP_EINVAL;
  if (n == 0) return SNAP_OK;
  std::vector<uint64_t> host(3 * n + 1);
  uint64_t* addr = host.data();
  uint64_t* bytes = addr + n;
  uint64_t* seg = bytes + n;
  seg[0] = 0;
  for (uint64_t b = 0; b < n; ++b) {
    if (bufs[b].bytes == 0 || bufs[b].addr % 256 || bufs[b].bytes % 256)
      return fail(ctx, SNAP_EINVAL, "digest_whole: ranges must be non-zero multiples of 256");
    RC(check_range(ctx, bufs[b].addr, bufs[b].bytes));
    addr[b] = bufs[b].addr;
    bytes[b] = bufs[b].bytes;
    seg[b + 1] = seg[b] + snap::whole_segments(bufs[b].bytes);
  }
  const uint64_t nseg = seg[n];
  CK(cudaSetDevice(ctx->device));
  DevMem meta, tab, res;
  auto done = [&](int rc) {
    release(meta);
    release(tab);
    release(res);
    return rc;
  };
  uint64_t *dm, *dt, *dr;
  int rc = ensure(ctx, meta, host.size(), &dm);
  if (!rc) rc = ensure(ctx, tab, nseg * 256, &dt);
  if (!rc) rc = ensure(ctx, res, n, &dr);
  if (rc) return done(rc);
  if (cudaMemcpyAsync(dm, host.data(), host.size() * 8, cudaMemcpyHostToDevice, ctx->stream) !=
      cudaSuccess)
    return done(fail(ctx, SNAP_ECUDA, "digest_whole: copy"));
  ctx->launches += snap::launch_whole_digest(ctx->arena, dm, dm + n, dm + 2 * n, uint32_t(n), nseg,
                                             dt, dr, ctx->stream);
  const cudaError_t e1 = cudaGetLastError();
  const cudaError_t e2 = cudaMemcpyAsync(out, dr, n * 8, cudaMemcpyDeviceToHost, ctx->stream);
  const cudaError_t e3 = cudaStreamSynchronize(ctx->stream);
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
    return done(fail(ctx, SNAP_ECUDA, "digest_whole: kernel"));
  return done(SNAP_OK);
}

// ---------------------------------------------------------------- K2

int snap_known_clear(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  ctx->kn_count = 0;
  if (ctx->kn_mask) {
    CK(cudaSetDevice(ctx->device));
    TableDev t{P<unsigned long long>(ctx->kn_keys), P<unsigned long long>(ctx->kn_vals),
               ctx->kn_mask};
    CKL(snap::launch_table_clear(t, ctx->stream));
  }
  return SNAP_OK;
}

int snap_known_add(snap_ctx* ctx, const uint64_t* digests, uint64_t n) {
  if (!ctx || (!digests && n)) return SNAP_EINVAL;
  if (n == 0) return SNAP_OK;
  CK(cudaSetDevice(ctx->device));
  uint64_t* tmp;
  RC(ensure(ctx, ctx->d_dig2, n, &tmp));
  CK(cudaMemcpyAsync(tmp, digests, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  RC(known_insert_dev(ctx, tmp, n));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

int snap_known_commit(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->hashed) return fail(ctx, SNAP_EINVAL, "known_commit before snap_hash");
  CK(cudaSetDevice(ctx->device));
  if (ctx->attached() && ctx->exchanged) {
    // the store is global: every rank's digests become known
    const uint64_t n = uint64_t(ctx->nranks) * ctx->maxn;
    std::vector<uint32_t> gl(n);
    std::vector<uint64_t> gd(n), live;
    CK(cudaMemcpyAsync(gl.data(), ctx->d_glens.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(gd.data(), gdig_region(ctx, ctx->xepoch), n * 8, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (uint64_t i = 0; i < n; ++i)
      if (gl[i]) live.push_back(gd[i]);
    return snap_known_add(ctx, live.data(), live.size());
  }
  return known_insert_dev(ctx, P<uint64_t>(ctx->d_dig), ctx->nchunks);
}

int snap_select(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->hashed) return fail(ctx, SNAP_EINVAL, "select before snap_hash");
  CK(cudaSetDevice(ctx->device));
  if (ctx->attached()) {
    {
      ProfScope ps(ctx, kProfExchange);
      RC(exchange_impl(ctx));
    }
    ProfScope ps(ctx, kProfSelect);
    return select_stripe_impl(ctx);
  }
  ProfScope ps(ctx, kProfSelect);
  const bool inserted = ctx->k1_inserted;
  ctx->k1_inserted = false;
  uint64_t* spec_next = nullptr;
  if (ctx->spec_used)  // the staging layout becomes the next speculation
    RC(ensure(ctx, ctx->d_spec[1 - ctx->spec_cur], ctx->nchunks, &spec_next));
  // snap_snapshot: the scan also does the K3 fix-up when the staging image
  // already holds a whole grid (nothing to grow before the copies)
  const bool fix = ctx->fixup_request && ctx->spec_used && ctx->staging.cap >= ctx->grid_bytes;
  RC(select_impl(ctx, P<uint64_t>(ctx->d_dig), P<uint32_t>(ctx->d_lens), ctx->nchunks, inserted,
                 spec_next, fix ? P<uint64_t>(ctx->d_spec[ctx->spec_cur]) : nullptr,
                 fix ? static_cast<uint8_t*>(ctx->staging.p) : nullptr));
  ctx->spec_next_done = spec_next != nullptr;
  ctx->fixup_done = fix;
  return SNAP_OK;
}

int snap_get_selection(snap_ctx* ctx, uint8_t* sel, uint64_t* owner, uint64_t* offsets,
                       uint64_t* staged_bytes, uint64_t* staged_chunks) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->selected) return fail(ctx, SNAP_EINVAL, "get_selection before snap_select");
  CK(cudaSetDevice(ctx->device));
  RC(global_offsets(ctx));
  const uint64_t n = ctx->sel_n;
  uint64_t tot[2] = {0, 0};
  if (n) {
    if (sel) CK(cudaMemcpyAsync(sel, ctx->sel.p, n, cudaMemcpyDeviceToHost, ctx->stream));
    if (owner) CK(cudaMemcpyAsync(owner, ctx->owner.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (offsets)
      CK(cudaMemcpyAsync(offsets, ctx->offsets.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(tot, ctx->totals.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (staged_chunks) *staged_chunks = tot[0];
  if (staged_bytes) *staged_bytes = tot[1];
  return SNAP_OK;
}

int snap_global_info(snap_ctx* ctx, uint64_t* n_global, uint64_t* max_per_rank) {
  if (!ctx) return SNAP_EINVAL;
  const bool g = ctx->attached() && ctx->exchanged;
  if (n_global) *n_global = g ? uint64_t(ctx->nranks) * ctx->maxn : ctx->nchunks;
  if (max_per_rank) *max_per_rank = g ? ctx->maxn : ctx->nchunks;
  return SNAP_OK;
}

int snap_get_global_digests(snap_ctx* ctx, uint64_t* gdig, uint32_t* glens) {
  if (!ctx) return SNAP_EINVAL;
  if (!(ctx->attached() && ctx->exchanged)) return fail(ctx, SNAP_EINVAL, "no exchanged digests");
  CK(cudaSetDevice(ctx->device));
  const uint64_t n = uint64_t(ctx->nranks) * ctx->maxn;
  if (gdig)
    CK(cudaMemcpyAsync(gdig, gdig_region(ctx, ctx->xepoch), n * 8, cudaMemcpyDeviceToHost,
                       ctx->stream));
  if (glens) CK(cudaMemcpyAsync(glens, ctx->d_glens.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

int snap_get_shard(snap_ctx* ctx, int32_t* writer, uint64_t* shard_off, uint64_t* my_bytes,
                   uint64_t* my_chunks) {
  if (!ctx) return SNAP_EINVAL;
  if (!(ctx->attached() && ctx->exchanged && ctx->selected))
    return fail(ctx, SNAP_EINVAL, "get_shard needs a multi-rank snap_select");
  CK(cudaSetDevice(ctx->device));
  const uint64_t n = uint64_t(ctx->nranks) * ctx->maxn;
  uint64_t tot[2] = {0, 0};
  CK(cudaMemcpyAsync(tot, ctx->d_my_totals.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
  if (shard_off) {
    // offsets inside every writer's shard: one shard scan per writer rank
    uint64_t *tt, *scan2;
    RC(ensure(ctx, ctx->d_nbad, 4, &tt));
    RC(ensure(ctx, ctx->scan2, snap::scan_state_words(n) + 1, &scan2));
    CK(cudaMemsetAsync(ctx->d_shard_off.p, 0xff, n * 8, ctx->stream));
    for (int q = 0; q < ctx->nranks; ++q)
      CKL(snap::launch_shard_scan(P<int32_t>(ctx->d_writer), P<uint32_t>(ctx->d_glens), ctx->nranks,
                                  ctx->maxn, q, false, scan2,
                                  P<uint64_t>(ctx->d_shard_off), nullptr, nullptr, tt, ctx->stream));
    CK(cudaMemcpyAsync(shard_off, ctx->d_shard_off.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (writer) CK(cudaMemcpyAsync(writer, ctx->d_writer.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (shard_off) ctx->shard_offsets_all = true;
  if (my_chunks) *my_chunks = tot[0];
  if (my_bytes) *my_bytes = tot[1];
  return SNAP_OK;
}

// ------------------------------------------------- resize / reshard (C5)

static int verify_grid(snap_ctx* ctx, const uint64_t* expect_dev);

int snap_ipc_export(snap_ctx* ctx, void* handle64) {
  if (!ctx || !handle64) return SNAP_EINVAL;
  if (!ctx->staging.p) return fail(ctx, SNAP_EINVAL, "ipc_export: no staging image yet");
  CK(cudaSetDevice(ctx->device));
  return ipc_handle(ctx, ctx->staging.p, handle64);
}

int snap_ipc_import(snap_ctx* ctx, int nranks, const void* handles) {
  if (!ctx || !handles || nranks != ctx->nranks) return SNAP_EINVAL;
  CK(cudaSetDevice(ctx->device));
  close_peer_staging(ctx);
  ctx->peer_staging.assign(nranks, nullptr);
  ctx->peer_opened.assign(nranks, false);
  for (int r = 0; r < nranks; ++r) {
    if (r == ctx->rank) {
      ctx->peer_staging[r] = ctx->staging.p;
      continue;
    }
    bool opened = false;
    RC(ipc_open(ctx, static_cast<const uint8_t*>(handles) + 64 * r, &ctx->peer_staging[r], &opened));
    ctx->peer_opened[r] = opened;
  }
  void** dp;
  RC(ensure(ctx, ctx->d_peers, nranks, &dp));
  CK(cudaMemcpyAsync(dp, ctx->peer_staging.data(), nranks * sizeof(void*), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

// restore_job materialization after a resize (ckpt.cpp:504-533): rank
// `src_rank`'s layout (= the installed grid) is rebuilt from the striped
// shards of the last multi-rank snapshot, reading peer shards over NVLink.
int snap_restore_shards(snap_ctx* ctx, int src_rank, int verify) {
  if (!ctx || !ctx->attached() || !ctx->exchanged || !ctx->selected || src_rank < 0 ||
      src_rank >= ctx->nranks)
    return fail(ctx, SNAP_EINVAL, "restore_shards needs a multi-rank snapshot");
  if (int(ctx->peer_staging.size()) != ctx->nranks)
    return fail(ctx, SNAP_EINVAL, "restore_shards: peers not imported (snap_ipc_import)");
  if (ctx->counts[src_rank] != ctx->nchunks)
    return fail(ctx, SNAP_EINVAL, "restore_shards: installed grid is not src_rank's layout");
  CK(cudaSetDevice(ctx->device));
  if (!ctx->shard_offsets_all) {
    uint64_t *tt, *scan2;
    const uint64_t n = uint64_t(ctx->nranks) * ctx->maxn;
    RC(ensure(ctx, ctx->d_nbad, 4, &tt));
    RC(ensure(ctx, ctx->scan2, snap::scan_state_words(n) + 1, &scan2));
    CK(cudaMemsetAsync(ctx->d_shard_off.p, 0xff, n * 8, ctx->stream));
    for (int q = 0; q < ctx->nranks; ++q)
      CKL(snap::launch_shard_scan(P<int32_t>(ctx->d_writer), P<uint32_t>(ctx->d_glens), ctx->nranks,
                                  ctx->maxn, q, false, scan2,
                                  P<uint64_t>(ctx->d_shard_off), nullptr, nullptr, tt, ctx->stream));
    ctx->shard_offsets_all = true;
  }
  unsigned long long* miss;
  RC(ensure(ctx, ctx->d_nbad, 4, &miss));
  {
    ProfScope ps(ctx, kProfRestore);
    CKL(snap::launch_scatter_shards(ctx->arena, ctx->grid, P<uint32_t>(ctx->d_lens),
                                    uint64_t(src_rank) * ctx->maxn, P<uint64_t>(ctx->owner),
                                    P<int32_t>(ctx->d_writer), P<uint64_t>(ctx->d_shard_off),
                                    P<const uint8_t*>(ctx->d_peers), miss + 1, ctx->stream));
  }
  unsigned long long missing = 0;
  CK(cudaMemcpyAsync(&missing, miss + 1, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (missing)
    return fail(ctx, SNAP_EFAULT, "restore_shards: " + std::to_string(missing) +
                                      " chunk(s) have no source (known/older blobs)");
  if (!verify) return SNAP_OK;
  // expected digests: src_rank's row of the allgathered vector
  return verify_grid(ctx, gdig_region(ctx, ctx->xepoch) + uint64_t(src_rank) * ctx->maxn);
}

// ---------------------------------------------------------------- K3

int snap_compact(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->selected) return fail(ctx, SNAP_EINVAL, "compact before snap_select");
  CK(cudaSetDevice(ctx->device));
  ProfScope ps(ctx, kProfCompact);
  return compact_impl(ctx);
}

int snap_snapshot(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  CK(cudaSetDevice(ctx->device));
  {
    ProfScope ps(ctx, kProfHash);
    RC(hash_fused(ctx));
  }
  ctx->hashed = true;
  ctx->selected = false;
  ctx->exchanged = false;
  ctx->fixup_request = true;
  const int rc = snap_select(ctx);
  ctx->fixup_request = false;
  if (rc != SNAP_OK) return rc;
  return snap_compact(ctx);
}

}  // extern "C"

namespace {

// Pipelined host-buffer snapshot: the image is copied in slabs on an H2D
// stream, each slab's complete chunks are hashed (+ speculatively staged) on
// the compute stream as soon as they land, and their staging bytes go back on
// a D2H stream while later slabs are still copying in, so PCIe runs both
// directions concurrently with the kernels. After selection, chunks the fix-up
// moved are copied again (ordered after the speculative copies).
int snapshot_host_pipelined(snap_ctx* ctx, const uint8_t* host_src, uint64_t addr,
                            uint64_t bytes, uint8_t* host_staging, uint64_t cap,
                            uint64_t* staged_bytes, uint64_t* host_digests) {
  const uint64_t n = ctx->nchunks;
  static const uint64_t slab = [] {  // SNAP_HOST_SLAB_MB: pipeline granularity
    const char* e = std::getenv("SNAP_HOST_SLAB_MB");
    const long mb = e ? std::atol(e) : 0;
    return uint64_t(mb > 0 ? mb : 64) << 20;
  }();
  const uint64_t nslab = (bytes + slab - 1) / slab;
  if (!ctx->h2d) CK(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
  if (!ctx->d2h) CK(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
  while (ctx->pipe_ev.size() < 2 * nslab + 2) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->pipe_ev.push_back(e);
  }
  const bool spec = ctx->kn_count == 0;
  if (spec) {
    if (!ctx->spec_ready) RC(init_spec(ctx));
    if (!ctx->h_spec_valid) {
      ctx->h_spec.resize(n);
      CK(cudaMemcpyAsync(ctx->h_spec.data(), ctx->d_spec[ctx->spec_cur].p, n * 8,
                         cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      ctx->h_spec_valid = true;
    }
  }
  uint8_t* st;
  RC(staging_reserve(ctx, staging_target(ctx), true, &st));
  uint32_t* moved;
  RC(ensure(ctx, ctx->d_moved, n + 1, &moved));
  // chunk end addresses (canonical order, increasing: checked by the caller)
  uint64_t next = 0, b = 0;
  auto chunk_end = [&](uint64_t g) {
    while (ctx->h_cstart[b + 1] <= g) ++b;
    const uint64_t k = g - ctx->h_cstart[b];
    return ctx->bufs[b].addr + (k << log2u(ctx->geom.chunk_bytes)) + ctx->h_lens[g];
  };
  {
    ProfScope ps(ctx, kProfHash);
    for (uint64_t k = 0; k < nslab; ++k) {
      const uint64_t s0 = k * slab, s1 = std::min(bytes, s0 + slab);
      CK(cudaMemcpyAsync(ctx->arena + addr + s0, host_src + s0, s1 - s0, cudaMemcpyHostToDevice,
                         ctx->h2d));
      CK(cudaEventRecord(ctx->pipe_ev[2 * k], ctx->h2d));
      uint64_t hi = next;
      while (hi < n && chunk_end(hi) <= addr + s1) ++hi;
      if (hi == next) continue;
      CK(cudaStreamWaitEvent(ctx->stream, ctx->pipe_ev[2 * k], 0));
      RC(hash_fused(ctx, next, hi));
      if (spec && host_staging) {
        uint64_t lo = ~0ull, top = 0;
        for (uint64_t g = next; g < hi; ++g)
          if (ctx->h_spec[g] != ~0ull) {
            lo = std::min(lo, ctx->h_spec[g]);
            top = std::max(top, ctx->h_spec[g] + ctx->h_lens[g]);
          }
        top = std::min(top, cap);
        if (lo < top) {
          CK(cudaEventRecord(ctx->pipe_ev[2 * k + 1], ctx->stream));
          CK(cudaStreamWaitEvent(ctx->d2h, ctx->pipe_ev[2 * k + 1], 0));
          CK(cudaMemcpyAsync(host_staging + lo, st + lo, top - lo, cudaMemcpyDeviceToHost,
                             ctx->d2h));
        }
      }
      next = hi;
    }
  }
  if (next != n) return fail(ctx, SNAP_EINTERNAL, "snapshot_host: chunks outside the image");
  ctx->hashed = true;
  ctx->selected = false;
  ctx->exchanged = false;
  RC(snap_select(ctx));
  {
    ProfScope ps(ctx, kProfCompact);
    RC(compact_impl(ctx, moved, reinterpret_cast<unsigned int*>(moved + n)));
  }
  st = static_cast<uint8_t*>(ctx->staging.p);  // the fix-up may have grown the image
  ctx->h_spec_valid = false;  // the fix-up wrote the next layout on the device
  const bool shard = ctx->attached() && ctx->exchanged;
  uint64_t tot[2] = {0, 0};
  uint32_t nmv = 0;
  CK(cudaMemcpyAsync(tot, shard ? ctx->d_my_totals.p : ctx->totals.p, 16, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaMemcpyAsync(&nmv, moved + n, 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (host_digests && n)
    CK(cudaMemcpyAsync(host_digests, ctx->d_dig.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (host_staging && tot[1] > cap)
    return fail(ctx, SNAP_EINVAL, "snapshot_host: staging buffer too small");
  if (host_staging) {
    CK(cudaEventRecord(ctx->pipe_ev[2 * nslab], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->d2h, ctx->pipe_ev[2 * nslab], 0));
    if (!spec) {
      if (tot[1])
        CK(cudaMemcpyAsync(host_staging, st, tot[1], cudaMemcpyDeviceToHost, ctx->d2h));
    } else if (nmv) {
      // chunks the fix-up rewrote: copy their final bytes (after the speculative copies)
      std::vector<uint32_t> idx(nmv), list;
      CK(cudaMemcpy(idx.data(), moved, nmv * 4ull, cudaMemcpyDeviceToHost));
      std::vector<uint64_t> off(shard ? ctx->maxn : n);
      std::vector<uint32_t> lst(shard ? ctx->maxn : n);
      CK(cudaMemcpy(off.data(), shard ? ctx->d_my_off.p : ctx->offsets.p, off.size() * 8,
                    cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(lst.data(), shard ? ctx->d_my_list.p : ctx->sel_list.p, lst.size() * 4,
                    cudaMemcpyDeviceToHost));
      for (uint32_t w : idx) {
        const uint32_t gc = lst[w];
        const uint64_t o = shard ? off[w] : off[gc];
        CK(cudaMemcpyAsync(host_staging + o, st + o, ctx->h_lens[gc], cudaMemcpyDeviceToHost,
                           ctx->d2h));
      }
    }
    CK(cudaStreamSynchronize(ctx->d2h));
  }
  ctx->staging_valid = ctx->staging.cap;
  if (staged_bytes) *staged_bytes = tot[1];
  return SNAP_OK;
}

// The pipelined path needs the grid's chunks in increasing address order
// inside [addr, addr + bytes).
bool pipelinable(const snap_ctx* ctx, uint64_t addr, uint64_t bytes) {
  uint64_t last = addr;
  for (const snap_buf& b : ctx->bufs) {
    if (b.addr < last || b.addr + b.bytes > addr + bytes) return false;
    last = b.addr + b.bytes;
  }
  return true;
}

}  // namespace

extern "C" {

int snap_snapshot_host(snap_ctx* ctx, const void* host_src, uint64_t addr, uint64_t bytes,
                       void* host_staging, uint64_t staging_cap, uint64_t* staged_bytes,
                       uint64_t* host_digests) {
  if (!ctx || (!host_src && bytes)) return SNAP_EINVAL;
  RC(check_range(ctx, addr, bytes));
  CK(cudaSetDevice(ctx->device));
  if (bytes && ctx->nchunks && pipelinable(ctx, addr, bytes))
    return snapshot_host_pipelined(ctx, static_cast<const uint8_t*>(host_src), addr, bytes,
                                   static_cast<uint8_t*>(host_staging), staging_cap,
                                   staged_bytes, host_digests);
  if (bytes)
    CK(cudaMemcpyAsync(ctx->arena + addr, host_src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  RC(snap_snapshot(ctx));
  uint64_t tot[2] = {0, 0};
  const bool shard = ctx->attached() && ctx->exchanged;
  CK(cudaMemcpyAsync(tot, shard ? ctx->d_my_totals.p : ctx->totals.p, 16, cudaMemcpyDeviceToHost,
                     ctx->stream));
  if (host_digests && ctx->nchunks)
    CK(cudaMemcpyAsync(host_digests, ctx->d_dig.p, ctx->nchunks * 8, cudaMemcpyDeviceToHost,
                       ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (tot[1] > staging_cap && host_staging)
    return fail(ctx, SNAP_EINVAL, "snapshot_host: staging buffer too small");
  if (host_staging && tot[1]) {
    CK(cudaMemcpyAsync(host_staging, ctx->staging.p, tot[1], cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  if (staged_bytes) *staged_bytes = tot[1];
  return SNAP_OK;
}

int snap_staging(snap_ctx* ctx, void** dev_ptr, uint64_t* bytes) {
  if (!ctx) return SNAP_EINVAL;
  if (dev_ptr) *dev_ptr = ctx->staging.p;
  if (bytes) *bytes = ctx->staging_valid;
  return SNAP_OK;
}

int snap_read_staging(snap_ctx* ctx, uint64_t off, void* dst, uint64_t bytes) {
  if (!ctx || (!dst && bytes)) return SNAP_EINVAL;
  if (off > ctx->staging_valid || bytes > ctx->staging_valid - off)
    return fail(ctx, SNAP_EINVAL, "read_staging: range outside the staging image");
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(dst, static_cast<uint8_t*>(ctx->staging.p) + off, bytes,
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

// ---------------------------------------------------------------- K4

static int verify_grid(snap_ctx* ctx, const uint64_t* expect_dev) {
  uint64_t* d2;
  unsigned long long* nbad;
  RC(ensure(ctx, ctx->d_dig2, ctx->nchunks, &d2));
  RC(ensure(ctx, ctx->d_nbad, 4, &nbad));
  CKL(snap::launch_hash(ctx->arena, ctx->grid, d2, nullptr, nullptr, ctx->stream));
  CKL(snap::launch_compare(d2, expect_dev, ctx->nchunks, nbad, ctx->stream));
  unsigned long long bad = 0;
  CK(cudaMemcpyAsync(&bad, nbad, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (bad)
    return fail(ctx, SNAP_EFAULT, "restore: digest verification failed on " + std::to_string(bad) +
                                      " chunk(s)");
  return SNAP_OK;
}

// K4 + verification in one pass (restore_job materialization, ckpt.cpp:517-528,
// with BlobStore::get's digest check of the blob it reads, ckpt.cpp:23-29):
// every chunk is read once from the image, written to its recorded address
// and hashed from shared memory on the way; mismatches against `expect` are
// counted by the kernel. 2 x restored bytes of traffic instead of 3.
static int restore_verified(snap_ctx* ctx, const uint8_t* image, const uint64_t* src_off_dev,
                            const uint64_t* expect_dev) {
  uint64_t* d2;
  unsigned long long* nbad;
  RC(ensure(ctx, ctx->d_dig2, ctx->nchunks, &d2));
  const bool fresh = ctx->d_vbad.p == nullptr;
  RC(ensure(ctx, ctx->d_vbad, 4, &nbad));
  if (!ctx->h_badflag) {
    // the mismatch flag lives in mapped pinned memory: the success path is one
    // kernel and a stream synchronize (no memset, no read-back copy)
    void* hp = nullptr;
    CK(cudaHostAlloc(&hp, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    ctx->h_badflag = static_cast<unsigned int*>(hp);
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->d_badflag), hp, 0));
  }
  // the counter stays zero between calls (reset below after a mismatch)
  if (fresh) CK(cudaMemsetAsync(nbad, 0, 8, ctx->stream));
  *reinterpret_cast<volatile unsigned int*>(ctx->h_badflag) = 0;
  // byte copy (padding included): the graph cache below keys on the bytes of g
  GridDev g;
  std::memcpy(static_cast<void*>(&g), &ctx->grid, sizeof(GridDev));
  g.reverse = 1;
  g.expect = expect_dev;
  g.nbad = nbad;
  g.bad_flag = ctx->d_badflag;
  static const bool graphs = [] {
    const char* e = std::getenv("SNAP_RESTORE_GRAPH");
    return !(e && e[0] == '0');
  }();
  if (graphs && !ctx->prof.on) {
    // repeated restores of the same layout (C1's loop, a resuming job's retries):
    // replay one instantiated graph instead of re-encoding the launch
    std::vector<uint8_t> key(sizeof(GridDev) + 4 * sizeof(void*));
    std::memcpy(key.data(), &g, sizeof(GridDev));
    const void* ptrs[4] = {image, src_off_dev, d2, ctx->arena};
    std::memcpy(key.data() + sizeof(GridDev), ptrs, sizeof(ptrs));
    if (!ctx->rv_exec || key != ctx->rv_key) {
      if (ctx->rv_exec) cudaGraphExecDestroy(ctx->rv_exec);
      ctx->rv_exec = nullptr;
      cudaGraph_t graph = nullptr;
      CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      const int n = snap::launch_hash(ctx->arena, g, d2, src_off_dev, const_cast<uint8_t*>(image),
                                      ctx->stream);
      const cudaError_t le = cudaGetLastError();
      CK(cudaStreamEndCapture(ctx->stream, &graph));
      if (le != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        CK(le);
      }
      const cudaError_t e = cudaGraphInstantiate(&ctx->rv_exec, graph, 0);
      cudaGraphDestroy(graph);
      CK(e);
      ctx->rv_key = std::move(key);
      ctx->rv_launches = n;
    }
    CK(cudaGraphLaunch(ctx->rv_exec, ctx->stream));
    ctx->launches += uint64_t(ctx->rv_launches);
  } else {
    ProfScope ps(ctx, kProfRestore);
    CKL(snap::launch_hash(ctx->arena, g, d2, src_off_dev, const_cast<uint8_t*>(image), ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (*reinterpret_cast<volatile unsigned int*>(ctx->h_badflag) == 0) return SNAP_OK;
  unsigned long long bad = 0;
  CK(cudaMemcpy(&bad, nbad, 8, cudaMemcpyDeviceToHost));
  CK(cudaMemset(nbad, 0, 8));
  return fail(ctx, SNAP_EFAULT, "restore: digest verification failed on " + std::to_string(bad) +
                                    " chunk(s)");
}

int snap_restore(snap_ctx* ctx, const void* image, uint64_t image_bytes, const uint64_t* src_off,
                 const uint64_t* expect_digests, int verify) {
  if (!ctx || (!src_off && ctx->nchunks) || (!image && ctx->nchunks)) return SNAP_EINVAL;
  if (ctx->nchunks == 0) return SNAP_OK;  // empty layout: nothing to write or verify
  for (uint64_t g = 0; g < ctx->nchunks; ++g)
    if (src_off[g] > image_bytes || ctx->h_lens[g] > image_bytes - src_off[g] || src_off[g] % 256)
      return fail(ctx, SNAP_EFAULT, "restore: chunk " + std::to_string(g) +
                                        " has no source in the image (missing blob)");
  CK(cudaSetDevice(ctx->device));
  uint64_t* so;
  RC(ensure(ctx, ctx->d_srcoff, ctx->nchunks, &so));
  CK(cudaMemcpyAsync(so, src_off, ctx->nchunks * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (verify) {
    const uint64_t* expect = P<uint64_t>(ctx->d_dig);
    if (expect_digests) {
      uint64_t* e;
      RC(ensure(ctx, ctx->d_expect, ctx->nchunks, &e));
      CK(cudaMemcpyAsync(e, expect_digests, ctx->nchunks * 8, cudaMemcpyHostToDevice, ctx->stream));
      expect = e;
    } else if (!ctx->hashed) {
      return fail(ctx, SNAP_EINVAL, "restore verify needs expect_digests or a prior snap_hash");
    }
    return restore_verified(ctx, static_cast<const uint8_t*>(image), so, expect);
  }
  {
    ProfScope ps(ctx, kProfRestore);
    CKL(snap::launch_scatter(ctx->arena, ctx->grid, P<uint32_t>(ctx->d_lens),
                             static_cast<const uint8_t*>(image), so, ctx->stream));
  }
  return snap_sync(ctx);
}

int snap_restore_self(snap_ctx* ctx, int verify) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->selected) return fail(ctx, SNAP_EINVAL, "restore_self needs a prior snapshot");
  if (ctx->kn_count)
    return fail(ctx, SNAP_EINVAL, "restore_self: incremental snapshot (known set) needs the "
                                  "older images; use snap_restore");
  if (ctx->attached() && ctx->exchanged)
    return fail(ctx, SNAP_EINVAL, "restore_self: multi-rank snapshots restore from the shards "
                                  "(snap_restore)");
  CK(cudaSetDevice(ctx->device));
  if (verify)
    return restore_verified(ctx, static_cast<const uint8_t*>(ctx->staging.p),
                            P<uint64_t>(ctx->offsets), P<uint64_t>(ctx->d_dig));
  {
    ProfScope ps(ctx, kProfRestore);
    CKL(snap::launch_scatter(ctx->arena, ctx->grid, P<uint32_t>(ctx->d_lens),
                             static_cast<const uint8_t*>(ctx->staging.p), P<uint64_t>(ctx->offsets),
                             ctx->stream));
  }
  return SNAP_OK;
}

// ---------------------------------------------------------------- K5

int snap_grad_sum(snap_ctx* ctx, int dtype, const uint64_t* src_addrs, uint32_t nsrc,
                  uint64_t dst_addr, uint64_t elems, int accumulate) {
  if (!ctx || !src_addrs || (dtype != SNAP_U64 && dtype != SNAP_F32 && dtype != SNAP_BF16) ||
      nsrc == 0 || nsrc > 16)
    return fail(ctx, SNAP_EINVAL, "grad_sum: bad arguments (1..16 sources, u64|f32|bf16)");
  const uint64_t esz = dtype == SNAP_F32 ? 4 : dtype == SNAP_BF16 ? 2 : 8;
  if (elems > ctx->arena_bytes / esz) return fail(ctx, SNAP_EINVAL, "grad_sum: size");
  for (uint32_t r = 0; r < nsrc; ++r) {
    if (src_addrs[r] % 16) return fail(ctx, SNAP_EINVAL, "grad_sum: sources must be 16-B aligned");
    RC(check_range(ctx, src_addrs[r], elems * esz));
  }
  if (dst_addr % 16) return fail(ctx, SNAP_EINVAL, "grad_sum: dst must be 16-B aligned");
  RC(check_range(ctx, dst_addr, elems * esz));
  CK(cudaSetDevice(ctx->device));
  ProfScope ps(ctx, kProfGrad);
  CKL(snap::launch_grad_sum(dtype, ctx->arena, src_addrs, nsrc, dst_addr, elems, accumulate,
                            ctx->stream));
  return SNAP_OK;
}

// ---------------------------------------------------------------- NCCL

int snap_comm_unique_id(void* id128) {
  if (!id128) return SNAP_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SNAP_ECUDA;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id128, &id, 128);
  return SNAP_OK;
}

int snap_comm_init(snap_ctx* ctx, int nranks, int rank, const void* id128) {
  if (!ctx || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return SNAP_EINVAL;
  CK(cudaSetDevice(ctx->device));
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  if (ctx->attached()) return fail(ctx, SNAP_EINVAL, "comm_init: destroy the current communicator "
                                               "first (snap_comm_destroy, collective)");
  CKN(ncclCommInitRank(&ctx->comm, nranks, id, rank));
  ctx->nranks = nranks;
  ctx->rank = rank;
  ctx->xepoch = 0;
  ctx->xwin_ready = false;
  ctx->k1_fanout = false;
  ctx->glens_valid = false;
  ctx->exchanged = false;
  ctx->spec_ready = false;
  return grid_exchange(ctx);  // the installed grid (possibly empty) of every rank
}

// Collective over the communicator's ranks (the rendezvous of a resize,
// collectives.cpp:37-59, rebuilds the device-level world afterwards).
int snap_comm_destroy(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->attached()) return SNAP_OK;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  close_peer_staging(ctx);
  close_peer_windows(ctx);
  ar_release(ctx);
  if (ctx->comm) {
    CKN(ncclCommDestroy(ctx->comm));
    ctx->comm = nullptr;
  }
  if (ctx->lgroup) {
    const bool ok = comm_barrier(ctx);  // no peer still reads this rank's buffers
    local_group_leave(ctx);
    if (!ok) return fail(ctx, SNAP_EINTERNAL, "comm_destroy: a peer rank never arrived");
  }
  ctx->nranks = 1;
  ctx->rank = 0;
  ctx->glens_valid = false;
  ctx->exchanged = false;
  ctx->selected = false;
  ctx->spec_ready = false;
  return SNAP_OK;
}

int snap_allreduce(snap_ctx* ctx, int dtype, uint64_t addr, uint64_t elems) {
  if (!ctx || !ctx->attached()) return fail(ctx, SNAP_EINVAL, "allreduce: no communicator");
  if (dtype != SNAP_U64 && dtype != SNAP_F32)
    return fail(ctx, SNAP_EINVAL, "allreduce: u64 | f32 (bf16: snap_allreduce_ordered)");
  const uint64_t esz = dtype == SNAP_F32 ? 4 : 8;
  RC(check_range(ctx, addr, elems * esz));
  CK(cudaSetDevice(ctx->device));
  return comm_allreduce(ctx, ctx->arena + addr, ctx->arena + addr, elems,
                        dtype == SNAP_F32 ? kCommF32 : kCommU64, kCommSum);
}

// ---------------------------------------------------------------- timing

int snap_timer_start(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  return SNAP_OK;
}

int snap_timer_stop(snap_ctx* ctx, float* ms) {
  if (!ctx || !ms) return SNAP_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  CK(cudaEventSynchronize(ctx->ev1));
  CK(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
  return SNAP_OK;
}

int snap_set_k1_variant(int variant) {
  snap::set_hash_variant(variant);
  return SNAP_OK;
}

const char* snap_last_k1_kernel(void) { return snap::last_k1_name(); }

int snap_prof_enable(snap_ctx* ctx, int on) {
  if (!ctx) return SNAP_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->prof.on = on != 0;
  ctx->prof.used = 0;
  ctx->prof.marks.clear();
  return SNAP_OK;
}

int snap_prof_read(snap_ctx* ctx, int kind, float* total_ms, uint64_t* count) {
  if (!ctx || !total_ms || !count) return SNAP_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  float tot = 0;
  uint64_t n = 0;
  for (auto& m : ctx->prof.marks)
    if (m.first == kind) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, m.second.first, m.second.second));
      tot += ms;
      ++n;
    }
  *total_ms = tot;
  *count = n;
  return SNAP_OK;
}

}  // extern "C"
