// window.cpp — digests of ad-hoc buffer lists on an auxiliary chunk grid, and
// the squash-window validation built on them:
//
//   snap_digest_ranges  Gpu::digest (vdev.cpp:118) for a batch of ranges
//   snap_window_open    WorkerExec::do_window_open, validation branch (worker.cpp:355-362)
//   snap_window_close   WorkerExec::do_window_close, validation branch (worker.cpp:411-421)
//   snap_validate_window  splice::validate_window (splice.cpp:21-61), host logic
//
// The reference re-hashes every live buffer of the rank byte-serially at window
// open and close; here both are one K1 launch over the rank's chunk grid (+ the
// per-buffer fold), on a grid of their own so the installed snapshot grid, its
// digests and its selection are untouched.
#include <map>

#include "ctx.h"

struct AuxGrid {
  DevMem d_addr, d_bytes, d_cstart, d_dig, d_bufdig;
  GridDev grid;
  // host-page snapshot scratch: paged image, slots, flags, counts, page + prev tables
  DevMem d_img, d_slot, d_flags, d_counts, pt_keys, pt_vals, pv_keys, pv_vals, d_prev;
};

struct WindowState {
  AuxGrid aux;
  // rank -> open snapshot addr -> (bytes, digest)   (ProxyWindow::open_snapshot)
  std::map<int, std::map<uint64_t, std::pair<uint64_t, uint64_t>>> open;
};

void window_release(snap_ctx* ctx) {
  WindowState* W = ctx->win;
  if (!W) return;
  AuxGrid& A = W->aux;
  for (DevMem* m : {&A.d_addr, &A.d_bytes, &A.d_cstart, &A.d_dig, &A.d_bufdig, &A.d_img,
                    &A.d_slot, &A.d_flags, &A.d_counts, &A.pt_keys, &A.pt_vals, &A.pv_keys,
                    &A.pv_vals, &A.d_prev})
    release(*m);
  delete W;
  ctx->win = nullptr;
}

namespace {

WindowState& state(snap_ctx* ctx) {
  if (!ctx->win) ctx->win = new WindowState();
  return *ctx->win;
}

// K1 + buffer fold over `bufs` on the auxiliary grid; buffer digests to the host.
int aux_digests(snap_ctx* ctx, const snap_buf* bufs, uint64_t n, const snap_geom& g,
                uint64_t* out) {
  if (!pow2(g.page_bytes) || !pow2(g.chunk_bytes) || g.page_bytes < 256 ||
      g.chunk_bytes < g.page_bytes || g.chunk_bytes / g.page_bytes > 32)
    return fail(ctx, SNAP_EINVAL, "geometry: page/chunk must be powers of two, page >= 256, "
                                  "chunk a multiple of page with <= 32 pages");
  if (n == 0) return SNAP_OK;
  std::vector<uint64_t> addr(n), bytes(n), cstart(n + 1, 0);
  for (uint64_t b = 0; b < n; ++b) {
    const snap_buf& x = bufs[b];
    if (x.bytes == 0 || x.addr % 256 || x.bytes % 256)
      return fail(ctx, SNAP_EINVAL, "buffer " + std::to_string(b) +
                                        ": address and size must be non-zero multiples of 256");
    RC(check_range(ctx, x.addr, x.bytes));
    addr[b] = x.addr;
    bytes[b] = x.bytes;
    cstart[b + 1] = cstart[b] + (x.bytes + g.chunk_bytes - 1) / g.chunk_bytes;
  }
  if (cstart[n] >= (1ull << 31)) return fail(ctx, SNAP_EINVAL, "too many chunks");
  CK(cudaSetDevice(ctx->device));
  AuxGrid& A = state(ctx).aux;
  uint64_t *da, *db, *dc, *dd, *bd;
  RC(ensure(ctx, A.d_addr, n, &da));
  RC(ensure(ctx, A.d_bytes, n, &db));
  RC(ensure(ctx, A.d_cstart, n + 1, &dc));
  RC(ensure(ctx, A.d_dig, cstart[n], &dd));
  RC(ensure(ctx, A.d_bufdig, n, &bd));
  CK(cudaMemcpyAsync(da, addr.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(db, bytes.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dc, cstart.data(), (n + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  A.grid = GridDev{da, db, dc, uint32_t(n), cstart[n], log2u(g.page_bytes), log2u(g.chunk_bytes)};
  CKL(snap::launch_hash(ctx->arena, A.grid, dd, nullptr, nullptr, ctx->stream));
  CKL(snap::launch_buf_fold(A.grid, dd, bd, ctx->stream));
  CK(cudaMemcpyAsync(out, bd, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // host vectors die here
  return SNAP_OK;
}

// the rank's live, non-pending buffers (worker.cpp:359-360, 415-416) and their digests
int live_digests(snap_ctx* ctx, const snap_buf* bufs, uint64_t n, std::vector<snap_buf>& live,
                 std::vector<uint64_t>& dig) {
  live.clear();
  for (uint64_t i = 0; i < n; ++i)
    if (!(bufs[i].flags & SNAP_BUF_PENDING)) live.push_back(bufs[i]);
  dig.assign(live.size(), 0);
  return aux_digests(ctx, live.data(), live.size(), snap_geom{4096, 65536}, dig.data());
}

}  // namespace

extern "C" {

int snap_digest_ranges(snap_ctx* ctx, const snap_buf* bufs, uint64_t n, const snap_geom* geom,
                       uint64_t* out) {
  if (!ctx || (n && (!bufs || !out))) return SNAP_EINVAL;
  return aux_digests(ctx, bufs, n, geom ? *geom : snap_geom{4096, 65536}, out);
}

int snap_window_open(snap_ctx* ctx, int rank, const snap_buf* bufs, uint64_t n) {
  if (!ctx || rank < 0 || (!bufs && n)) return SNAP_EINVAL;
  std::vector<snap_buf> live;
  std::vector<uint64_t> dig;
  RC(live_digests(ctx, bufs, n, live, dig));
  auto& snap = state(ctx).open[rank];
  snap.clear();
  for (size_t i = 0; i < live.size(); ++i) snap[live[i].addr] = {live[i].bytes, dig[i]};
  return SNAP_OK;
}

int snap_window_close(snap_ctx* ctx, int rank, const snap_buf* bufs, uint64_t n,
                      snap_mutation* out, uint64_t cap, uint64_t* n_out) {
  if (!ctx || rank < 0 || (!bufs && n) || !n_out) return SNAP_EINVAL;
  auto it = state(ctx).open.find(rank);
  if (it == state(ctx).open.end())
    return fail(ctx, SNAP_EINTERNAL, "window close without open");  // worker.cpp:386
  std::vector<snap_buf> live;
  std::vector<uint64_t> dig;
  RC(live_digests(ctx, bufs, n, live, dig));
  std::map<uint64_t, std::pair<uint64_t, uint64_t>> mut;  // rec.mutations (address order)
  for (size_t i = 0; i < live.size(); ++i) {
    auto s = it->second.find(live[i].addr);
    if (s == it->second.end() || s->second.second != dig[i] || s->second.first != live[i].bytes)
      mut[live[i].addr] = {live[i].bytes, dig[i]};
  }
  *n_out = mut.size();
  if (out) {
    if (cap < mut.size()) return fail(ctx, SNAP_EINVAL, "window_close: output capacity");
    size_t k = 0;
    for (const auto& [a, bd] : mut) out[k++] = snap_mutation{a, bd.first, bd.second};
  }
  state(ctx).open.erase(it);
  return SNAP_OK;
}

int snap_host_pages(snap_ctx* ctx, const void* const* bufs, const uint64_t* words, uint64_t nbufs,
                    const uint64_t* prev, uint64_t n_prev, uint64_t* page_digests, uint64_t cap,
                    uint8_t* flags, snap_pages_stats* st) {
  if (!ctx || (nbufs && (!bufs || !words)) || (n_prev && !prev)) return SNAP_EINVAL;
  constexpr uint64_t kPage = 4096;
  uint64_t total = 0;
  for (uint64_t i = 0; i < nbufs; ++i) total += words[i] * 8;
  const uint64_t npages = (total + kPage - 1) / kPage;
  snap_pages_stats out{npages, npages * kPage, 0, 0};
  if (st) *st = out;
  if ((page_digests || flags) && cap < npages)
    return fail(ctx, SNAP_EINVAL, "host_pages: output capacity below the page count");
  if (npages == 0) return SNAP_OK;
  if (npages >= (1ull << 31)) return fail(ctx, SNAP_EINVAL, "host_pages: too many pages");
  CK(cudaSetDevice(ctx->device));
  AuxGrid& A = state(ctx).aux;
  uint8_t *img, *fl;
  uint64_t *da, *db, *dc, *dd, *slot, *dp;
  unsigned long long *cnt, *pk, *pv, *vk, *vv;
  const uint64_t pcap = table_cap(npages), vcap = table_cap(std::max<uint64_t>(n_prev, 1));
  RC(ensure(ctx, A.d_img, npages * kPage, &img));
  RC(ensure(ctx, A.d_addr, 1, &da));
  RC(ensure(ctx, A.d_bytes, 1, &db));
  RC(ensure(ctx, A.d_cstart, 2, &dc));
  RC(ensure(ctx, A.d_dig, npages, &dd));
  RC(ensure(ctx, A.d_slot, npages, &slot));
  RC(ensure(ctx, A.d_flags, npages, &fl));
  RC(ensure(ctx, A.d_counts, 2, &cnt));
  RC(ensure(ctx, A.pt_keys, pcap + 1, &pk));
  RC(ensure(ctx, A.pt_vals, pcap + 1, &pv));
  RC(ensure(ctx, A.pv_keys, vcap + 1, &vk));
  RC(ensure(ctx, A.pv_vals, vcap + 1, &vv));
  RC(ensure(ctx, A.d_prev, std::max<uint64_t>(n_prev, 1), &dp));
  // paged_host_words (ckpt.cpp:59-68): buffers back to back, zero tail
  uint64_t off = 0;
  for (uint64_t i = 0; i < nbufs; ++i) {
    if (words[i])
      CK(cudaMemcpyAsync(img + off, bufs[i], words[i] * 8, cudaMemcpyHostToDevice, ctx->stream));
    off += words[i] * 8;
  }
  if (npages * kPage > off) CK(cudaMemsetAsync(img + off, 0, npages * kPage - off, ctx->stream));
  const uint64_t one[3] = {0, npages * kPage, npages};
  CK(cudaMemcpyAsync(da, &one[0], 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(db, &one[1], 8, cudaMemcpyHostToDevice, ctx->stream));
  const uint64_t cs[2] = {0, npages};
  CK(cudaMemcpyAsync(dc, cs, 16, cudaMemcpyHostToDevice, ctx->stream));
  if (n_prev) CK(cudaMemcpyAsync(dp, prev, n_prev * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(cnt, 0, 16, ctx->stream));
  // K1: one "buffer" over the paged image, page == chunk == 4 KiB -> digest_of_words(page)
  const GridDev g{da, db, dc, 1u, npages, 12u, 12u};
  CKL(snap::launch_hash(img, g, dd, nullptr, nullptr, ctx->stream));
  const TableDev pt{pk, pv, pcap - 1}, vt{vk, vv, vcap - 1};
  CKL(snap::launch_table_clear(pt, ctx->stream));
  if (n_prev) {
    CKL(snap::launch_table_clear(vt, ctx->stream));
    CKL(snap::launch_table_insert_min(vt, dp, n_prev, 0, ctx->stream));
  }
  const TableDev kn{P<unsigned long long>(ctx->kn_keys), P<unsigned long long>(ctx->kn_vals),
                    ctx->kn_mask};
  CKL(snap::launch_page_classify(pt, kn, ctx->kn_count > 0, vt, n_prev > 0, dd, npages,
                                 slot, fl, cnt, ctx->stream));
  unsigned long long c[2];
  CK(cudaMemcpyAsync(c, cnt, 16, cudaMemcpyDeviceToHost, ctx->stream));
  if (page_digests)
    CK(cudaMemcpyAsync(page_digests, dd, npages * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (flags) CK(cudaMemcpyAsync(flags, fl, npages, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // `one`, `cs` die here
  out.upload_bytes = c[0] * kPage;
  out.s_cr_inc = c[1] * kPage;
  if (st) *st = out;
  return SNAP_OK;
}

int snap_validate_window(const snap_window_record* recs, uint64_t n, char* reason, uint64_t cap) {
  if (!recs && n) return SNAP_EINVAL;
  auto say = [&](const std::string& m) {
    if (reason && cap) {
      const size_t k = std::min<size_t>(m.size(), size_t(cap - 1));
      std::memcpy(reason, m.data(), k);
      reason[k] = 0;
    }
    return 0;
  };
  if (reason && cap) reason[0] = 0;
  if (n <= 1) return 1;
  // std::map<RankId, ValidationRecord> iteration order: by rank; duplicates collapse
  std::map<int, const snap_window_record*> by;
  for (uint64_t i = 0; i < n; ++i) by[recs[i].rank] = &recs[i];
  if (by.size() <= 1) return 1;
  auto it = by.begin();
  const snap_window_record& ref = *it->second;
  const int ref_rank = it->first;
  for (++it; it != by.end(); ++it) {
    const snap_window_record& rec = *it->second;
    if (rec.n_mutations != ref.n_mutations)
      return say("mutation count differs between rank " + std::to_string(ref_rank) +
                 " and rank " + std::to_string(it->first));
    for (uint64_t k = 0; k < ref.n_mutations; ++k) {
      const snap_mutation& a = ref.mutations[k];
      const snap_mutation& b = rec.mutations[k];
      // the reference prints decimal after "0x" (std::to_string); kept verbatim
      if (a.addr != b.addr)
        return say("mutation addresses differ (0x" + std::to_string(a.addr) + " vs 0x" +
                   std::to_string(b.addr) + ")");
      if (a.bytes != b.bytes) return say("mutation sizes differ at addr " + std::to_string(a.addr));
      if (a.digest != b.digest)
        return say("mutation digests differ at addr " + std::to_string(a.addr));
    }
    bool same = rec.n_d2h == ref.n_d2h;
    for (uint64_t k = 0; same && k < 2 * ref.n_d2h; ++k) same = rec.d2h[k] == ref.d2h[k];
    if (!same) return say("in-window d2h copies differ across ranks");
  }
  return 1;
}

}  // extern "C"
