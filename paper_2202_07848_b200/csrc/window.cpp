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
};

struct WindowState {
  AuxGrid aux;
  // rank -> open snapshot addr -> (bytes, digest)   (ProxyWindow::open_snapshot)
  std::map<int, std::map<uint64_t, std::pair<uint64_t, uint64_t>>> open;
};

void window_release(snap_ctx* ctx) {
  WindowState* W = ctx->win;
  if (!W) return;
  for (DevMem* m : {&W->aux.d_addr, &W->aux.d_bytes, &W->aux.d_cstart, &W->aux.d_dig,
                    &W->aux.d_bufdig})
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
