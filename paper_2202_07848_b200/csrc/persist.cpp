// persist.cpp — the on-disk format of a snapshot.
//
//   <dir>/blobs/<2hex>/<16hex>   one file per blob, content = the blob's bytes
//                                (BlobStore::persist, ckpt.cpp:42-52; name from
//                                BlobStore::blob_rel_path, ckpt.cpp:35-40)
//   <dir>/layout.<rank>.snapl    binary layout of one rank: header, buffer records
//                                (DevRec, ckpt.hpp:64-71), chunk digests, FNV trailer
//   <dir>/manifest.dev.<rank>.json  the same as readable JSON, with the field names
//                                of Manifest::to_json's device section (ckpt.cpp:194-262)
//
// Blobs are chunks: the name is the chunk digest of the installed geometry. With
// page_bytes == chunk_bytes that digest is digest_of_words(content) (sim.hpp:67-70),
// so the files are byte-identical to what the reference's BlobStore writes.
//
// Data path: the staged bytes (this rank's selection, or its shard of a multi-rank
// snapshot) leave the device through two pinned slabs on the D2H stream while a
// pool of writer threads turns the previous slab into files; snap_load runs the
// mirror image (reader threads fill a pinned slab, H2D on the copy stream, next
// slab fills meanwhile) and finishes with the K4 scatter + K1 verification of
// snap_restore.
#include <fcntl.h>
#include <sys/stat.h>
#include <sys/types.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cerrno>
#include <filesystem>
#include <functional>
#include <mutex>
#include <thread>
#include <unordered_map>

#include "ctx.h"

namespace {

constexpr uint64_t kLayoutMagic = 0x314c50414e53ull;  // "SNAPL1"
constexpr uint32_t kLayoutVersion = 1;
constexpr uint64_t kSlab = 64ull << 20;

struct LayoutHdr {
  uint64_t magic;
  uint32_t version;
  int32_t rank;
  uint32_t page_bytes, chunk_bytes;
  uint64_t nbufs, nchunks;
};
struct LayoutRec {  // DevRec {slot, addr, words, cat, digest} + rank, flags, exact bytes
  uint32_t rank;
  int32_t slot;
  uint64_t addr, bytes;
  int32_t cat;
  uint32_t flags;
  uint64_t digest;
};
static_assert(sizeof(LayoutHdr) == 40 && sizeof(LayoutRec) == 40, "layout record sizes");

// FNV-1a over bytes: integrity trailer of the layout file (same function as sim.hpp:55-65)
uint64_t fnv_bytes(const void* p, size_t n, uint64_t h = 0xcbf29ce484222325ull) {
  const uint8_t* b = static_cast<const uint8_t*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

struct Blob {
  uint64_t digest, off;  // offset in the staging image (persist) / load image (load)
  uint32_t len;
};

struct Errors {
  std::mutex mu;
  std::atomic<int> code{0};
  std::string msg;
  void set(int c, const std::string& m) {
    std::lock_guard<std::mutex> g(mu);
    if (!code.load()) {
      msg = m;
      code.store(c);
    }
  }
};

int pick_threads(int n) {
  if (n > 0) return std::min(n, 64);
  const unsigned hc = std::thread::hardware_concurrency();
  return int(std::max(1u, std::min(hc ? hc : 1u, 16u)));
}

// f(i) for i in [0, n) on `threads` threads, dynamic blocks of 16
void parallel_for(uint64_t n, int threads, const std::function<void(uint64_t)>& f) {
  if (threads <= 1 || n < 32) {
    for (uint64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<uint64_t> next{0};
  std::vector<std::thread> ts;
  const int t = int(std::min<uint64_t>(uint64_t(threads), (n + 15) / 16));
  for (int k = 0; k < t; ++k)
    ts.emplace_back([&] {
      for (;;) {
        const uint64_t i0 = next.fetch_add(16);
        if (i0 >= n) return;
        for (uint64_t i = i0; i < std::min(n, i0 + 16); ++i) f(i);
      }
    });
  for (auto& th : ts) th.join();
}

std::string rel_path(uint64_t d) {
  char b[40];
  snap_blob_rel_path(d, b, sizeof b);
  return b;
}

bool write_all(int fd, const uint8_t* p, size_t n) {
  while (n) {
    const ssize_t w = ::write(fd, p, n);
    if (w < 0) {
      if (errno == EINTR) continue;
      return false;
    }
    p += w;
    n -= size_t(w);
  }
  return true;
}

int put_file(const std::string& path, const void* p, size_t n, bool skip_existing);

// Blob files: a file already present with the blob's size counts as present
// (one stat, like a non-fresh BlobStore::put); otherwise the blob is written to
// a temp file in the same directory and renamed into place, so a crash never
// leaves a torn file under the content-addressed name (a wrong-size file left
// by an older writer is rewritten). Returns 1 written, 0 present, -errno.
int put_blob(const std::string& path, const void* p, size_t n) {
  struct stat sb;
  if (::stat(path.c_str(), &sb) == 0 && S_ISREG(sb.st_mode) && uint64_t(sb.st_size) == n) return 0;
  return put_file(path, p, n, false);
}

// Layout / manifest files: tmp in the same directory + rename (atomic replace).
int put_file(const std::string& path, const void* p, size_t n, bool skip_existing) {
  struct stat sb;
  if (skip_existing && ::stat(path.c_str(), &sb) == 0) return 0;
  const std::string tmp = path + ".tmp." + std::to_string(::getpid()) + "." +
                          std::to_string(std::hash<std::thread::id>()(std::this_thread::get_id()));
  const int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (fd < 0) return -errno;
  const bool ok = write_all(fd, static_cast<const uint8_t*>(p), n);
  const int e = errno;
  ::close(fd);
  if (!ok) {
    ::unlink(tmp.c_str());
    return -e;
  }
  if (::rename(tmp.c_str(), path.c_str()) != 0) {
    const int e2 = errno;
    ::unlink(tmp.c_str());
    return -e2;
  }
  return 1;
}

// the ctx's two pinned slabs, grown to `cap` bytes on first use
int io_slabs(snap_ctx* ctx, uint64_t cap, uint8_t** p) {
  if (cap > ctx->io_pin_cap) {
    for (uint8_t*& q : ctx->io_pin)
      if (q) {
        cudaFreeHost(q);
        q = nullptr;
      }
    ctx->io_pin_cap = 0;
    for (uint8_t*& q : ctx->io_pin) {
      cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&q), cap, 0);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, SNAP_ENOMEM, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
      }
    }
    ctx->io_pin_cap = cap;
  }
  p[0] = ctx->io_pin[0];
  p[1] = ctx->io_pin[1];
  return SNAP_OK;
}

// SNAP_PERSIST_TRACE=1: phase times of persist/load on stderr
struct Trace {
  bool on;
  std::chrono::steady_clock::time_point t0;
  Trace() : on(std::getenv("SNAP_PERSIST_TRACE") != nullptr), t0(std::chrono::steady_clock::now()) {}
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[snap persist] %-24s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

// Writes the blobs of one contiguous image range [base, base + span) held at `src`.
void write_range(const std::string& root, const Blob* b, uint64_t n, const uint8_t* src,
                 uint64_t base, int threads, std::atomic<uint8_t>* made, std::atomic<uint64_t>& wr,
                 std::atomic<uint64_t>& pres, std::atomic<uint64_t>& bytes, Errors& err) {
  parallel_for(n, threads, [&](uint64_t i) {
    if (err.code.load()) return;
    const Blob& x = b[i];
    const unsigned pre = unsigned(x.digest >> 56);
    if (!made[pre].load(std::memory_order_acquire)) {
      char sub[8];
      std::snprintf(sub, sizeof sub, "/%02x", pre);
      const std::string d = root + "/blobs" + sub;
      if (::mkdir(d.c_str(), 0755) != 0 && errno != EEXIST) {
        err.set(SNAP_EINVAL, "persist: mkdir " + d + ": " + std::strerror(errno));
        return;
      }
      made[pre].store(1, std::memory_order_release);
    }
    const std::string path = root + "/" + rel_path(x.digest);
    const int r = put_blob(path, src + (x.off - base), x.len);
    if (r < 0) {
      err.set(SNAP_EINVAL, "persist: write " + path + ": " + std::strerror(-r));
      return;
    }
    if (r) {
      wr.fetch_add(1);
      bytes.fetch_add(x.len);
    } else {
      pres.fetch_add(1);
    }
  });
}

// groups blobs (sorted by offset) into slabs of at most kSlab image bytes
std::vector<std::pair<uint64_t, uint64_t>> slabs_of(const std::vector<Blob>& b, uint64_t slab) {
  std::vector<std::pair<uint64_t, uint64_t>> s;  // [first, last) blob index
  uint64_t i = 0;
  while (i < b.size()) {
    uint64_t j = i + 1;
    while (j < b.size() && b[j].off + b[j].len - b[i].off <= slab) ++j;
    s.push_back({i, j});
    i = j;
  }
  return s;
}

int ensure_copy_streams(snap_ctx* ctx) {
  if (!ctx->h2d) CK(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
  if (!ctx->d2h) CK(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
  for (int k = int(ctx->pipe_ev.size()); k < 2; ++k) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->pipe_ev.push_back(e);
  }
  return SNAP_OK;
}

std::string json_layout(const snap_ctx* ctx, int rank, const std::vector<uint64_t>& bufdig,
                        uint64_t layout_digest, const snap_persist_stats& st, uint64_t s_g,
                        uint64_t staged_bytes) {
  std::string j;
  char t[512];
  std::snprintf(t, sizeof t,
                "{\n  \"version\": 1,\n  \"format\": \"snap-b200/dev\",\n  \"rank\": %d,\n"
                "  \"geometry\": {\"page_bytes\": %u, \"chunk_bytes\": %u},\n"
                "  \"layout\": \"layout.%d.snapl\",\n  \"layout_digest\": %llu,\n"
                "  \"chunks\": %llu,\n  \"blobs\": %llu,\n",
                rank, ctx->geom.page_bytes, ctx->geom.chunk_bytes, rank,
                (unsigned long long)layout_digest, (unsigned long long)st.layout_chunks,
                (unsigned long long)st.layout_blobs);
  j += t;
  std::snprintf(t, sizeof t,
                "  \"sizes\": {\"s_g\": %llu, \"upload_bytes\": %llu, \"dump_d2h_max\": %llu, "
                "\"total_blob_bytes\": %llu},\n  \"dev\": [",
                (unsigned long long)s_g, (unsigned long long)st.bytes,
                (unsigned long long)staged_bytes, (unsigned long long)st.layout_bytes);
  j += t;
  for (size_t b = 0; b < ctx->bufs.size(); ++b) {
    const snap_buf& x = ctx->bufs[b];
    std::snprintf(t, sizeof t,
                  "%s\n    {\"rank\": %u, \"slot\": %d, \"addr\": %llu, \"words\": %llu, "
                  "\"bytes\": %llu, \"cat\": %d, \"digest\": %llu}",
                  b ? "," : "", x.rank, x.slot, (unsigned long long)x.addr,
                  (unsigned long long)(x.bytes / 8), (unsigned long long)x.bytes, x.cat,
                  (unsigned long long)bufdig[b]);
    j += t;
  }
  j += "\n  ]\n}\n";
  return j;
}

}  // namespace

extern "C" int snap_blob_rel_path(uint64_t digest, char* out, uint64_t cap) {
  if (!out || cap < 32) return SNAP_EINVAL;
  std::snprintf(out, size_t(cap), "blobs/%02x/%016llx", unsigned(digest >> 56),
                static_cast<unsigned long long>(digest));
  return SNAP_OK;
}

extern "C" int snap_persist(snap_ctx* ctx, const char* dir, const void* host_image,
                            uint64_t host_bytes, int nthreads, snap_persist_stats* stats) {
  if (!ctx) return SNAP_EINVAL;
  return snap_persist_rank(ctx, dir, ctx->rank, host_image, host_bytes, nthreads, stats);
}

extern "C" int snap_persist_rank(snap_ctx* ctx, const char* dir, int layout_rank,
                                 const void* host_image, uint64_t host_bytes, int nthreads,
                                 snap_persist_stats* stats) {
  if (!ctx || !dir || layout_rank < 0) return SNAP_EINVAL;
  if (!ctx->selected) return fail(ctx, SNAP_EINVAL, "persist needs a prior snapshot");
  const int threads = pick_threads(nthreads);
  const uint64_t nch = ctx->nchunks;
  Trace tr;

  // 1. this rank's blobs (digest, staging offset, length) and the layout digests
  std::vector<uint64_t> dig(nch), bufdig(ctx->bufs.size());
  RC(snap_get_digests(ctx, dig.data(), nullptr, bufdig.data()));
  std::vector<Blob> blobs;
  uint64_t s_g = 0, staged = 0;
  if (ctx->attached() && ctx->exchanged) {
    uint64_t n = 0;
    RC(snap_global_info(ctx, &n, nullptr));
    std::vector<uint64_t> gdig(n), soff(n);
    std::vector<uint32_t> glen(n);
    std::vector<int32_t> writer(n);
    RC(snap_get_global_digests(ctx, gdig.data(), glen.data()));
    RC(snap_get_shard(ctx, writer.data(), soff.data(), &staged, nullptr));
    for (uint64_t g = 0; g < n; ++g) {
      if (writer[g] >= 0) s_g += glen[g];
      if (writer[g] == ctx->rank) blobs.push_back({gdig[g], soff[g], glen[g]});
    }
  } else {
    std::vector<uint8_t> sel(nch);
    std::vector<uint64_t> off(nch);
    RC(snap_get_selection(ctx, sel.data(), nullptr, off.data(), &staged, nullptr));
    for (uint64_t g = 0; g < nch; ++g)
      if (sel[g]) blobs.push_back({dig[g], off[g], ctx->h_lens[g]});
    s_g = staged;
  }
  std::sort(blobs.begin(), blobs.end(), [](const Blob& a, const Blob& b) { return a.off < b.off; });
  tr.mark("selection to host");
  const uint64_t image = blobs.empty() ? 0 : blobs.back().off + blobs.back().len;
  if (host_image && host_bytes < image)
    return fail(ctx, SNAP_EINVAL, "persist: host image smaller than the staged bytes");
  if (!host_image && image > ctx->staging.cap)
    return fail(ctx, SNAP_EINTERNAL, "persist: staging image missing");

  // 2. directories
  std::error_code ec;
  const std::string root(dir), blobdir = root + "/blobs";
  std::filesystem::create_directories(blobdir, ec);
  if (ec) return fail(ctx, SNAP_EINVAL, "persist: cannot create " + blobdir + ": " + ec.message());
  std::atomic<uint8_t> made[256];
  for (auto& m : made) m.store(0);

  // 3. blobs: from the host image, or streamed out of HBM through pinned slabs
  Errors err;
  std::atomic<uint64_t> wr{0}, pres{0}, bytes{0};
  if (host_image || blobs.empty()) {
    write_range(root, blobs.data(), blobs.size(), static_cast<const uint8_t*>(host_image), 0,
                threads, made, wr, pres, bytes, err);
  } else {
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));  // staging complete
    const auto sl = slabs_of(blobs, kSlab);
    uint64_t cap = 0;
    for (auto [a, b] : sl) cap = std::max(cap, blobs[b - 1].off + blobs[b - 1].len - blobs[a].off);
    uint8_t* pin[2];
    RC(io_slabs(ctx, cap, pin));
    RC(ensure_copy_streams(ctx));
    tr.mark("pinned slabs");
    const uint8_t* st = static_cast<const uint8_t*>(ctx->staging.p);
    auto issue = [&](size_t k) -> cudaError_t {
      const auto [a, b] = sl[k];
      const uint64_t base = blobs[a].off, span = blobs[b - 1].off + blobs[b - 1].len - base;
      cudaError_t e = cudaMemcpyAsync(pin[k & 1], st + base, span, cudaMemcpyDeviceToHost, ctx->d2h);
      if (e == cudaSuccess) e = cudaEventRecord(ctx->pipe_ev[k & 1], ctx->d2h);
      return e;
    };
    CK(issue(0));
    for (size_t k = 0; k < sl.size() && !err.code.load(); ++k) {
      if (k + 1 < sl.size()) CK(issue(k + 1));  // buffer (k+1)&1 was written out at k-1
      CK(cudaEventSynchronize(ctx->pipe_ev[k & 1]));
      const auto [a, b] = sl[k];
      write_range(root, blobs.data() + a, b - a, pin[k & 1], blobs[a].off, threads, made, wr,
                  pres, bytes, err);
    }
    CK(cudaStreamSynchronize(ctx->d2h));
  }
  if (err.code.load()) return fail(ctx, err.code.load(), err.msg);
  tr.mark("blobs written");

  // 4. the rank's layout (binary, read by snap_load) and its JSON manifest
  snap_persist_stats st{};
  st.blobs = blobs.size();
  st.written = wr.load();
  st.present = pres.load();
  st.bytes = bytes.load();
  st.layout_chunks = nch;
  st.layout_bufs = ctx->bufs.size();
  {
    std::unordered_map<uint64_t, uint32_t> uniq;
    uniq.reserve(size_t(nch * 2));
    for (uint64_t g = 0; g < nch; ++g)
      if (uniq.emplace(dig[g], ctx->h_lens[g]).second) st.layout_bytes += ctx->h_lens[g];
    st.layout_blobs = uniq.size();
  }
  std::vector<uint8_t> lay(sizeof(LayoutHdr) + ctx->bufs.size() * sizeof(LayoutRec) + nch * 8 + 8);
  LayoutHdr h{kLayoutMagic, kLayoutVersion, layout_rank, ctx->geom.page_bytes, ctx->geom.chunk_bytes,
              uint64_t(ctx->bufs.size()), nch};
  std::memcpy(lay.data(), &h, sizeof h);
  uint8_t* q = lay.data() + sizeof h;
  for (size_t b = 0; b < ctx->bufs.size(); ++b, q += sizeof(LayoutRec)) {
    const snap_buf& x = ctx->bufs[b];
    LayoutRec r{x.rank, x.slot, x.addr, x.bytes, x.cat, x.flags, bufdig[b]};
    std::memcpy(q, &r, sizeof r);
  }
  if (nch) std::memcpy(q, dig.data(), nch * 8);
  q += nch * 8;
  const uint64_t trailer = fnv_bytes(lay.data(), size_t(q - lay.data()));
  std::memcpy(q, &trailer, 8);
  const std::string rk = std::to_string(layout_rank);
  int r = put_file(root + "/layout." + rk + ".snapl", lay.data(), lay.size(), false);
  if (r < 0) return fail(ctx, SNAP_EINVAL, std::string("persist: layout: ") + std::strerror(-r));
  const std::string js = json_layout(ctx, layout_rank, bufdig, trailer, st, s_g, staged);
  r = put_file(root + "/manifest.dev." + rk + ".json", js.data(), js.size(), false);
  if (r < 0) return fail(ctx, SNAP_EINVAL, std::string("persist: manifest: ") + std::strerror(-r));
  tr.mark("layout + manifest");
  if (stats) *stats = st;
  return SNAP_OK;
}

namespace {

struct Layout {
  LayoutHdr h{};
  std::vector<snap_buf> bufs;
  std::vector<uint64_t> dig;
};

// layout.<rank>.snapl: header, records, digests, FNV trailer (all checked)
int read_layout(snap_ctx* ctx, const std::string& root, int rank, Layout& L) {
  const std::string lp = root + "/layout." + std::to_string(rank) + ".snapl";
  std::vector<uint8_t> lay;
  const int fd = ::open(lp.c_str(), O_RDONLY | O_CLOEXEC);
  if (fd < 0) return fail(ctx, SNAP_EINVAL, "load: " + lp + ": " + std::strerror(errno));
  struct stat sb;
  if (::fstat(fd, &sb) != 0) {
    ::close(fd);
    return fail(ctx, SNAP_EINVAL, "load: stat " + lp);
  }
  lay.resize(size_t(sb.st_size));
  size_t got = 0;
  while (got < lay.size()) {
    const ssize_t n = ::pread(fd, lay.data() + got, lay.size() - got, off_t(got));
    if (n <= 0) break;
    got += size_t(n);
  }
  ::close(fd);
  if (got != lay.size()) return fail(ctx, SNAP_EINVAL, "load: short read of " + lp);
  LayoutHdr& h = L.h;
  if (lay.size() < sizeof h + 8) return fail(ctx, SNAP_EFAULT, "load: layout truncated");
  std::memcpy(&h, lay.data(), sizeof h);
  if (h.magic != kLayoutMagic || h.version != kLayoutVersion)
    return fail(ctx, SNAP_EINVAL, "load: not a snap layout (unknown version)");
  const uint64_t want = sizeof h + h.nbufs * sizeof(LayoutRec) + h.nchunks * 8 + 8;
  if (h.nbufs > (1ull << 32) || h.nchunks > (1ull << 40) || lay.size() != want)
    return fail(ctx, SNAP_EFAULT, "load: layout size mismatch");
  uint64_t trailer;
  std::memcpy(&trailer, lay.data() + want - 8, 8);
  if (fnv_bytes(lay.data(), size_t(want - 8)) != trailer)
    return fail(ctx, SNAP_EFAULT, "load: layout digest verification failed");
  L.bufs.resize(h.nbufs);
  const uint8_t* q = lay.data() + sizeof h;
  for (uint64_t b = 0; b < h.nbufs; ++b, q += sizeof(LayoutRec)) {
    LayoutRec r;
    std::memcpy(&r, q, sizeof r);
    L.bufs[b] = snap_buf{r.rank, r.slot, r.addr, r.bytes, r.cat, r.flags};
  }
  L.dig.resize(h.nchunks);
  if (h.nchunks) std::memcpy(L.dig.data(), q, h.nchunks * 8);
  return SNAP_OK;
}

// chunk lengths of a layout's grid (the same arithmetic as snap_set_buffers)
std::vector<uint32_t> layout_lens(const Layout& L) {
  std::vector<uint32_t> lens;
  for (const snap_buf& b : L.bufs)
    for (uint64_t o = 0; o < b.bytes; o += L.h.chunk_bytes)
      lens.push_back(uint32_t(std::min<uint64_t>(L.h.chunk_bytes, b.bytes - o)));
  return lens;
}

// distinct blobs in first-reference order, laid out 256-B aligned in one image;
// src[g] = image offset of chunk g's blob. Returns the image size.
uint64_t plan_image(const std::vector<uint64_t>& dig, const std::vector<uint32_t>& lens,
                    std::vector<Blob>& blobs, std::vector<uint64_t>& src) {
  std::unordered_map<uint64_t, uint64_t> at;  // digest -> image offset
  at.reserve(dig.size() * 2);
  src.assign(dig.size(), 0);
  uint64_t image = 0;
  for (uint64_t g = 0; g < dig.size(); ++g) {
    auto [it, fresh] = at.emplace(dig[g], image);
    if (fresh) {
      blobs.push_back({dig[g], image, lens[g]});
      image += (uint64_t(lens[g]) + 255) & ~255ull;
    }
    src[g] = it->second;
  }
  return image;
}

// blob files -> pinned slabs (reader threads) -> device image (copy stream).
// A missing, truncated or unreadable blob is SNAP_EFAULT (BlobStore::get).
int stream_blobs(snap_ctx* ctx, const std::string& root, int threads,
                 const std::vector<Blob>& blobs, uint8_t* dimg, uint64_t* bytes_read) {
  Errors err;
  std::atomic<uint64_t> rd{0};
  if (!blobs.empty()) {
    const auto sl = slabs_of(blobs, kSlab);
    uint64_t cap = 0;
    for (auto [a, b] : sl) cap = std::max(cap, blobs[b - 1].off + blobs[b - 1].len - blobs[a].off);
    uint8_t* pin[2];
    RC(io_slabs(ctx, cap, pin));
    RC(ensure_copy_streams(ctx));
    for (size_t k = 0; k < sl.size(); ++k) {
      if (k >= 2) CK(cudaEventSynchronize(ctx->pipe_ev[k & 1]));  // slab buffer free again
      const auto [a, b] = sl[k];
      const uint64_t base = blobs[a].off;
      uint8_t* dst = pin[k & 1];
      parallel_for(b - a, threads, [&](uint64_t i) {
        if (err.code.load()) return;
        const Blob& x = blobs[a + i];
        const std::string path = root + "/" + rel_path(x.digest);
        const int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
        if (fd < 0) {
          err.set(SNAP_EFAULT, "blob store: missing blob " + path);
          return;
        }
        struct stat sb;
        if (::fstat(fd, &sb) != 0 || uint64_t(sb.st_size) != x.len) {
          ::close(fd);
          err.set(SNAP_EFAULT, "blob store: blob " + path + " has the wrong size");
          return;
        }
        size_t got = 0;
        while (got < x.len) {
          const ssize_t n = ::pread(fd, dst + (x.off - base) + got, x.len - got, off_t(got));
          if (n <= 0) break;
          got += size_t(n);
        }
        ::close(fd);
        if (got != x.len) {
          err.set(SNAP_EFAULT, "blob store: short read of " + path);
          return;
        }
        rd.fetch_add(x.len);
      });
      if (err.code.load()) break;
      const uint64_t span = blobs[b - 1].off + blobs[b - 1].len - base;
      CK(cudaMemcpyAsync(dimg + base, dst, span, cudaMemcpyHostToDevice, ctx->h2d));
      CK(cudaEventRecord(ctx->pipe_ev[k & 1], ctx->h2d));
    }
    CK(cudaStreamSynchronize(ctx->h2d));
  }
  if (bytes_read) *bytes_read = rd.load();
  if (err.code.load()) return fail(ctx, err.code.load(), err.msg);
  return SNAP_OK;
}

// the ctx staging buffer as the load image (nothing in flight may still read it)
int load_image(snap_ctx* ctx, uint64_t bytes, uint8_t** dimg) {
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  RC(ensure(ctx, ctx->staging, bytes, dimg));
  ctx->selected = false;  // the staging image now holds loaded blobs
  ctx->staging_valid = 0;
  ctx->spec_ready = false;
  return SNAP_OK;
}

}  // namespace

extern "C" int snap_load(snap_ctx* ctx, const char* dir, int rank, int verify, int nthreads,
                         snap_persist_stats* stats) {
  if (!ctx || !dir) return SNAP_EINVAL;
  const int threads = pick_threads(nthreads);
  const std::string root(dir);
  Trace tr;
  Layout L;
  RC(read_layout(ctx, root, rank, L));
  tr.mark("layout read");
  // install the layout; distinct blobs in first-reference order
  snap_geom geom{L.h.page_bytes, L.h.chunk_bytes};
  uint64_t nch = 0;
  RC(snap_set_buffers(ctx, L.bufs.data(), L.bufs.size(), &geom, &nch));
  if (nch != L.h.nchunks) return fail(ctx, SNAP_EFAULT, "load: layout chunk count mismatch");
  std::vector<Blob> blobs;
  std::vector<uint64_t> src;
  const uint64_t image = plan_image(L.dig, ctx->h_lens, blobs, src);
  tr.mark("layout installed");
  if (stats) {  // the layout is installed from here on, even if a blob fails
    *stats = snap_persist_stats{};
    stats->layout_chunks = nch;
    stats->layout_bufs = L.bufs.size();
  }
  uint8_t* dimg;
  RC(load_image(ctx, image, &dimg));
  uint64_t rd = 0;
  RC(stream_blobs(ctx, root, threads, blobs, dimg, &rd));
  tr.mark("blobs read + H2D");
  if (stats) {
    stats->blobs = blobs.size();
    stats->bytes = rd;
    stats->layout_blobs = blobs.size();
    for (const Blob& x : blobs) stats->layout_bytes += x.len;
  }
  // K4 scatter to the recorded addresses (+ K1 verification against the layout digests)
  RC(snap_restore(ctx, dimg, image, src.data(), L.dig.data(), verify));
  tr.mark("K4 scatter + verify");
  // the layout's digests become the context's (verified against the restored
  // bytes when verify != 0): snap_get_digests works right after a load
  if (nch) {
    CK(cudaMemcpyAsync(ctx->d_dig.p, L.dig.data(), nch * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  ctx->hashed = true;
  return SNAP_OK;
}

extern "C" int snap_splice_load(snap_ctx* ctx, const char* dir, int layout_rank, int splice_rank,
                                int nthreads, snap_persist_stats* stats) {
  if (!ctx || !dir || splice_rank < 0) return SNAP_EINVAL;
  if (!ctx->splice) return fail(ctx, SNAP_EINVAL, "splice_load needs snap_splice_init");
  const int threads = pick_threads(nthreads);
  const std::string root(dir);
  Layout L;
  RC(read_layout(ctx, root, layout_rank, L));
  // the persisted content of every buffer is real content: none is pending here
  for (snap_buf& b : L.bufs) b.flags &= ~SNAP_BUF_PENDING;
  snap_geom geom{L.h.page_bytes, L.h.chunk_bytes};
  RC(snap_splice_set_rank(ctx, splice_rank, L.bufs.data(), L.bufs.size(), &geom));
  const std::vector<uint32_t> lens = layout_lens(L);
  if (lens.size() != L.dig.size()) return fail(ctx, SNAP_EFAULT, "load: layout chunk count mismatch");
  std::vector<Blob> blobs;
  std::vector<uint64_t> src;
  const uint64_t image = plan_image(L.dig, lens, blobs, src);
  uint8_t* dimg;
  RC(load_image(ctx, image, &dimg));
  uint64_t rd = 0;
  RC(stream_blobs(ctx, root, threads, blobs, dimg, &rd));
  RC(splice_seed(ctx, splice_rank, dimg, src.data(), L.dig.data()));
  if (stats) {
    *stats = snap_persist_stats{};
    stats->blobs = blobs.size();
    stats->bytes = rd;
    stats->layout_chunks = L.dig.size();
    stats->layout_bufs = L.bufs.size();
    stats->layout_blobs = blobs.size();
    for (const Blob& x : blobs) stats->layout_bytes += x.len;
  }
  return SNAP_OK;
}
