// capi.cpp — the C ABI (include/snap.h): one snap_ctx per (job, GPU), the
// B200 analogue of proxy::ProxyServer (proxy.hpp:32-122) + vdev::Gpu memory
// (vdev.hpp:65-122). Host code only; every byte of device work is one of the
// sm_100a kernels in k_*.cu, issued on the ctx stream.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "snap_internal.h"

using snap::GridDev;
using snap::TableDev;

namespace {

struct DevMem {
  void* p = nullptr;
  size_t cap = 0;
};

struct Status {
  int code;
};

}  // namespace

struct snap_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint8_t* arena = nullptr;
  uint64_t arena_bytes = 0;
  std::string err;
  uint64_t launches = 0;

  // installed grid
  std::vector<snap_buf> bufs;
  snap_geom geom{4096, 65536};
  uint64_t nchunks = 0;
  uint64_t grid_bytes = 0;
  std::vector<uint64_t> h_cstart;
  std::vector<uint32_t> h_lens;
  DevMem d_addr, d_bytes, d_cstart, d_lens, d_dig, d_bufdig;
  GridDev grid;
  bool hashed = false;

  // dedup table (per snapshot) and known set (store index)
  DevMem dd_keys, dd_vals;
  uint64_t dd_mask = 0;
  DevMem kn_keys, kn_vals, kn_list;
  uint64_t kn_mask = 0, kn_count = 0;

  // selection
  DevMem scan, sel, owner, offsets, sel_list, totals;
  bool selected = false;
  DevMem staging;
  uint64_t staging_valid = 0;  // upper bound of staged bytes of the last compact

  // verify / restore scratch
  DevMem d_dig2, d_expect, d_nbad, d_srcoff;

  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

namespace {

int fail(snap_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(ctx, SNAP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CKN(call)                                                                        \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                               \
      return fail(ctx, SNAP_ECUDA, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// Checks the last launch of the ctx stream (launch-configuration errors).
#define CKL(n)                                                                           \
  do {                                                                                   \
    ctx->launches += (n);                                                                \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess)                                                               \
      return fail(ctx, SNAP_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
int ensure(snap_ctx* ctx, DevMem& m, size_t count, T** out) {
  size_t bytes = std::max<size_t>(count * sizeof(T), 256);
  if (bytes > m.cap) {
    if (m.p) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(m.p);
      m.p = nullptr;
      m.cap = 0;
    }
    cudaError_t e = cudaMalloc(&m.p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, e == cudaErrorMemoryAllocation ? SNAP_ENOMEM : SNAP_ECUDA,
                  std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    m.cap = bytes;
  }
  *out = static_cast<T*>(m.p);
  return SNAP_OK;
}

// Like ensure(), but keeps the first `keep` bytes when it has to grow.
template <typename T>
int ensure_keep(snap_ctx* ctx, DevMem& m, size_t count, size_t keep, T** out) {
  size_t bytes = std::max<size_t>(count * sizeof(T), 256);
  if (bytes > m.cap) {
    bytes = std::max(bytes, 2 * m.cap);
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, e == cudaErrorMemoryAllocation ? SNAP_ENOMEM : SNAP_ECUDA,
                  std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    if (m.p) {
      if (keep) cudaMemcpyAsync(p, m.p, keep, cudaMemcpyDeviceToDevice, ctx->stream);
      cudaStreamSynchronize(ctx->stream);
      cudaFree(m.p);
    }
    m.p = p;
    m.cap = bytes;
  }
  *out = static_cast<T*>(m.p);
  return SNAP_OK;
}

void release(DevMem& m) {
  if (m.p) cudaFree(m.p);
  m.p = nullptr;
  m.cap = 0;
}

bool pow2(uint64_t x) { return x && !(x & (x - 1)); }
uint32_t log2u(uint64_t x) {
  uint32_t s = 0;
  while ((1ull << s) < x) ++s;
  return s;
}
uint64_t table_cap(uint64_t n) {
  uint64_t c = 1024;
  while (c < 2 * n) c <<= 1;
  return c;
}

int check_range(snap_ctx* ctx, uint64_t addr, uint64_t bytes) {
  if (addr > ctx->arena_bytes || bytes > ctx->arena_bytes - addr)
    return fail(ctx, SNAP_EINVAL, "range outside the arena");
  return SNAP_OK;
}

int ensure_known(snap_ctx* ctx, uint64_t extra) {
  // grows (and rebuilds) the known-set table to keep load <= 1/2
  const uint64_t need = ctx->kn_count + extra;
  uint64_t* list;
  if (int rc = ensure_keep(ctx, ctx->kn_list, need, ctx->kn_count * 8, &list)) return rc;
  if (ctx->kn_mask && 2 * need <= ctx->kn_mask + 1) return SNAP_OK;
  const uint64_t cap = table_cap(need);
  unsigned long long *k, *v;
  if (int rc = ensure(ctx, ctx->kn_keys, cap + 1, &k)) return rc;
  if (int rc = ensure(ctx, ctx->kn_vals, cap + 1, &v)) return rc;
  ctx->kn_mask = cap - 1;
  TableDev t{k, v, ctx->kn_mask};
  CKL(snap::launch_table_clear(t, ctx->stream));
  CKL(snap::launch_table_insert_min(t, static_cast<uint64_t*>(ctx->kn_list.p), ctx->kn_count, 0,
                                    ctx->stream));
  return SNAP_OK;
}

int known_insert_dev(snap_ctx* ctx, const uint64_t* dev_digests, uint64_t n) {
  if (n == 0) return SNAP_OK;
  if (int rc = ensure_known(ctx, n)) return rc;
  uint64_t* list = static_cast<uint64_t*>(ctx->kn_list.p);
  CK(cudaMemcpyAsync(list + ctx->kn_count, dev_digests, n * 8, cudaMemcpyDeviceToDevice,
                     ctx->stream));
  TableDev t{static_cast<unsigned long long*>(ctx->kn_keys.p),
             static_cast<unsigned long long*>(ctx->kn_vals.p), ctx->kn_mask};
  CKL(snap::launch_table_insert_min(t, list + ctx->kn_count, n, 0, ctx->stream));
  ctx->kn_count += n;
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
  snap_ctx* ctx = nullptr;
  if (!out || arena_bytes == 0 || arena_bytes % 256) return SNAP_EINVAL;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return SNAP_ECUDA;
  }
  if (device < 0 || device >= ndev) return SNAP_EINVAL;
  ctx = new snap_ctx();
  ctx->device = device;
  auto bail = [&](int code) {
    snap_close(ctx);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(SNAP_ECUDA);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(SNAP_ECUDA);
  e = cudaMalloc(&ctx->arena, arena_bytes);
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
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  for (DevMem* m : {&ctx->d_addr, &ctx->d_bytes, &ctx->d_cstart, &ctx->d_lens, &ctx->d_dig,
                    &ctx->d_bufdig, &ctx->dd_keys, &ctx->dd_vals, &ctx->kn_keys, &ctx->kn_vals,
                    &ctx->kn_list, &ctx->scan, &ctx->sel, &ctx->owner, &ctx->offsets,
                    &ctx->sel_list, &ctx->totals, &ctx->staging, &ctx->d_dig2, &ctx->d_expect,
                    &ctx->d_nbad, &ctx->d_srcoff})
    release(*m);
  if (ctx->arena) cudaFree(ctx->arena);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
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

int snap_write(snap_ctx* ctx, uint64_t addr, const void* src, uint64_t bytes) {
  if (!ctx || (!src && bytes)) return SNAP_EINVAL;
  if (int rc = check_range(ctx, addr, bytes)) return rc;
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(ctx->arena + addr, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

int snap_read(snap_ctx* ctx, uint64_t addr, void* dst, uint64_t bytes) {
  if (!ctx || (!dst && bytes)) return SNAP_EINVAL;
  if (int rc = check_range(ctx, addr, bytes)) return rc;
  CK(cudaSetDevice(ctx->device));
  CK(cudaMemcpyAsync(dst, ctx->arena + addr, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

int snap_fill_mix64(snap_ctx* ctx, uint64_t addr, uint64_t bytes, uint64_t seed, uint64_t base) {
  if (!ctx || addr % 8 || bytes % 8) return fail(ctx, SNAP_EINVAL, "fill: unaligned range");
  if (int rc = check_range(ctx, addr, bytes)) return rc;
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
  if (int rc = ensure(ctx, ctx->d_srcoff, n, &d)) return rc;
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
    if (int rc = check_range(ctx, x.addr, x.bytes)) return rc;
    addr[b] = x.addr;
    bytes[b] = x.bytes;
    const uint64_t nc = (x.bytes + g.chunk_bytes - 1) / g.chunk_bytes;
    cstart[b + 1] = cstart[b] + nc;
    for (uint64_t k = 0; k < nc; ++k)
      lens.push_back(static_cast<uint32_t>(std::min<uint64_t>(g.chunk_bytes, x.bytes - k * g.chunk_bytes)));
    total += x.bytes;
  }
  if (cstart[n] >= (1ull << 32)) return fail(ctx, SNAP_EINVAL, "too many chunks");
  CK(cudaSetDevice(ctx->device));
  uint64_t *da, *db, *dc, *dd;
  uint32_t* dl;
  if (int rc = ensure(ctx, ctx->d_addr, n, &da)) return rc;
  if (int rc = ensure(ctx, ctx->d_bytes, n, &db)) return rc;
  if (int rc = ensure(ctx, ctx->d_cstart, n + 1, &dc)) return rc;
  if (int rc = ensure(ctx, ctx->d_lens, cstart[n], &dl)) return rc;
  if (int rc = ensure(ctx, ctx->d_dig, cstart[n], &dd)) return rc;
  CK(cudaMemcpyAsync(da, addr.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(db, bytes.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dc, cstart.data(), (n + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dl, lens.data(), lens.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // host vectors die here
  ctx->bufs.assign(bufs, bufs + n);
  ctx->geom = g;
  ctx->nchunks = cstart[n];
  ctx->grid_bytes = total;
  ctx->h_cstart = std::move(cstart);
  ctx->h_lens = std::move(lens);
  ctx->grid = GridDev{da, db, dc, static_cast<uint32_t>(n), ctx->nchunks, log2u(g.page_bytes),
                      log2u(g.chunk_bytes)};
  ctx->hashed = false;
  ctx->selected = false;
  if (n_chunks) *n_chunks = ctx->nchunks;
  return SNAP_OK;
}

int snap_hash(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CKL(snap::launch_hash(ctx->arena, ctx->grid, static_cast<uint64_t*>(ctx->d_dig.p), ctx->stream));
  ctx->hashed = true;
  ctx->selected = false;
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
    if (int rc = ensure(ctx, ctx->d_bufdig, ctx->bufs.size(), &bd)) return rc;
    CKL(snap::launch_buf_fold(ctx->grid, static_cast<uint64_t*>(ctx->d_dig.p), bd, ctx->stream));
    CK(cudaMemcpyAsync(buf_digests, bd, ctx->bufs.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (chunk_lens && ctx->nchunks) std::memcpy(chunk_lens, ctx->h_lens.data(), ctx->nchunks * 4);
  return SNAP_OK;
}

int snap_digest_ranges(snap_ctx* ctx, const snap_buf* bufs, uint64_t n, const snap_geom* geom,
                       uint64_t* out) {
  uint64_t nc = 0;
  if (int rc = snap_set_buffers(ctx, bufs, n, geom, &nc)) return rc;
  if (int rc = snap_hash(ctx)) return rc;
  return snap_get_digests(ctx, nullptr, nullptr, out);
}

// ---------------------------------------------------------------- K2

int snap_known_clear(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  ctx->kn_count = 0;
  if (ctx->kn_mask) {
    CK(cudaSetDevice(ctx->device));
    TableDev t{static_cast<unsigned long long*>(ctx->kn_keys.p),
               static_cast<unsigned long long*>(ctx->kn_vals.p), ctx->kn_mask};
    CKL(snap::launch_table_clear(t, ctx->stream));
  }
  return SNAP_OK;
}

int snap_known_add(snap_ctx* ctx, const uint64_t* digests, uint64_t n) {
  if (!ctx || (!digests && n)) return SNAP_EINVAL;
  if (n == 0) return SNAP_OK;
  CK(cudaSetDevice(ctx->device));
  uint64_t* tmp;
  if (int rc = ensure(ctx, ctx->d_dig2, n, &tmp)) return rc;
  CK(cudaMemcpyAsync(tmp, digests, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (int rc = known_insert_dev(ctx, tmp, n)) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

int snap_known_commit(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->hashed) return fail(ctx, SNAP_EINVAL, "known_commit before snap_hash");
  CK(cudaSetDevice(ctx->device));
  return known_insert_dev(ctx, static_cast<uint64_t*>(ctx->d_dig.p), ctx->nchunks);
}

int snap_select(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->hashed) return fail(ctx, SNAP_EINVAL, "select before snap_hash");
  CK(cudaSetDevice(ctx->device));
  const uint64_t n = ctx->nchunks;
  const uint64_t cap = table_cap(n);
  unsigned long long *k, *v;
  uint64_t *scan, *owner, *offsets, *totals;
  uint8_t* sel;
  uint32_t* list;
  if (int rc = ensure(ctx, ctx->dd_keys, cap + 1, &k)) return rc;
  if (int rc = ensure(ctx, ctx->dd_vals, cap + 1, &v)) return rc;
  if (int rc = ensure(ctx, ctx->scan, snap::scan_state_words(n) + 1, &scan)) return rc;
  if (int rc = ensure(ctx, ctx->sel, n, &sel)) return rc;
  if (int rc = ensure(ctx, ctx->owner, n, &owner)) return rc;
  if (int rc = ensure(ctx, ctx->offsets, n, &offsets)) return rc;
  if (int rc = ensure(ctx, ctx->sel_list, n, &list)) return rc;
  if (int rc = ensure(ctx, ctx->totals, 4, &totals)) return rc;
  ctx->dd_mask = cap - 1;
  TableDev dd{k, v, ctx->dd_mask};
  TableDev kn{static_cast<unsigned long long*>(ctx->kn_keys.p),
              static_cast<unsigned long long*>(ctx->kn_vals.p), ctx->kn_mask};
  const uint64_t* dig = static_cast<uint64_t*>(ctx->d_dig.p);
  CKL(snap::launch_table_clear(dd, ctx->stream));
  CKL(snap::launch_table_insert_min(dd, dig, n, 0, ctx->stream));
  CKL(snap::launch_select(dd, kn, ctx->kn_count > 0, dig, static_cast<uint32_t*>(ctx->d_lens.p), n,
                          scan, sel, owner, offsets, list, totals, ctx->stream));
  CKL(snap::launch_resolve_dups(sel, owner, offsets, n, ctx->stream));
  ctx->selected = true;
  return SNAP_OK;
}

int snap_get_selection(snap_ctx* ctx, uint8_t* sel, uint64_t* owner, uint64_t* offsets,
                       uint64_t* staged_bytes, uint64_t* staged_chunks) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->selected) return fail(ctx, SNAP_EINVAL, "get_selection before snap_select");
  CK(cudaSetDevice(ctx->device));
  const uint64_t n = ctx->nchunks;
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

// ---------------------------------------------------------------- K3

int snap_compact(snap_ctx* ctx) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->selected) return fail(ctx, SNAP_EINVAL, "compact before snap_select");
  CK(cudaSetDevice(ctx->device));
  uint8_t* st;
  if (int rc = ensure(ctx, ctx->staging, ctx->grid_bytes, &st)) return rc;
  CKL(snap::launch_gather(ctx->arena, ctx->grid, static_cast<uint32_t*>(ctx->d_lens.p),
                          static_cast<uint32_t*>(ctx->sel_list.p),
                          static_cast<uint64_t*>(ctx->totals.p),
                          static_cast<uint64_t*>(ctx->offsets.p), st, ctx->nchunks, ctx->stream));
  ctx->staging_valid = ctx->grid_bytes;
  return SNAP_OK;
}

int snap_snapshot(snap_ctx* ctx) {
  if (int rc = snap_hash(ctx)) return rc;
  if (int rc = snap_select(ctx)) return rc;
  return snap_compact(ctx);
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
  if (int rc = ensure(ctx, ctx->d_dig2, ctx->nchunks, &d2)) return rc;
  if (int rc = ensure(ctx, ctx->d_nbad, 1, &nbad)) return rc;
  CKL(snap::launch_hash(ctx->arena, ctx->grid, d2, ctx->stream));
  CKL(snap::launch_compare(d2, expect_dev, ctx->nchunks, nbad, ctx->stream));
  unsigned long long bad = 0;
  CK(cudaMemcpyAsync(&bad, nbad, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (bad)
    return fail(ctx, SNAP_EFAULT, "restore: digest verification failed on " + std::to_string(bad) +
                                      " chunk(s)");
  return SNAP_OK;
}

int snap_restore(snap_ctx* ctx, const void* image, uint64_t image_bytes, const uint64_t* src_off,
                 const uint64_t* expect_digests, int verify) {
  if (!ctx || (!src_off && ctx->nchunks) || (!image && ctx->nchunks)) return SNAP_EINVAL;
  for (uint64_t g = 0; g < ctx->nchunks; ++g)
    if (src_off[g] > image_bytes || ctx->h_lens[g] > image_bytes - src_off[g] || src_off[g] % 256)
      return fail(ctx, SNAP_EFAULT, "restore: chunk " + std::to_string(g) +
                                        " has no source in the image (missing blob)");
  CK(cudaSetDevice(ctx->device));
  uint64_t* so;
  if (int rc = ensure(ctx, ctx->d_srcoff, ctx->nchunks, &so)) return rc;
  CK(cudaMemcpyAsync(so, src_off, ctx->nchunks * 8, cudaMemcpyHostToDevice, ctx->stream));
  CKL(snap::launch_scatter(ctx->arena, ctx->grid, static_cast<uint32_t*>(ctx->d_lens.p),
                           static_cast<const uint8_t*>(image), so, ctx->stream));
  if (!verify) return snap_sync(ctx);
  const uint64_t* expect = static_cast<uint64_t*>(ctx->d_dig.p);
  if (expect_digests) {
    uint64_t* e;
    if (int rc = ensure(ctx, ctx->d_expect, ctx->nchunks, &e)) return rc;
    CK(cudaMemcpyAsync(e, expect_digests, ctx->nchunks * 8, cudaMemcpyHostToDevice, ctx->stream));
    expect = e;
  } else if (!ctx->hashed) {
    return fail(ctx, SNAP_EINVAL, "restore verify needs expect_digests or a prior snap_hash");
  }
  return verify_grid(ctx, expect);
}

int snap_restore_self(snap_ctx* ctx, int verify) {
  if (!ctx) return SNAP_EINVAL;
  if (!ctx->selected) return fail(ctx, SNAP_EINVAL, "restore_self needs a prior snapshot");
  if (ctx->kn_count)
    return fail(ctx, SNAP_EINVAL, "restore_self: incremental snapshot (known set) needs the "
                                  "older images; use snap_restore");
  CK(cudaSetDevice(ctx->device));
  CKL(snap::launch_scatter(ctx->arena, ctx->grid, static_cast<uint32_t*>(ctx->d_lens.p),
                           static_cast<const uint8_t*>(ctx->staging.p),
                           static_cast<uint64_t*>(ctx->offsets.p), ctx->stream));
  if (!verify) return SNAP_OK;
  return verify_grid(ctx, static_cast<uint64_t*>(ctx->d_dig.p));
}

// ---------------------------------------------------------------- K5

int snap_grad_sum(snap_ctx* ctx, int dtype, const uint64_t* src_addrs, uint32_t nsrc,
                  uint64_t dst_addr, uint64_t elems, int accumulate) {
  if (!ctx || !src_addrs || (dtype != SNAP_U64 && dtype != SNAP_F32) || nsrc == 0 || nsrc > 16)
    return fail(ctx, SNAP_EINVAL, "grad_sum: bad arguments (1..16 sources, u64|f32)");
  const uint64_t esz = dtype == SNAP_F32 ? 4 : 8;
  if (elems > ctx->arena_bytes / esz) return fail(ctx, SNAP_EINVAL, "grad_sum: size");
  for (uint32_t r = 0; r < nsrc; ++r) {
    if (src_addrs[r] % 16) return fail(ctx, SNAP_EINVAL, "grad_sum: sources must be 16-B aligned");
    if (int rc = check_range(ctx, src_addrs[r], elems * esz)) return rc;
  }
  if (dst_addr % 16) return fail(ctx, SNAP_EINVAL, "grad_sum: dst must be 16-B aligned");
  if (int rc = check_range(ctx, dst_addr, elems * esz)) return rc;
  CK(cudaSetDevice(ctx->device));
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
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  ctx->comm = nullptr;
  CKN(ncclCommInitRank(&ctx->comm, nranks, id, rank));
  ctx->nranks = nranks;
  ctx->rank = rank;
  return SNAP_OK;
}

int snap_allreduce(snap_ctx* ctx, int dtype, uint64_t addr, uint64_t elems) {
  if (!ctx || !ctx->comm) return fail(ctx, SNAP_EINVAL, "allreduce: no communicator");
  const uint64_t esz = dtype == SNAP_F32 ? 4 : 8;
  if (int rc = check_range(ctx, addr, elems * esz)) return rc;
  CK(cudaSetDevice(ctx->device));
  CKN(ncclAllReduce(ctx->arena + addr, ctx->arena + addr, elems,
                    dtype == SNAP_F32 ? ncclFloat32 : ncclUint64, ncclSum, ctx->comm, ctx->stream));
  return SNAP_OK;
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

}  // extern "C"
