// ctx.h — the snap_ctx definition and host helpers shared by the C-ABI
// translation units (capi.cpp, splice_host.cpp).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "snap_internal.h"

using snap::GridDev;
using snap::TableDev;

struct SpliceState;
struct WindowState;
struct LocalGroup;

// Communicator collectives (comm.cpp): NCCL or the in-process group.
enum CommType { kCommU8, kCommI32, kCommU32, kCommU64, kCommF32 };
enum CommOp { kCommSum, kCommMax, kCommMin };
// sliced ranks per GPU in one fixed-order allreduce call
constexpr uint32_t kArMaxLocal = 16;

struct DevMem {
  void* p = nullptr;
  size_t cap = 0;
};

// Per-kernel-class CUDA event pairs, recorded on the ctx stream when enabled
// (bench.py reads the live duration of the dominant kernel from these).
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
};

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
  DevMem d_addr, d_bytes, d_cstart, d_lens, d_dig, d_bufdig, d_chunk_buf, d_chunk_addr;
  GridDev grid;
  bool hashed = false;

  // dedup table (per snapshot) and known set (store index)
  DevMem dd_keys, dd_vals, dd_slot;
  uint64_t dd_mask = 0;
  // the dedup table / select scan state are left empty by the resolve pass;
  // dd_clean_mask / scan_clean_words = the extents known to be empty
  bool dd_clean = false;
  uint64_t dd_clean_mask = 0, scan_clean_words = 0;
  bool k1_inserted = false;  // the last K1 (single-GPU snapshot) did the K2 insert
  bool spec_next_done = false;  // the selection scan wrote the next speculative layout
  DevMem scan2;              // scan state of the per-writer shard scans
  DevMem kn_keys, kn_vals, kn_list;
  uint64_t kn_mask = 0, kn_count = 0;

  // selection over the (local or global) canonical chunk vector
  DevMem scan, sel, owner, offsets, sel_list, totals;
  uint64_t sel_n = 0;  // entries of the selection vectors (nchunks, or nranks * maxn)
  bool selected = false;
  DevMem staging;
  uint64_t staging_valid = 0;
  // speculative layout for the fused hash+compaction pass (double-buffered:
  // the gather/fix-up writes the actual layout as the next prediction)
  DevMem d_spec[2];
  int spec_cur = 0;
  bool spec_ready = false;
  bool spec_used = false;

  // cross-rank exchange (NCCL allgather of digest vectors) and striping;
  // the communicator is NCCL (one process per GPU) or an in-process group
  ncclComm_t comm = nullptr;
  LocalGroup* lgroup = nullptr;
  bool attached() const { return comm != nullptr || lgroup != nullptr; }
  int nranks = 1, rank = 0;
  bool exchanged = false;
  uint64_t maxn = 0;
  std::vector<uint64_t> counts;
  bool glens_valid = false;
  DevMem d_counts, d_gdig, d_glens, d_writer, d_shard_off, d_my_list, d_my_off, d_my_totals;
  // Exchange window = d_gdig: [nranks flag lines of 128 B][2 gathered digest
  // vectors of nranks * maxn, by epoch parity]. Every rank maps every peer's
  // window (CUDA IPC); K1 stores its digests into all of them (fused exchange).
  std::vector<void*> xpeer;   // [nranks] window bases (own = d_gdig.p)
  DevMem d_xdig, d_xflag, d_xh;
  bool xwin_ready = false;    // peers mapped for the current grid
  bool k1_fanout = false;     // K1 stored the digests of the coming exchange
  uint64_t xepoch = 0;        // exchanges done (gathered vector = parity xepoch & 1)

  // verify / restore scratch
  DevMem d_dig2, d_expect, d_nbad, d_srcoff;
  // verified restore: set to 1 by any CTA that sees a digest mismatch (mapped
  // pinned host word; the success path needs no memset and no read-back copy)
  unsigned int* h_badflag = nullptr;
  bool k1_insert_now = false;  // this snapshot's K1 does the K2 insert (hash_fused)
  // the verified restore's launch as an instantiated CUDA graph, reused while its
  // parameters (grid, image, offsets, digests) stay the same
  cudaGraphExec_t rv_exec = nullptr;
  std::vector<uint8_t> rv_key;
  int rv_launches = 0;
  unsigned int* d_badflag = nullptr;
  DevMem d_vbad;  // its mismatch counter, zero between calls

  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  Prof prof;
  SpliceState* splice = nullptr;
  WindowState* win = nullptr;  // auxiliary grid + open window snapshots (window.cpp)

  // host-buffer pipeline (snap_snapshot_host): copy streams, events, host
  // mirror of the speculative layout, fix-up list
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> pipe_ev;
  std::vector<uint64_t> h_spec;
  bool h_spec_valid = false;
  DevMem d_moved;

  // resize / reshard: peer ranks' staging shards mapped over CUDA IPC
  std::vector<void*> peer_staging;  // [nranks]; own rank = local staging
  std::vector<bool> peer_opened;    // mapped through cudaIpcOpenMemHandle (closed on release)
  DevMem d_peers;
  bool shard_offsets_all = false;   // d_shard_off valid for every writer
  // multi-rank step: global staging offsets (offsets/sel_list/totals) not yet
  // computed from the step's owners (global_offsets() does it on demand)
  bool global_offsets_pending = false;
  // snap_snapshot asks the single-GPU selection to do the K3 fix-up too
  // (fixup_request); fixup_done tells compact_impl nothing is left to copy
  bool fixup_request = false, fixup_done = false;
  DevMem d_tmaps;  // per-buffer TMA tensor maps of the installed grid
  // predicted staging bytes (multi-rank shards are sized to the prediction and
  // grown on demand instead of reserving a whole image per GPU)
  uint64_t spec_bytes = 0;
  // fixed-order allreduce: every rank's arena + flag lines (peer memory)
  std::vector<void*> ar_peer_arena, ar_peer_flag;
  std::vector<bool> ar_opened;
  bool ar_ready = false;
  uint64_t ar_epoch = 0;
  DevMem d_arflag, d_arh, d_arrec, d_arptr, d_arcnt;
  // pinned slabs of the persist/load file path (allocated once, reused)
  uint8_t* io_pin[2] = {nullptr, nullptr};
  uint64_t io_pin_cap = 0;
};

inline int fail(snap_ctx* c, int code, const std::string& msg) {
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

// Counts kernels of the last launcher call and checks launch-configuration errors.
#define CKL(n)                                                                               \
  do {                                                                                       \
    ctx->launches += (n);                                                                    \
    cudaError_t e_ = cudaGetLastError();                                                     \
    if (e_ != cudaSuccess)                                                                   \
      return fail(ctx, SNAP_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

#define RC(x)             \
  do {                    \
    int rc_ = (x);        \
    if (rc_) return rc_;  \
  } while (0)

template <typename T>
inline int ensure(snap_ctx* ctx, DevMem& m, size_t count, T** out) {
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
inline int ensure_keep(snap_ctx* ctx, DevMem& m, size_t count, size_t keep, T** out) {
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

template <typename T>
inline T* P(DevMem& m) {
  return static_cast<T*>(m.p);
}

inline void release(DevMem& m) {
  if (m.p) cudaFree(m.p);
  m.p = nullptr;
  m.cap = 0;
}

inline bool pow2(uint64_t x) { return x && !(x & (x - 1)); }
inline uint32_t log2u(uint64_t x) {
  uint32_t s = 0;
  while ((1ull << s) < x) ++s;
  return s;
}
// GridDev::chunk_buf of a grid: buffer index of every chunk, uploaded on the ctx
// stream (the caller synchronizes before `host` goes away)
// GridDev::chunk_buf / chunk_addr of a grid (buffer index and arena offset of every
// chunk), uploaded on the ctx stream (the caller synchronizes before `host` and
// `haddr` go away). SNAP_CHUNK_BUF=0 (A/B): neither, the kernels search cstart.
inline int upload_chunk_buf(snap_ctx* ctx, DevMem& m, DevMem& ma,
                            const std::vector<uint64_t>& cstart, const uint64_t* buf_addr,
                            uint32_t chunk_shift, std::vector<uint32_t>& host,
                            std::vector<uint64_t>& haddr, const uint32_t** out,
                            const uint64_t** out_addr) {
  static const bool off = std::getenv("SNAP_CHUNK_BUF") && std::getenv("SNAP_CHUNK_BUF")[0] == '0';
  *out = nullptr;
  *out_addr = nullptr;
  if (off) return SNAP_OK;
  const uint64_t nb = cstart.size() - 1, n = cstart[nb];
  host.resize(n);
  haddr.resize(n);
  for (uint64_t b = 0; b < nb; ++b)
    for (uint64_t c = cstart[b]; c < cstart[b + 1]; ++c) {
      host[c] = uint32_t(b);
      haddr[c] = buf_addr[b] + ((c - cstart[b]) << chunk_shift);
    }
  uint32_t* d;
  uint64_t* da;
  RC(ensure(ctx, m, std::max<uint64_t>(n, 1), &d));
  RC(ensure(ctx, ma, std::max<uint64_t>(n, 1), &da));
  if (n) {
    CK(cudaMemcpyAsync(d, host.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(da, haddr.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  }
  *out = d;
  *out_addr = da;
  return SNAP_OK;
}

inline uint64_t table_cap(uint64_t n) {
  uint64_t c = 1024;
  while (c < 2 * n) c <<= 1;
  return c;
}

// comm.cpp
int comm_allgather(snap_ctx* ctx, const void* send, void* recv, uint64_t count, CommType t);
int comm_allreduce(snap_ctx* ctx, const void* send, void* recv, uint64_t count, CommType t,
                   CommOp op);
bool comm_barrier(snap_ctx* ctx);
int ipc_handle(snap_ctx* ctx, void* dev_ptr, void* handle64);
int ipc_open(snap_ctx* ctx, const void* handle64, void** out, bool* opened);
void ipc_close(void* p, bool opened);
void ar_release(snap_ctx* ctx);
void local_group_leave(snap_ctx* ctx);
// capi.cpp: per-grid part of the exchange (collective)
int grid_exchange(snap_ctx* ctx);

// splice_host.cpp: seed the splice chunk cache with a rank's content (restore_job)
int splice_seed(snap_ctx* ctx, int rank, const uint8_t* image, const uint64_t* src_off,
                const uint64_t* dig);

int select_with_known(snap_ctx* ctx, const uint64_t* dig, const uint32_t* lens, uint64_t n,
                      TableDev kn, bool use_known, bool inserted = false,
                      uint64_t* spec_next = nullptr, const uint64_t* fix_spec = nullptr,
                      uint8_t* fix_staging = nullptr);

// Per-buffer TMA tensor maps for the hash-only TMA K1 (4 KiB pages; not built
// when a cp.async variant is forced). On any
// encode failure the grid simply keeps the cp.async kernel (tmaps = nullptr).
inline void build_tmaps(snap_ctx* ctx, DevMem& m, const uint64_t* addr, const uint64_t* bytes,
                        uint32_t n, GridDev& g) {
  g.tmaps = nullptr;
  g.tmaps64 = nullptr;
  g.tmaps64c = nullptr;
  g.gsched = nullptr;
  g.gs_bins = 0;
  if (!snap::hash_tma_selected() || g.page_shift != 12 || n == 0) return;
  // n per-buffer maps with 128-byte boxes (k_hash_tma), then the arena-wide
  // maps of k_hash_mma: 16 with 32-page boxes, 16 with chunk boxes (8-32 pages)
  const int ppc = 1 << (g.chunk_shift - g.page_shift);
  const bool chunk_maps = ppc >= 8 && ppc <= 32;
  // + the balanced k_hash_mma group schedule after the maps
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device) != cudaSuccess) sms = 0;
  std::vector<uint32_t> sched;
  g.mma_cw = snap::mma_cw_for(g.nchunks << (g.chunk_shift - g.page_shift), sms);
  const uint32_t bins =
      snap::mma_schedule(addr, bytes, n, g.page_shift, g.chunk_shift, sms, sched, g.mma_cw);
  std::vector<uint8_t> host(size_t(n) * 128 + 32 * 128 + sched.size() * 4);
  if (!sched.empty()) std::memcpy(host.data() + size_t(n) * 128 + 32 * 128, sched.data(), sched.size() * 4);
  if (snap::encode_tensor_maps(ctx->arena, addr, bytes, n, host.data(), 128) != 0) return;
  uint8_t* a64 = host.data() + size_t(n) * 128;
  if (snap::encode_arena_maps(ctx->arena, ctx->arena_bytes, 64, 32, a64) != 0) return;
  if (chunk_maps && snap::encode_arena_maps(ctx->arena, ctx->arena_bytes, 64, ppc, a64 + 16 * 128) != 0)
    return;
  uint8_t* d;
  if (ensure(ctx, m, host.size(), &d) != SNAP_OK) return;
  if (cudaMemcpyAsync(d, host.data(), host.size(), cudaMemcpyHostToDevice, ctx->stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess)
    return;
  g.tmaps = d;
  g.tmaps64 = d + size_t(n) * 128;
  if (chunk_maps) g.tmaps64c = d + size_t(n) * 128 + 16 * 128;
  g.gsched = bins ? reinterpret_cast<const uint32_t*>(d + size_t(n) * 128 + 32 * 128) : nullptr;
  g.gs_bins = bins;
}

inline int check_range(snap_ctx* ctx, uint64_t addr, uint64_t bytes) {
  if (addr > ctx->arena_bytes || bytes > ctx->arena_bytes - addr)
    return fail(ctx, SNAP_EINVAL, "range outside the arena");
  return SNAP_OK;
}

// ---- profiler ----
// kinds of snap_prof_read (SNAP_PROF_* in snap.h); kProfSwitch = one whole splice switch
enum { kProfHash = 0, kProfSelect, kProfCompact, kProfRestore, kProfGrad, kProfExchange, kProfSwitch, kProfN };

inline cudaEvent_t prof_event(snap_ctx* ctx) {
  Prof& p = ctx->prof;
  if (p.used == p.pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    p.pool.push_back(e);
  }
  return p.pool[p.used++];
}

struct ProfScope {
  snap_ctx* ctx;
  int kind;
  cudaEvent_t a = nullptr;
  ProfScope(snap_ctx* c, int k) : ctx(c), kind(k) {
    if (ctx->prof.on) {
      a = prof_event(ctx);
      if (a) cudaEventRecord(a, ctx->stream);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = prof_event(ctx);
      if (b) {
        cudaEventRecord(b, ctx->stream);
        ctx->prof.marks.push_back({kind, {a, b}});
      }
    }
  }
};
