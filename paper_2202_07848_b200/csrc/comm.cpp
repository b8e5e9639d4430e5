// comm.cpp — the device-level communicator of a ctx (the reference's
// CollectiveEngine world of one rank per GPU, collectives.cpp:37-59,147-154)
// and the fixed-order gradient allreduce built on peer memory.
//
// Two transports behind the same calls:
//  * NCCL (one process per GPU, snap_comm_init): allgather / allreduce over
//    NVLink; peer buffers (staging shards, arenas, flag lines) mapped through
//    CUDA IPC;
//  * an in-process group (snap_comm_init_local: several ctxs driven by threads
//    of one process, e.g. N ranks emulated on one GPU, the reference's own
//    whole-fleet-in-one-process model): collectives through host memory and a
//    host barrier; "IPC" handles of the same process resolve to the exporting
//    ctx's device pointer through a process-wide registry.
// Every collective is issued in the same order by every rank (snap.h).
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <memory>
#include <mutex>

#include "ctx.h"

struct LocalGroup {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  int refs = 0;
  std::vector<const void*> ptrs;
  std::vector<int> devices;

  bool broken = false;

  // false when a peer never arrived within the timeout (it failed before this
  // collective): the group is then broken for every member, like a NCCL error
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (broken) return false;
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    static const long secs = [] {
      const char* e = std::getenv("SNAP_LOCAL_TIMEOUT_S");
      return e && std::atol(e) > 0 ? std::atol(e) : 120L;
    }();
    if (!cv.wait_for(lk, std::chrono::seconds(secs), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

#define BARRIER(G)                                                                     \
  do {                                                                                 \
    if (!(G)->barrier())                                                               \
      return fail(ctx, SNAP_EINTERNAL, "in-process communicator: a peer rank did not " \
                                       "reach this collective (it failed or diverged)"); \
  } while (0)

namespace {

std::mutex g_reg_mu;
std::map<std::string, LocalGroup*> g_groups;  // rendezvous by key
// handle bytes -> device pointer of a buffer exported by this process
std::map<std::string, void*> g_ipc;

std::string hkey(const void* h) { return std::string(static_cast<const char*>(h), 64); }

}  // namespace

// ---------------------------------------------------------------- IPC

int ipc_handle(snap_ctx* ctx, void* dev_ptr, void* handle64) {
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  CK(cudaIpcGetMemHandle(&h, dev_ptr));
  std::memcpy(handle64, &h, 64);
  std::lock_guard<std::mutex> lk(g_reg_mu);
  g_ipc[hkey(handle64)] = dev_ptr;
  return SNAP_OK;
}

// A peer's buffer: the registry when the exporter lives in this process
// (cudaIpcOpenMemHandle refuses same-process handles), else CUDA IPC.
int ipc_open(snap_ctx* ctx, const void* handle64, void** out, bool* opened) {
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto it = g_ipc.find(hkey(handle64));
    if (it != g_ipc.end()) {
      *out = it->second;
      *opened = false;
      return SNAP_OK;
    }
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  CK(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  *opened = true;
  return SNAP_OK;
}

void ipc_close(void* p, bool opened) {
  if (p && opened) cudaIpcCloseMemHandle(p);
}

// ---------------------------------------------------------------- collectives

namespace {

size_t type_size(CommType t) {
  switch (t) {
    case kCommU8: return 1;
    case kCommI32: case kCommU32: case kCommF32: return 4;
    case kCommU64: return 8;
  }
  return 1;
}

ncclDataType_t nccl_type(CommType t) {
  switch (t) {
    case kCommU8: return ncclUint8;
    case kCommI32: return ncclInt32;
    case kCommU32: return ncclUint32;
    case kCommF32: return ncclFloat32;
    case kCommU64: return ncclUint64;
  }
  return ncclUint8;
}

template <typename T>
void reduce_into(T* acc, const T* x, uint64_t n, CommOp op) {
  for (uint64_t i = 0; i < n; ++i) {
    if (op == kCommSum)
      acc[i] = static_cast<T>(acc[i] + x[i]);
    else if (op == kCommMax)
      acc[i] = std::max(acc[i], x[i]);
    else
      acc[i] = std::min(acc[i], x[i]);
  }
}

}  // namespace

int comm_allgather(snap_ctx* ctx, const void* send, void* recv, uint64_t count, CommType t) {
  const uint64_t bytes = count * type_size(t);
  if (ctx->comm) {
    CKN(ncclAllGather(send, recv, count, nccl_type(t), ctx->comm, ctx->stream));
    return SNAP_OK;
  }
  LocalGroup* G = ctx->lgroup;
  if (!G) return fail(ctx, SNAP_EINTERNAL, "allgather without a communicator");
  CK(cudaStreamSynchronize(ctx->stream));
  G->ptrs[ctx->rank] = send;
  BARRIER(G);
  for (int q = 0; q < G->n; ++q) {
    uint8_t* dst = static_cast<uint8_t*>(recv) + q * bytes;
    if (dst != G->ptrs[q] && bytes)
      CK(cudaMemcpyAsync(dst, G->ptrs[q], bytes, cudaMemcpyDefault, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  BARRIER(G);  // no rank reuses its send buffer before every peer copied it
  return SNAP_OK;
}

int comm_allreduce(snap_ctx* ctx, const void* send, void* recv, uint64_t count, CommType t,
                   CommOp op) {
  if (ctx->comm) {
    const ncclRedOp_t o = op == kCommSum ? ncclSum : op == kCommMax ? ncclMax : ncclMin;
    CKN(ncclAllReduce(send, recv, count, nccl_type(t), o, ctx->comm, ctx->stream));
    return SNAP_OK;
  }
  LocalGroup* G = ctx->lgroup;
  if (!G) return fail(ctx, SNAP_EINTERNAL, "allreduce without a communicator");
  const uint64_t bytes = count * type_size(t);
  CK(cudaStreamSynchronize(ctx->stream));
  G->ptrs[ctx->rank] = send;
  BARRIER(G);
  // every rank reduces all contributions in rank order (the same bits everywhere)
  std::vector<uint8_t> acc(bytes), x(bytes);
  for (int q = 0; q < G->n; ++q) {
    CK(cudaMemcpy(q ? x.data() : acc.data(), G->ptrs[q], bytes, cudaMemcpyDefault));
    if (q == 0) continue;
    switch (t) {
      case kCommI32: reduce_into(reinterpret_cast<int32_t*>(acc.data()), reinterpret_cast<const int32_t*>(x.data()), count, op); break;
      case kCommU32: reduce_into(reinterpret_cast<uint32_t*>(acc.data()), reinterpret_cast<const uint32_t*>(x.data()), count, op); break;
      case kCommU64: reduce_into(reinterpret_cast<uint64_t*>(acc.data()), reinterpret_cast<const uint64_t*>(x.data()), count, op); break;
      case kCommF32: reduce_into(reinterpret_cast<float*>(acc.data()), reinterpret_cast<const float*>(x.data()), count, op); break;
      case kCommU8: reduce_into(acc.data(), x.data(), count, op); break;
    }
  }
  BARRIER(G);  // every rank has read every send buffer
  CK(cudaMemcpyAsync(recv, acc.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SNAP_OK;
}

bool comm_barrier(snap_ctx* ctx) { return ctx->lgroup ? ctx->lgroup->barrier() : true; }

// Releases the peer mappings of the fixed-order allreduce.
void ar_release(snap_ctx* ctx) {
  for (size_t q = 0; q < ctx->ar_peer_arena.size(); ++q)
    if (int(q) != ctx->rank) ipc_close(ctx->ar_peer_arena[q], ctx->ar_opened[2 * q]);
  for (size_t q = 0; q < ctx->ar_peer_flag.size(); ++q)
    if (int(q) != ctx->rank) ipc_close(ctx->ar_peer_flag[q], ctx->ar_opened[2 * q + 1]);
  ctx->ar_peer_arena.clear();
  ctx->ar_peer_flag.clear();
  ctx->ar_opened.clear();
  ctx->ar_ready = false;
}

void local_group_leave(snap_ctx* ctx) {
  LocalGroup* G = ctx->lgroup;
  if (!G) return;
  ctx->lgroup = nullptr;
  std::lock_guard<std::mutex> lk(g_reg_mu);
  if (--G->refs == 0) delete G;
}

namespace {

// Peer arenas + flag lines of every rank, mapped once per communicator
// (collective). Flag lines: [ready slot q][done slot q], 128 B each.
int ar_setup(snap_ctx* ctx) {
  if (ctx->ar_ready) return SNAP_OK;
  const int R = ctx->nranks;
  uint64_t* fl;
  RC(ensure(ctx, ctx->d_arflag, 2 * uint64_t(R) * 16, &fl));
  CK(cudaMemsetAsync(fl, 0, 2 * uint64_t(R) * 128, ctx->stream));
  ctx->ar_epoch = 0;
  uint8_t* xh;
  RC(ensure(ctx, ctx->d_arh, 128 * uint64_t(R) + 128, &xh));
  uint8_t mine[128];
  RC(ipc_handle(ctx, ctx->arena, mine));
  RC(ipc_handle(ctx, ctx->d_arflag.p, mine + 64));
  uint8_t* sendp = xh + 128 * uint64_t(R);
  CK(cudaMemcpyAsync(sendp, mine, 128, cudaMemcpyHostToDevice, ctx->stream));
  RC(comm_allgather(ctx, sendp, xh, 128, kCommU8));
  std::vector<uint8_t> all(128 * size_t(R));
  CK(cudaMemcpyAsync(all.data(), xh, all.size(), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->ar_peer_arena.assign(R, nullptr);
  ctx->ar_peer_flag.assign(R, nullptr);
  ctx->ar_opened.assign(2 * R, false);
  for (int q = 0; q < R; ++q) {
    if (q == ctx->rank) {
      ctx->ar_peer_arena[q] = ctx->arena;
      ctx->ar_peer_flag[q] = ctx->d_arflag.p;
      continue;
    }
    bool o1 = false, o2 = false;
    RC(ipc_open(ctx, all.data() + 128 * q, &ctx->ar_peer_arena[q], &o1));
    RC(ipc_open(ctx, all.data() + 128 * q + 64, &ctx->ar_peer_flag[q], &o2));
    ctx->ar_opened[2 * q] = o1;
    ctx->ar_opened[2 * q + 1] = o2;
  }
  if (ctx->lgroup) {
    // in-process ranks on different devices read each other directly
    for (int q = 0; q < R; ++q) {
      const int dq = ctx->lgroup->devices[q];
      if (dq == ctx->device) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, ctx->device, dq);
      if (!can) return fail(ctx, SNAP_EINVAL, "local group: devices without peer access");
      const cudaError_t e = cudaDeviceEnablePeerAccess(dq, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(ctx, SNAP_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      cudaGetLastError();
    }
  }
  ctx->ar_ready = true;
  return SNAP_OK;
}

}  // namespace

extern "C" {

int snap_comm_init_local(snap_ctx* ctx, int nranks, int rank, const char* key) {
  if (!ctx || !key || nranks < 1 || rank < 0 || rank >= nranks) return SNAP_EINVAL;
  if (ctx->attached())
    return fail(ctx, SNAP_EINVAL, "comm_init_local: destroy the current communicator first");
  CK(cudaSetDevice(ctx->device));
  LocalGroup* G;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto it = g_groups.find(key);
    if (it == g_groups.end()) {
      G = new LocalGroup();
      G->n = nranks;
      G->ptrs.assign(nranks, nullptr);
      G->devices.assign(nranks, -1);
      g_groups[key] = G;
    } else {
      G = it->second;
    }
    if (G->n != nranks) return fail(ctx, SNAP_EINVAL, "comm_init_local: group size mismatch");
    G->refs += 1;
    G->devices[rank] = ctx->device;
    if (G->refs == nranks) g_groups.erase(key);  // complete: the key can be reused
  }
  ctx->lgroup = G;
  if (!G->barrier()) {  // every member joined
    local_group_leave(ctx);
    return fail(ctx, SNAP_EINTERNAL, "comm_init_local: not every rank joined");
  }
  ctx->nranks = nranks;
  ctx->rank = rank;
  ctx->xepoch = 0;
  ctx->xwin_ready = false;
  ctx->k1_fanout = false;
  ctx->glens_valid = false;
  ctx->exchanged = false;
  ctx->spec_ready = false;
  return grid_exchange(ctx);
}

// Fixed-order device-level gradient allreduce (CollectiveEngine sum,
// collectives.cpp:137-154, with the north star's fixed-order fp32 mode).
int snap_allreduce_ordered(snap_ctx* ctx, int dtype, const uint32_t* keys, const uint64_t* src_addrs,
                           uint32_t nlocal, uint64_t dst_addr, uint64_t elems) {
  if (!ctx || !ctx->attached()) return fail(ctx, SNAP_EINVAL, "allreduce_ordered: no communicator");
  if (dtype != SNAP_U64 && dtype != SNAP_F32 && dtype != SNAP_BF16)
    return fail(ctx, SNAP_EINVAL, "allreduce_ordered: dtype u64 | f32 | bf16");
  if (nlocal > kArMaxLocal || (nlocal && (!keys || !src_addrs)))
    return fail(ctx, SNAP_EINVAL, "allreduce_ordered: at most 16 local sources");
  const uint64_t esz = dtype == SNAP_U64 ? 8 : dtype == SNAP_F32 ? 4 : 2;
  if (elems > ctx->arena_bytes / esz) return fail(ctx, SNAP_EINVAL, "allreduce_ordered: size");
  for (uint32_t i = 0; i < nlocal; ++i) {
    if (src_addrs[i] % 16) return fail(ctx, SNAP_EINVAL, "allreduce_ordered: 16-B aligned sources");
    RC(check_range(ctx, src_addrs[i], elems * esz));
  }
  if (dst_addr % 16) return fail(ctx, SNAP_EINVAL, "allreduce_ordered: 16-B aligned dst");
  RC(check_range(ctx, dst_addr, elems * esz));
  CK(cudaSetDevice(ctx->device));
  RC(ar_setup(ctx));
  const int N = ctx->nranks;
  // every GPU's record: [nlocal, dst, elems, (key, addr) x kArMaxLocal]
  constexpr uint64_t kRec = 3 + 2 * kArMaxLocal;
  uint64_t rec[kRec] = {};
  rec[0] = nlocal;
  rec[1] = dst_addr;
  rec[2] = elems;
  for (uint32_t i = 0; i < nlocal; ++i) {
    rec[3 + 2 * i] = keys[i];
    rec[4 + 2 * i] = src_addrs[i];
  }
  uint64_t* xr;
  RC(ensure(ctx, ctx->d_arrec, (N + 1) * kRec, &xr));
  CK(cudaMemcpyAsync(xr + N * kRec, rec, sizeof rec, cudaMemcpyHostToDevice, ctx->stream));
  RC(comm_allgather(ctx, xr + N * kRec, xr, kRec, kCommU64));
  std::vector<uint64_t> all(N * kRec);
  CK(cudaMemcpyAsync(all.data(), xr, all.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  // global source order: ascending key over every GPU's sliced ranks
  std::vector<std::pair<uint64_t, const uint8_t*>> srcs;
  std::vector<uint8_t*> dsts(N);
  for (int q = 0; q < N; ++q) {
    const uint64_t* r = all.data() + q * kRec;
    if (r[2] != elems)
      return fail(ctx, SNAP_EINVAL, "allreduce_ordered: ranks disagree on the element count");
    dsts[q] = static_cast<uint8_t*>(ctx->ar_peer_arena[q]) + r[1];
    for (uint64_t i = 0; i < r[0]; ++i)
      srcs.push_back({r[3 + 2 * i], static_cast<const uint8_t*>(ctx->ar_peer_arena[q]) + r[4 + 2 * i]});
  }
  std::sort(srcs.begin(), srcs.end(),
            [](const auto& a, const auto& b) { return a.first < b.first; });
  for (size_t i = 1; i < srcs.size(); ++i)
    if (srcs[i].first == srcs[i - 1].first)
      return fail(ctx, SNAP_EINVAL, "allreduce_ordered: duplicate order key");
  if (srcs.empty()) return fail(ctx, SNAP_EINVAL, "allreduce_ordered: no sources on any rank");
  const uint32_t R = uint32_t(srcs.size());
  std::vector<uint64_t> ptrs(R + 2 * N);
  for (uint32_t i = 0; i < R; ++i) ptrs[i] = reinterpret_cast<uint64_t>(srcs[i].second);
  for (int q = 0; q < N; ++q) {
    ptrs[R + q] = reinterpret_cast<uint64_t>(dsts[q]);
    ptrs[R + N + q] = reinterpret_cast<uint64_t>(ctx->ar_peer_flag[q]);
  }
  uint64_t* dp;
  RC(ensure(ctx, ctx->d_arptr, ptrs.size(), &dp));
  CK(cudaMemcpyAsync(dp, ptrs.data(), ptrs.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  const uint64_t epoch = ++ctx->ar_epoch;
  snap::ArArgs a;
  a.src = reinterpret_cast<const uint8_t* const*>(dp);
  a.dst = reinterpret_cast<uint8_t* const*>(dp + R);
  a.flags = reinterpret_cast<uint64_t* const*>(dp + R + N);
  a.myflag = P<uint64_t>(ctx->d_arflag);
  a.R = R;
  a.N = uint32_t(N);
  a.me = uint32_t(ctx->rank);
  a.dtype = dtype;
  a.elems = elems;
  a.epoch = epoch;
  a.use_flags = ctx->lgroup ? 0 : 1;
  unsigned int* cnt;
  RC(ensure(ctx, ctx->d_arcnt, 4, &cnt));
  a.cta_count = cnt;
  if (ctx->lgroup) {
    // same-process ranks may share one GPU: the host barrier replaces the
    // device flag barrier (a spinning kernel could starve a peer's kernel)
    CK(cudaMemsetAsync(cnt, 0, 4, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    BARRIER(ctx->lgroup);  // every rank's sources are final
    CKL(snap::launch_ordered_allreduce(a, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    BARRIER(ctx->lgroup);  // every slice is in every dst
    return SNAP_OK;
  }
  if (epoch == 1) CK(cudaMemsetAsync(cnt, 0, 4, ctx->stream));
  CKL(snap::launch_ordered_allreduce(a, ctx->stream));
  return SNAP_OK;
}

}  // extern "C"
