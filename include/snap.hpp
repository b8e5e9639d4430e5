// snap.hpp — C++ mirror of the reference's hot-path API (fleetsim, C++20) over
// the C ABI in snap.h. Same class and method names, same argument meaning and
// the same error behaviour (SimFault / ConfigError / InternalError exceptions,
// std::nullopt on allocator OOM), so a fleetsim maintainer can switch headers:
//
//   fleetsim::vdev::Gpu              -> snapb200::vdev::Gpu        (vdev.hpp:65-122)
//   fleetsim::mem::BidiAllocator     -> snapb200::mem::BidiAllocator (alloc.hpp:17-62)
//   fleetsim::splice::DeviceLayout   -> snapb200::splice::DeviceLayout (splice.hpp:17-24)
//   GpuLedger::plan/execute_switch   -> snapb200::splice::Splicer::switch_to (splice.cpp:167-306)
//   build_manifest device section    -> snapb200::ckpt::Snapshotter (ckpt.cpp:147-167)
//   restore_job materialization      -> snapb200::ckpt::Snapshotter::restore* (ckpt.cpp:517-533)
//   CollectiveEngine sum (sliced DP) -> snapb200::coll::grad_sum (collectives.cpp:137-144)
//   splice::validate_window          -> snapb200::splice::validate_window (splice.cpp:21-61)
//   window open/close mutation sets  -> snapb200::splice::WindowTracker (worker.cpp:351-421)
//   BlobStore::persist + restore_job -> snapb200::ckpt::Snapshotter::persist/load (ckpt.cpp:42-52)
//
// Header-only; link libsnap.so.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "snap.h"

namespace snapb200 {

using u8 = std::uint8_t;
using u64 = std::uint64_t;
using RankId = int;
constexpr RankId kNoRank = -1;

// common.hpp:31-49
struct SimFault : std::runtime_error {
  explicit SimFault(const std::string& w) : std::runtime_error(w) {}
};
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
struct InternalError : std::logic_error {
  explicit InternalError(const std::string& w) : std::logic_error(w) {}
};

inline void check(int rc, const snap_ctx* ctx = nullptr) {
  if (rc == SNAP_OK) return;
  const std::string msg = ctx ? snap_last_error(ctx) : snap_strerror(rc);
  if (rc == SNAP_EFAULT) throw SimFault(msg);
  if (rc == SNAP_EINTERNAL) throw InternalError(msg);
  if (rc == SNAP_EINVAL) throw ConfigError(msg);
  throw std::runtime_error(msg + " (" + snap_strerror(rc) + ")");
}

namespace sim {
// sim.hpp:49-53
struct Digest {
  u64 value = 0;
  friend bool operator==(const Digest&, const Digest&) = default;
  friend auto operator<=>(const Digest&, const Digest&) = default;
};
}  // namespace sim

namespace vdev {

enum class BufCat { Param, OptState, Grad, Activation, Scratch };  // vdev.hpp:17

struct MemRange {  // vdev.hpp:49-53
  u64 addr = 0;
  u64 bytes = 0;
  u64 end() const { return addr + bytes; }
};

// vdev::Gpu: the device arena is real HBM (one cudaMalloc reservation).
class Gpu {
 public:
  Gpu(int id, u64 mem_bytes) { check(snap_open(id, mem_bytes, &ctx_)); }
  ~Gpu() { snap_close(ctx_); }
  Gpu(const Gpu&) = delete;
  Gpu& operator=(const Gpu&) = delete;

  u64 mem_bytes() const {
    u64 b = 0;
    snap_arena(ctx_, nullptr, &b);
    return b;
  }
  std::vector<u64> words(MemRange r) const {  // vdev.cpp:106-116 (a host copy)
    std::vector<u64> w(r.bytes / 8);
    check(snap_read(ctx_, r.addr, w.data(), r.bytes), ctx_);
    return w;
  }
  void write_words(MemRange r, std::span<const u64> src) {  // vdev.cpp:120-124
    if (src.size() * 8 != r.bytes) throw InternalError("write_words: size mismatch");
    check(snap_write(ctx_, r.addr, src.data(), r.bytes), ctx_);
  }
  // vdev.cpp:118 — chunk-Merkle digest of the range (equality-equivalent to the
  // whole-range FNV-1a)
  sim::Digest digest(MemRange r) const {
    snap_buf b{0, 0, r.addr, r.bytes, 0, 0};
    u64 d = 0;
    check(snap_digest_ranges(ctx_, &b, 1, nullptr, &d), ctx_);
    return {d};
  }
  // vdev.cpp:118 VALUE-equal: digest_of_words over the whole range (opt-in path)
  sim::Digest digest_exact(MemRange r) const {
    snap_buf b{0, 0, r.addr, r.bytes, 0, 0};
    u64 d = 0;
    check(snap_digest_whole(ctx_, &b, 1, &d), ctx_);
    return {d};
  }
  snap_ctx* ctx() const { return ctx_; }

 private:
  snap_ctx* ctx_ = nullptr;
};

}  // namespace vdev

namespace mem {

enum class Stability { Stable, Transient };

// alloc.hpp:17-62
class BidiAllocator {
 public:
  static constexpr u64 kAlign = 256;
  BidiAllocator(u64 low, u64 high) {
    if (snap_alloc_create(low, high, &h_) != SNAP_OK)
      throw InternalError("allocator region must be aligned and non-empty");
  }
  ~BidiAllocator() { snap_alloc_destroy(h_); }
  BidiAllocator(const BidiAllocator&) = delete;
  BidiAllocator& operator=(const BidiAllocator&) = delete;

  std::optional<u64> alloc(u64 bytes, Stability st) {
    u64 a = 0;
    const int rc = snap_alloc_alloc(h_, bytes, st == Stability::Stable, &a);
    if (rc == SNAP_ENOMEM) return std::nullopt;
    if (rc == SNAP_EFAULT) throw SimFault("alloc: zero size");
    check(rc);
    return a;
  }
  void free(u64 addr) {
    if (snap_alloc_free(h_, addr) == SNAP_EFAULT) throw SimFault("free: unknown allocation");
  }
  u64 transient_cursor() const { return cursors()[0]; }
  u64 stable_cursor() const { return cursors()[1]; }
  u64 live_bytes() const { return cursors()[2]; }
  sim::Digest stable_state_digest() const { return {snap_alloc_stable_digest(h_)}; }

  using Snapshot = std::vector<u64>;  // exact state image (alloc.cpp:116-140)
  Snapshot snapshot() const {
    u64 n = 0;
    snap_alloc_snapshot(h_, nullptr, 0, &n);
    Snapshot s(n);
    check(snap_alloc_snapshot(h_, s.data(), n, &n));
    return s;
  }
  void restore(const Snapshot& s) { check(snap_alloc_restore(h_, s.data(), s.size())); }

 private:
  std::vector<u64> cursors() const {
    std::vector<u64> c(3);
    snap_alloc_cursors(h_, &c[0], &c[1], &c[2]);
    return c;
  }
  void* h_ = nullptr;
};

}  // namespace mem

namespace splice {

// splice.hpp:17-24
struct DeviceLayout {
  u64 rank_region_end = 0;
  u64 scratch_base = 0;
  u64 scratch_bytes = 0;
  static DeviceLayout carve(u64 mem_bytes, u64 max_buffer_bytes, double slack_fraction) {
    u64 o[3];
    if (snap_layout_carve(mem_bytes, max_buffer_bytes, slack_fraction, o) != SNAP_OK)
      throw InternalError("device too small for layout");
    return {o[0], o[1], o[2]};
  }
};

// splice.hpp:26-34
struct RankBuf {
  int slot = -1;
  u64 addr = 0;
  u64 bytes = 0;
  vdev::BufCat cat{};
  bool live = false;
  bool pending_result = false;
};

// splice.hpp:36-48 (byte counters of the plan)
struct SwitchPlan {
  u64 hashed_bytes = 0;
  u64 swap_out_bytes = 0;
  u64 swap_in_bytes = 0;
  u64 resident_bytes = 0;
  u64 cache_bytes = 0;
  u64 install_bytes = 0;  // queued collective results applied (switch_report, job.cpp:165-171)
};

// GpuLedger's switch machinery on the GPU: plan_switch + execute_switch in one
// call, host cache -> digest-indexed chunk cache in HBM.
class Splicer {
 public:
  Splicer(vdev::Gpu& gpu, u64 cache_bytes) : gpu_(&gpu) {
    check(snap_splice_init(gpu.ctx(), cache_bytes), gpu.ctx());
  }
  void set_rank_bufs(RankId r, const std::vector<RankBuf>& bufs) {
    std::vector<snap_buf> b;
    for (const auto& x : bufs)
      if (x.live)
        b.push_back({u32(r), x.slot, x.addr, x.bytes, int(x.cat),
                     x.pending_result ? SNAP_BUF_PENDING : 0u});
    check(snap_splice_set_rank(gpu_->ctx(), r, b.data(), b.size(), nullptr), gpu_->ctx());
  }
  // restore_job cache seeding for a co-resident rank (ckpt.cpp:526-528): its persisted
  // layout becomes rank r's buffer map and its chunks enter the HBM chunk cache
  snap_persist_stats seed_from(const std::string& dir, RankId layout_rank, RankId r) {
    snap_persist_stats st{};
    check(snap_splice_load(gpu_->ctx(), dir.c_str(), layout_rank, r, 0, &st), gpu_->ctx());
    return st;
  }
  SwitchPlan switch_to(RankId from, RankId to) {
    snap_switch_stats s{};
    check(snap_splice_switch(gpu_->ctx(), from, to, &s), gpu_->ctx());
    return {s.hashed_bytes, s.swap_out_bytes, s.swap_in_bytes, s.resident_bytes, s.cache_bytes,
            s.install_bytes};
  }
  // JobRuntime::on_coll_complete (job.cpp:206-222): the result at src goes into every
  // listed rank's G slot — the active rank now, the others at their next switch_to
  void install_result(const std::vector<RankId>& ranks, const std::vector<u64>& slot_addrs,
                      u64 src_addr, u64 bytes) {
    std::vector<int> r(ranks.begin(), ranks.end());
    check(snap_splice_install(gpu_->ctx(), r.data(), slot_addrs.data(), uint32_t(r.size()),
                              src_addr, bytes),
          gpu_->ctx());
  }
  u64 pending_install_bytes(RankId r) const {
    u64 c = 0, b = 0;
    check(snap_splice_pending(gpu_->ctx(), r, &c, &b), gpu_->ctx());
    return b;
  }

 private:
  using u32 = std::uint32_t;
  vdev::Gpu* gpu_;
};

// splice.hpp:50-59
struct ValidationRecord {
  std::map<u64, std::pair<u64, sim::Digest>> mutations;  // addr -> (bytes, digest after window)
  std::vector<std::pair<u64, sim::Digest>> d2h_copies;    // (bytes, digest)
};
struct ValidationOutcome {
  bool pass = true;
  std::string reason;
};

// splice.cpp:21-61 (same comparison order and reason text)
inline ValidationOutcome validate_window(const std::map<RankId, ValidationRecord>& records) {
  std::vector<std::vector<snap_mutation>> m;
  std::vector<std::vector<u64>> d;
  std::vector<snap_window_record> r;
  for (const auto& [rank, rec] : records) {
    m.emplace_back();
    for (const auto& [a, bd] : rec.mutations) m.back().push_back({a, bd.first, bd.second.value});
    d.emplace_back();
    for (const auto& [b, dg] : rec.d2h_copies) {
      d.back().push_back(b);
      d.back().push_back(dg.value);
    }
  }
  size_t i = 0;
  for (const auto& [rank, rec] : records) {
    r.push_back({rank, m[i].data(), m[i].size(), d[i].data(), rec.d2h_copies.size()});
    ++i;
  }
  char why[512];
  const int rc = snap_validate_window(r.data(), r.size(), why, sizeof why);
  if (rc < 0) check(rc);
  return {rc == 1, rc == 1 ? std::string() : std::string(why)};
}

// The validation branch of WorkerExec::do_window_open / do_window_close
// (worker.cpp:355-362, 411-421) for one rank's live buffers.
class WindowTracker {
 public:
  explicit WindowTracker(vdev::Gpu& gpu) : gpu_(&gpu) {}
  void open(RankId r, const std::vector<RankBuf>& bufs) {
    const auto b = live(r, bufs);
    check(snap_window_open(gpu_->ctx(), r, b.data(), b.size()), gpu_->ctx());
  }
  // fills rec.mutations (d2h_copies are the caller's, worker.cpp:664-669)
  void close(RankId r, const std::vector<RankBuf>& bufs, ValidationRecord& rec) {
    const auto b = live(r, bufs);
    std::vector<snap_mutation> out(b.size());
    u64 n = 0;
    check(snap_window_close(gpu_->ctx(), r, b.data(), b.size(), out.data(), out.size(), &n),
          gpu_->ctx());
    rec.mutations.clear();
    for (u64 i = 0; i < n; ++i) rec.mutations[out[i].addr] = {out[i].bytes, {out[i].digest}};
  }

 private:
  static std::vector<snap_buf> live(RankId r, const std::vector<RankBuf>& bufs) {
    std::vector<snap_buf> b;
    for (const auto& x : bufs)
      if (x.live)
        b.push_back({std::uint32_t(r), x.slot, x.addr, x.bytes, int(x.cat),
                     x.pending_result ? SNAP_BUF_PENDING : 0u});
    return b;
  }
  vdev::Gpu* gpu_;
};

}  // namespace splice

namespace ckpt {

// The device section of build_manifest + restore_job materialization.
class Snapshotter {
 public:
  explicit Snapshotter(vdev::Gpu& gpu) : gpu_(&gpu) {}
  // (rank, slot) ordered DevRecs of the cut (ckpt.hpp:64-71)
  u64 set_buffers(const std::vector<snap_buf>& bufs, u64 page_bytes = 4096,
                  u64 chunk_bytes = 65536) {
    snap_geom g{uint32_t(page_bytes), uint32_t(chunk_bytes)};
    u64 n = 0;
    check(snap_set_buffers(gpu_->ctx(), bufs.data(), bufs.size(), &g, &n), gpu_->ctx());
    nchunks_ = n;
    return n;
  }
  void snapshot() { check(snap_snapshot(gpu_->ctx()), gpu_->ctx()); }
  std::vector<sim::Digest> chunk_digests() const {
    std::vector<u64> d(nchunks_);
    check(snap_get_digests(gpu_->ctx(), d.data(), nullptr, nullptr), gpu_->ctx());
    std::vector<sim::Digest> out;
    for (u64 x : d) out.push_back({x});
    return out;
  }
  // staged bytes (the BlobStore-fresh bytes of this snapshot, ckpt.cpp:162-164)
  u64 staged_bytes() const {
    u64 b = 0, c = 0;
    check(snap_get_selection(gpu_->ctx(), nullptr, nullptr, nullptr, &b, &c), gpu_->ctx());
    return b;
  }
  std::vector<u8> staging(u64 off, u64 bytes) const {
    std::vector<u8> v(bytes);
    check(snap_read_staging(gpu_->ctx(), off, v.data(), bytes), gpu_->ctx());
    return v;
  }
  void commit() { check(snap_known_commit(gpu_->ctx()), gpu_->ctx()); }  // next one is incremental
  void restore_self(bool verify = true) {
    check(snap_restore_self(gpu_->ctx(), verify ? 1 : 0), gpu_->ctx());
  }
  // BlobStore::persist layout (ckpt.cpp:35-52) for this snapshot's staged chunks,
  // plus the rank's layout + manifest; returns the stats
  snap_persist_stats persist(const std::string& dir, int threads = 0) {
    snap_persist_stats st{};
    check(snap_persist(gpu_->ctx(), dir.c_str(), nullptr, 0, threads, &st), gpu_->ctx());
    return st;
  }
  // the same under an explicit layout id (one cut per time-sliced rank of a GPU)
  snap_persist_stats persist_as(const std::string& dir, RankId layout_rank, int threads = 0) {
    snap_persist_stats st{};
    check(snap_persist_rank(gpu_->ctx(), dir.c_str(), layout_rank, nullptr, 0, threads, &st),
          gpu_->ctx());
    return st;
  }
  // restore_job materialization from a directory (ckpt.cpp:504-533); SimFault on a
  // missing or corrupt blob (BlobStore::get, ckpt.cpp:23-29)
  snap_persist_stats load(const std::string& dir, int rank = 0, bool verify = true) {
    snap_persist_stats st{};
    check(snap_load(gpu_->ctx(), dir.c_str(), rank, verify ? 1 : 0, 0, &st), gpu_->ctx());
    nchunks_ = st.layout_chunks;
    return st;
  }
  static std::string blob_rel_path(sim::Digest d) {  // ckpt.cpp:35-40
    char b[40];
    check(snap_blob_rel_path(d.value, b, sizeof b));
    return b;
  }

 private:
  vdev::Gpu* gpu_;
  u64 nchunks_ = 0;
};

}  // namespace ckpt

namespace coll {
// collectives.cpp:140-141 (u64) / fixed ascending-dp-order fp32 sum into dst
inline void grad_sum(vdev::Gpu& gpu, int dtype, const std::vector<u64>& src_addrs, u64 dst_addr,
                     u64 elems, bool accumulate = false) {
  check(snap_grad_sum(gpu.ctx(), dtype, src_addrs.data(), uint32_t(src_addrs.size()), dst_addr,
                      elems, accumulate ? 1 : 0),
        gpu.ctx());
}
// The device-level sum over GPUs in a fixed key order (collectives.cpp:137-154 with the
// fixed-order fp32 mode): collective over the ctx's communicator
inline void allreduce_ordered(vdev::Gpu& gpu, int dtype, const std::vector<uint32_t>& keys,
                              const std::vector<u64>& src_addrs, u64 dst_addr, u64 elems) {
  if (keys.size() != src_addrs.size()) throw ConfigError("allreduce_ordered: keys / sources");
  check(snap_allreduce_ordered(gpu.ctx(), dtype, keys.data(), src_addrs.data(),
                               uint32_t(keys.size()), dst_addr, elems),
        gpu.ctx());
}
}  // namespace coll

}  // namespace snapb200
