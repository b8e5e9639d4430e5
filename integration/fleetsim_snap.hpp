// fleetsim_snap.hpp — glue between the reference's own checkpoint types
// (fleetsim, proj/include/fleetsim/ckpt.hpp) and libsnap's C ABI (include/snap.h):
// the two places where a fleetsim maintainer swaps the reference's CPU loops for
// the B200 path. Header-only; include it from fleetsim_core and link libsnap.so.
//
//   restore_device_state   restore_job's materialization (ckpt.cpp:504-533): every
//                          DevRec's blob (BlobStore::get, digest-verified) written
//                          at its recorded address of its rank's GPU, then one
//                          verified K4 pass on the GPU;
//   snapshot_device_state  build_manifest's device section (ckpt.cpp:147-167): the
//                          ranks' live buffers in rank / slot order through
//                          snap_snapshot — first occurrence across ranks (S_G),
//                          store freshness (upload bytes), staged image.
//
// Here one snap_ctx holds every GPU of the job (gpu_base[key] = where GPU key's
// memory starts in the arena): the single-process model of the reference itself.
// On real GPUs each ProxyServer owns one ctx with a communicator (snap_comm_init)
// and the same calls run collectively. Compiled against the
// reference headers and exercised on the GPU by tests/test_gpu_manifest.py.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "fleetsim/ckpt.hpp"
#include "snap.h"

namespace fleetsim::snapglue {

inline void check(int rc, const snap_ctx* ctx, const char* what) {
  if (rc == SNAP_OK) return;
  const std::string msg = std::string(what) + ": " + snap_last_error(ctx);
  if (rc == SNAP_EFAULT) throw SimFault(msg);          // common.hpp:33-35
  if (rc == SNAP_EINTERNAL) throw InternalError(msg);  // common.hpp:42-49
  throw ConfigError(msg);
}

// Arena offsets of the job's GPUs, one `gpu_mem_bytes` region each, by GpuKey order.
inline std::map<GpuKey, u64> gpu_bases(const std::map<RankId, GpuKey>& placement,
                                       u64 gpu_mem_bytes) {
  std::map<GpuKey, u64> base;
  for (const auto& [r, key] : placement) base.emplace(key, 0);
  u64 off = 0;
  for (auto& [key, b] : base) {
    b = off;
    off += gpu_mem_bytes;
  }
  return base;
}

// The manifest's device records as libsnap buffers, canonical (rank, slot) order
// (ckpt.cpp:104,147); `geom` picks one chunk per buffer when every buffer fits one
// chunk, so a chunk digest is the reference's whole-buffer digest.
inline std::vector<snap_buf> device_buffers(const ckpt::Manifest& m,
                                            const std::map<RankId, GpuKey>& placement,
                                            const std::map<GpuKey, u64>& base, snap_geom* geom) {
  std::vector<snap_buf> bufs;
  u64 largest = 0;
  for (const auto& ws : m.workers)
    for (const auto& d : ws.dev) {
      const u64 at = base.at(placement.at(ws.rank)) + d.addr;
      bufs.push_back({uint32_t(ws.rank), d.slot, at, d.words * 8, d.cat, 0});
      largest = std::max<u64>(largest, d.words * 8);
    }
  *geom = largest <= 65536 ? snap_geom{65536, 65536} : snap_geom{4096, 65536};
  return bufs;
}

// restore_job materialization (ckpt.cpp:504-533) onto the ctx: the first
// resident's blobs at the recorded addresses, read through BlobStore::get (which
// re-verifies the digest, ckpt.cpp:23-29), staged contiguously in the arena's
// spare region, then scattered and re-hashed on the GPU by one verified pass.
inline void restore_device_state(const ckpt::Manifest& m, const ckpt::BlobStore& store,
                                 const std::map<RankId, GpuKey>& placement,
                                 const std::map<GpuKey, u64>& base, u64 staging_at,
                                 snap_ctx* ctx) {
  snap_geom geom{};
  const std::vector<snap_buf> bufs = device_buffers(m, placement, base, &geom);
  u64 nchunks = 0;
  check(snap_set_buffers(ctx, bufs.data(), bufs.size(), &geom, &nchunks), ctx, "set_buffers");
  std::vector<u64> src_off, expect;
  u64 off = 0;
  for (const auto& ws : m.workers)
    for (const auto& d : ws.dev) {
      const auto& words = store.get(sim::Digest{d.digest});
      check(snap_write(ctx, staging_at + off, words.data(), words.size() * 8), ctx, "write");
      // the buffer's chunks, in order, at consecutive image offsets
      for (u64 k = 0; k < d.words * 8; k += geom.chunk_bytes) src_off.push_back(off + k);
      off += (words.size() * 8 + 255) / 256 * 256;
    }
  void* arena = nullptr;
  check(snap_arena(ctx, &arena, nullptr), ctx, "arena");
  const uint8_t* image = static_cast<uint8_t*>(arena) + staging_at;
  if (geom.page_bytes == geom.chunk_bytes) {
    // one chunk per buffer: the DevRec digests ARE the chunk digests -> one pass that
    // scatters and verifies (K4 + K1)
    for (const auto& ws : m.workers)
      for (const auto& d : ws.dev) expect.push_back(d.digest);
    check(snap_restore(ctx, image, off, src_off.data(), expect.data(), 1), ctx, "restore");
    return;
  }
  // larger buffers: scatter, then the value-equal whole-buffer digest of every range
  // against its DevRec (Gpu::digest, vdev.cpp:118)
  check(snap_restore(ctx, image, off, src_off.data(), nullptr, 0), ctx, "restore");
  std::vector<u64> got(bufs.size());
  check(snap_digest_whole(ctx, bufs.data(), bufs.size(), got.data()), ctx, "digest_whole");
  size_t i = 0;
  for (const auto& ws : m.workers)
    for (const auto& d : ws.dev)
      if (got[i++] != d.digest) throw SimFault("restore: device digest mismatch");
}

struct DeviceSection {
  u64 staged_bytes = 0;   // S_G on a first checkpoint, the device upload bytes after
  u64 staged_chunks = 0;
  std::vector<u64> chunk_digests;
};

// build_manifest's device section (ckpt.cpp:147-167) of the state in the ctx: K1 ->
// K2 (first occurrence across ranks, minus the store's known set) -> K3. Call
// snap_known_commit(ctx) after persisting so the next call is incremental.
inline DeviceSection snapshot_device_state(const ckpt::Manifest& layout,
                                           const std::map<RankId, GpuKey>& placement,
                                           const std::map<GpuKey, u64>& base, snap_ctx* ctx) {
  snap_geom geom{};
  const std::vector<snap_buf> bufs = device_buffers(layout, placement, base, &geom);
  u64 nchunks = 0;
  check(snap_set_buffers(ctx, bufs.data(), bufs.size(), &geom, &nchunks), ctx, "set_buffers");
  check(snap_snapshot(ctx), ctx, "snapshot");
  DeviceSection out;
  out.chunk_digests.resize(nchunks);
  check(snap_get_digests(ctx, out.chunk_digests.data(), nullptr, nullptr), ctx, "digests");
  check(snap_get_selection(ctx, nullptr, nullptr, nullptr, &out.staged_bytes, &out.staged_chunks),
        ctx, "selection");
  return out;
}

}  // namespace fleetsim::snapglue
