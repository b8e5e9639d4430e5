// ref_shim.cpp — extern "C" wrapper over the REFERENCE library (fleetsim_core),
// compiled from /root/reference/proj/src by oracle/Makefile into oracle/_ref/.
// TEST INFRASTRUCTURE ONLY: it lets the tests pin the CPU restatement
// (oracle/snap_oracle.c) and the product against the reference's own code,
// and lets bench.py time the reference's CPU path (`--impl reference`,
// cpu_baseline kind "reference"). Nothing in the product links it.
#include <atomic>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <thread>
#include <vector>

#include "fleetsim/alloc.hpp"
#include "fleetsim/ckpt.hpp"
#include "fleetsim/oracle.hpp"
#include "fleetsim/runner.hpp"
#include "fleetsim/scenario.hpp"
#include "fleetsim/sched.hpp"
#include "fleetsim/trace.hpp"
#include "fleetsim/sim.hpp"
#include "fleetsim/splice.hpp"
#include "fleetsim/vdev.hpp"

using namespace fleetsim;

extern "C" {

// sim.hpp:67-70
uint64_t ref_digest_of_words(const uint64_t* w, uint64_t n) {
  return sim::digest_of_words(std::span<const u64>(w, n)).value;
}
// sim.hpp:58-65
uint64_t ref_digest_of_bytes(const uint8_t* p, uint64_t n) {
  return sim::digest_of(std::span<const u8>(p, n)).value;
}
uint64_t ref_mix64(uint64_t x) { return sim::mix64(x); }

// ---- ckpt::BlobStore (ckpt.cpp:16-52) ----
void* ref_store_new() { return new ckpt::BlobStore(); }
void ref_store_free(void* s) { delete static_cast<ckpt::BlobStore*>(s); }
int ref_store_put(void* s, const uint64_t* w, uint64_t n, uint64_t* digest) {
  auto r = static_cast<ckpt::BlobStore*>(s)->put(std::span<const u64>(w, n));
  *digest = r.digest.value;
  return r.fresh ? 1 : 0;
}
// 0 ok, -1 missing / verification failure (SimFault), -2 size mismatch
int ref_store_get(void* s, uint64_t digest, uint64_t* out, uint64_t n) {
  try {
    const auto& v = static_cast<ckpt::BlobStore*>(s)->get(sim::Digest{digest});
    if (v.size() != n) return -2;
    std::memcpy(out, v.data(), n * 8);
    return 0;
  } catch (const SimFault&) {
    return -1;
  }
}
uint64_t ref_store_total_bytes(void* s) { return static_cast<ckpt::BlobStore*>(s)->total_bytes(); }
uint64_t ref_store_count(void* s) { return static_cast<ckpt::BlobStore*>(s)->count(); }
// BlobStore::persist / blob_rel_path (ckpt.cpp:35-52); 0 ok, -1 on any exception
int ref_store_persist(void* s, const char* dir) {
  try {
    static_cast<ckpt::BlobStore*>(s)->persist(dir);
    return 0;
  } catch (...) {
    return -1;
  }
}
// splice::validate_window (splice.cpp:21-61) over flattened records:
// muts = (addr, bytes, digest) triples, d2h = (bytes, digest) pairs, rank-major.
int ref_validate_window(int n, const int* ranks, const uint64_t* nmut, const uint64_t* muts,
                        const uint64_t* nd2h, const uint64_t* d2h, char* reason, uint64_t cap) {
  std::map<RankId, splice::ValidationRecord> recs;
  uint64_t m = 0, c = 0;
  for (int i = 0; i < n; ++i) {
    splice::ValidationRecord r;
    for (uint64_t k = 0; k < nmut[i]; ++k, ++m)
      r.mutations[muts[3 * m]] = {muts[3 * m + 1], sim::Digest{muts[3 * m + 2]}};
    for (uint64_t k = 0; k < nd2h[i]; ++k, ++c)
      r.d2h_copies.push_back({d2h[2 * c], sim::Digest{d2h[2 * c + 1]}});
    recs[ranks[i]] = std::move(r);
  }
  const auto out = splice::validate_window(recs);
  const size_t k = std::min<size_t>(out.reason.size(), size_t(cap - 1));
  std::memcpy(reason, out.reason.data(), k);
  reason[k] = 0;
  return out.pass ? 1 : 0;
}
int ref_blob_rel_path(uint64_t digest, char* out, uint64_t cap) {
  const std::string p = ckpt::BlobStore::blob_rel_path(sim::Digest{digest});
  if (p.size() + 1 > cap) return -1;
  std::memcpy(out, p.c_str(), p.size() + 1);
  return 0;
}

// ---- mem::BidiAllocator (alloc.cpp:62-155) ----
void* ref_alloc_new(uint64_t low, uint64_t high) { return new mem::BidiAllocator(low, high); }
void ref_alloc_free_obj(void* a) { delete static_cast<mem::BidiAllocator*>(a); }
// 0 ok, 1 OOM (nullopt), -1 SimFault
int ref_alloc_alloc(void* a, uint64_t bytes, int stable, uint64_t* addr) {
  try {
    auto r = static_cast<mem::BidiAllocator*>(a)->alloc(
        bytes, stable ? mem::Stability::Stable : mem::Stability::Transient);
    if (!r) return 1;
    *addr = *r;
    return 0;
  } catch (const SimFault&) {
    return -1;
  }
}
int ref_alloc_free(void* a, uint64_t addr) {
  try {
    static_cast<mem::BidiAllocator*>(a)->free(addr);
    return 0;
  } catch (const SimFault&) {
    return -1;
  }
}
uint64_t ref_alloc_stable_digest(void* a) {
  return static_cast<mem::BidiAllocator*>(a)->stable_state_digest().value;
}
void ref_alloc_cursors(void* a, uint64_t* tc, uint64_t* sc, uint64_t* live) {
  auto* x = static_cast<mem::BidiAllocator*>(a);
  *tc = x->transient_cursor();
  *sc = x->stable_cursor();
  *live = x->live_bytes();
}

// ---- splice::DeviceLayout::carve (splice.cpp:7-19) ----
int ref_carve(uint64_t mem, uint64_t max_buf, double slack, uint64_t out[3]) {
  try {
    auto l = splice::DeviceLayout::carve(mem, max_buf, slack);
    out[0] = l.rank_region_end;
    out[1] = l.scratch_base;
    out[2] = l.scratch_bytes;
    return 0;
  } catch (const InternalError&) {
    return -1;
  }
}

// ---- the reference's CPU snapshot path, timed as the baseline ----
// Per 64 KiB chunk: BlobStore::put (digest_of_words + dedup map + copy),
// exactly what build_manifest does per device buffer (ckpt.cpp:157-164), at
// chunk granularity. One BlobStore per thread (the class is not thread-safe).
// Returns store-fresh bytes; digests[g] receives the put digest.
uint64_t ref_snapshot_chunks(const uint8_t* image, uint64_t bytes, uint32_t chunk_bytes,
                             int nthreads, uint64_t* digests) {
  uint64_t nchunks = (bytes + chunk_bytes - 1) / chunk_bytes;
  if (nthreads < 1) nthreads = 1;
  std::atomic<uint64_t> fresh{0};
  auto work = [&](int t) {
    ckpt::BlobStore store;
    uint64_t f = 0;
    for (uint64_t g = t; g < nchunks; g += nthreads) {
      uint64_t off = g * chunk_bytes;
      uint64_t len = std::min<uint64_t>(chunk_bytes, bytes - off);
      auto r = store.put(std::span<const u64>(reinterpret_cast<const u64*>(image + off), len / 8));
      if (digests) digests[g] = r.digest.value;
      if (r.fresh) f += len;
    }
    fresh += f;
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nthreads; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  return fresh.load();
}

// Reference restore path: BlobStore::get (digest-verified, ckpt.cpp:23-29) +
// Gpu::write_words at the recorded address (ckpt.cpp:522-523).
// Returns 0, or -1 on a verification failure.
int ref_restore_chunks(const uint8_t* image, uint64_t bytes, uint32_t chunk_bytes, int nthreads,
                       uint8_t* out) {
  uint64_t nchunks = (bytes + chunk_bytes - 1) / chunk_bytes;
  if (nthreads < 1) nthreads = 1;
  std::atomic<int> bad{0};
  auto work = [&](int t) {
    ckpt::BlobStore store;
    std::vector<sim::Digest> ds;
    for (uint64_t g = t; g < nchunks; g += nthreads) {
      uint64_t off = g * chunk_bytes;
      uint64_t len = std::min<uint64_t>(chunk_bytes, bytes - off);
      ds.push_back(store.put(std::span<const u64>(reinterpret_cast<const u64*>(image + off), len / 8))
                       .digest);
    }
    size_t i = 0;
    for (uint64_t g = t; g < nchunks; g += nthreads, ++i) {
      uint64_t off = g * chunk_bytes;
      try {
        const auto& v = store.get(ds[i]);
        std::memcpy(out + off, v.data(), v.size() * 8);
      } catch (const SimFault&) {
        bad = 1;
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nthreads; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  return bad ? -1 : 0;
}

// Reference gradient sum (collectives.cpp:140-141) over nranks contributions.
void ref_grad_sum_u64(const uint64_t* const* g, uint32_t nranks, uint64_t n, uint64_t* out,
                      int nthreads) {
  if (nthreads < 1) nthreads = 1;
  auto work = [&](int t) {
    uint64_t lo = n * t / nthreads, hi = n * (t + 1) / nthreads;
    std::vector<u64> sum(hi - lo, 0);
    for (uint32_t r = 0; r < nranks; ++r)
      for (uint64_t i = lo; i < hi; ++i) sum[i - lo] += g[r][i];
    std::memcpy(out + lo, sum.data(), (hi - lo) * 8);
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nthreads; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
}

// ---- splice::GpuLedger + vdev::Gpu (splice.cpp:150-354, vdev.cpp:72-124) ----
// Scripted driver for the splice parity test. Before every plan the outgoing
// rank's digests are refreshed (refresh_digests also updates the ledger
// entries), which is the one-line fix of SURVEY App. A-1 (stale Entry::digest).
struct RefSplice {
  std::unique_ptr<vdev::Gpu> gpu;
  std::unique_ptr<splice::GpuLedger> led;
  // JobRuntime's side of result installs (job.cpp:164-171, 206-222): the rank
  // of the last switch is active; the others queue (ProxyServer::install_queue)
  RankId active = kNoRank;
  std::map<RankId, std::vector<std::pair<int, std::vector<u64>>>> queue;
};

void* ref_splice_new(uint64_t mem_bytes, uint64_t max_buf) {
  auto* s = new RefSplice();
  s->gpu = std::make_unique<vdev::Gpu>(0, mem_bytes);
  s->led = std::make_unique<splice::GpuLedger>(*s->gpu,
                                               splice::DeviceLayout::carve(mem_bytes, max_buf, 0.0));
  return s;
}
void ref_splice_free(void* s) { delete static_cast<RefSplice*>(s); }

// the active rank allocates a buffer (worker.cpp:145-148): ledger + registry
int ref_splice_alloc(void* p, int rank, int slot, uint64_t addr, uint64_t bytes, int cat,
                     int pending) {
  auto* s = static_cast<RefSplice*>(p);
  try {
    s->led->on_alloc(rank, slot, addr, bytes, static_cast<vdev::BufCat>(cat));
    s->gpu->register_buffer({addr, bytes}, static_cast<vdev::BufCat>(cat));
    if (pending) s->led->mark_pending_result(rank, slot);
    return 0;
  } catch (const SimFault&) {
    return -1;
  } catch (const InternalError&) {
    return -2;
  }
}

int ref_splice_write(void* p, uint64_t addr, const uint64_t* words, uint64_t n) {
  auto* s = static_cast<RefSplice*>(p);
  s->gpu->write_words({addr, n * 8}, std::span<const u64>(words, n));
  return 0;
}

int ref_splice_read(void* p, uint64_t addr, uint64_t* words, uint64_t n) {
  auto* s = static_cast<RefSplice*>(p);
  auto sp = s->gpu->words({addr, n * 8});
  std::memcpy(words, sp.data(), n * 8);
  return 0;
}

// out = {swap_out_bytes, swap_in_bytes, d2d_bytes, moves, host_cache_bytes}
int ref_splice_switch(void* p, int from, int to, uint64_t* out) {
  auto* s = static_cast<RefSplice*>(p);
  try {
    if (from >= 0) s->led->refresh_digests(from);
    auto plan = s->led->plan_switch(from < 0 ? kNoRank : from, to < 0 ? kNoRank : to);
    s->led->execute_switch(from < 0 ? kNoRank : from, to < 0 ? kNoRank : to, plan);
    out[0] = plan.swap_out_bytes;
    out[1] = plan.swap_in_bytes;
    out[2] = plan.d2d_bytes;
    out[3] = plan.moves.size();
    out[4] = s->led->host_cache_bytes();
    return 0;
  } catch (const SimFault&) {
    return -1;
  } catch (const InternalError&) {
    return -2;
  }
}

// ---- build_manifest through the reference's own scheduler (ckpt.cpp:79-189) ----
// Runs a scenario (Scenario::parse JSON) the way cli::run_scenario does
// (runner.cpp:20-80) but in small steps of simulated time, capturing every
// checkpoint manifest of job 1 as it is produced, plus the device content of
// every DevRec (BlobStore::get of its digest, digest-verified). device_upload =
// bytes of the manifest's unique device blobs whose digest the store did not
// hold before this checkpoint (build_manifest's `fresh`, device part only).
struct RefManifests {
  struct M {
    uint64_t s_g, s_cr, s_cr_inc, upload, dump_d2h_max, total_blob, device_upload, world;
    std::vector<std::vector<ckpt::WorkerSnapshot::DevRec>> dev;  // [rank]
    std::vector<std::vector<std::vector<u64>>> content;          // [rank][i]
  };
  std::vector<M> ms;
};

void* ref_manifest_run(const char* scenario_json) {
  try {
    auto sc = cli::Scenario::parse(Json::parse(scenario_json));
    sim::Engine eng;
    TraceSink trace(false);
    ckpt::BlobStore store;
    sched::Scheduler sched(eng, sc.cost, trace, store, sc.fleet, sc.sla);
    std::map<std::string, int> ids;
    for (size_t i = 0; i < sc.jobs.size(); ++i) {
      auto spec = sc.jobs[i].spec;
      spec.seed = sim::mix3(sc.seed, i, spec.seed);
      auto cfg = sc.jobs[i].cfg;
      std::vector<Dur> mb;
      if (cli::oracle_feasible(spec, nullptr)) mb = oracle::run(wl::build_job(spec), sc.cost).minibatch_ns;
      eng.schedule(from_secs(sc.jobs[i].arrival_sec), [&sched, &ids, spec, cfg, mb]() {
        ids[spec.name] = sched.submit(spec, cfg, mb);
      });
    }
    for (const auto& ev : sc.events)
      if (ev.kind == "checkpoint")
        eng.schedule(from_secs(ev.at_sec), [&sched, &ids, ev]() {
          auto it = ids.find(ev.job);
          if (it != ids.end()) sched.request_checkpoint(it->second);
        });
    auto* out = new RefManifests();
    std::set<u64> seen;  // every digest the store held before a checkpoint
    int count = 0;
    const Time step = 5 * kUsec;
    for (Time h = step;; h += step) {
      const bool drained = eng.run(h);
      if (!sched.jobs().empty()) {
        auto& rec = sched.rec(sched.jobs().begin()->first);
        if (rec.ckpt_count > count && rec.last_manifest) {
          count = rec.ckpt_count;
          const auto& m = *rec.last_manifest;
          RefManifests::M x{m.s_g, m.s_cr, m.s_cr_inc, m.upload_bytes, m.dump_d2h_max,
                            m.total_blob_bytes, 0, uint64_t(m.workers.size()), {}, {}};
          for (const auto& [d, b] : m.device_blobs)
            if (!seen.count(d)) x.device_upload += b;
          for (const auto& ws : m.workers) {
            x.dev.push_back(ws.dev);
            x.content.emplace_back();
            for (const auto& d : ws.dev) x.content.back().push_back(store.get(sim::Digest{d.digest}));
            for (u64 p : ws.pages) seen.insert(p);
            for (const auto& f : ws.files)
              if (!f.deleted) seen.insert(f.digest);
          }
          for (const auto& [d, b] : m.device_blobs) seen.insert(d);
          out->ms.push_back(std::move(x));
        }
      }
      if (drained) break;
      if (h > 3600 * kSecond) break;
    }
    return out;
  } catch (...) {
    return nullptr;
  }
}
void ref_manifest_free(void* h) { delete static_cast<RefManifests*>(h); }
int ref_manifest_count(void* h) { return int(static_cast<RefManifests*>(h)->ms.size()); }
// out = {s_g, s_cr, s_cr_inc, upload_bytes, dump_d2h_max, total_blob_bytes, device_upload, world}
void ref_manifest_stats(void* h, int k, uint64_t* out) {
  const auto& m = static_cast<RefManifests*>(h)->ms.at(k);
  const uint64_t v[8] = {m.s_g, m.s_cr, m.s_cr_inc, m.upload, m.dump_d2h_max, m.total_blob,
                         m.device_upload, m.world};
  std::memcpy(out, v, sizeof v);
}
int ref_manifest_ndev(void* h, int k, int rank) {
  return int(static_cast<RefManifests*>(h)->ms.at(k).dev.at(rank).size());
}
// rec = {slot, addr, words, cat, digest}
void ref_manifest_dev(void* h, int k, int rank, int i, uint64_t* rec, uint64_t* words) {
  const auto& m = static_cast<RefManifests*>(h)->ms.at(k);
  const auto& d = m.dev.at(rank).at(i);
  rec[0] = uint64_t(int64_t(d.slot));
  rec[1] = d.addr;
  rec[2] = d.words;
  rec[3] = uint64_t(int64_t(d.cat));
  rec[4] = d.digest;
  if (words) std::memcpy(words, m.content.at(rank).at(i).data(), d.words * 8);
}

// switch_to (job.cpp:146-171): plan, execute, then the queued installs of
// `to`. out = {swap_out, swap_in, d2d, moves, host_cache_bytes, install_bytes}
int ref_splice_switch2(void* p, int from, int to, uint64_t* out) {
  auto* s = static_cast<RefSplice*>(p);
  const int rc = ref_splice_switch(p, from, to, out);
  if (rc != 0) return rc;
  uint64_t inst = 0;
  try {
    if (to >= 0) {
      for (auto& [slot, words] : s->queue[to]) {
        s->led->install_result(to, slot, words);
        inst += words.size() * 8;
      }
      s->queue[to].clear();
    }
  } catch (const InternalError&) {
    return -2;
  }
  s->active = to < 0 ? kNoRank : to;
  out[5] = inst;
  return 0;
}

// WorkerExec::do_collective marks the issuer's gradient pending (worker.cpp:298)
int ref_splice_mark_pending(void* p, int rank, int slot) {
  try {
    static_cast<RefSplice*>(p)->led->mark_pending_result(rank, slot);
    return 0;
  } catch (...) {
    return -1;
  }
}

// on_coll_complete (job.cpp:206-222): active rank installs now, others queue
int ref_splice_install(void* p, int rank, int slot, const uint64_t* words, uint64_t n) {
  auto* s = static_cast<RefSplice*>(p);
  try {
    if (s->active == rank)
      s->led->install_result(rank, slot, std::span<const u64>(words, n));
    else
      s->queue[rank].push_back({slot, std::vector<u64>(words, words + n)});
    return 0;
  } catch (const InternalError&) {
    return -2;
  } catch (...) {
    return -1;
  }
}

}  // extern "C"
