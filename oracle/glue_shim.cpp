// glue_shim.cpp — TEST INFRASTRUCTURE: runs a scenario on the REFERENCE's own
// scheduler (like ref_shim.cpp's ref_manifest_run) and, at every checkpoint,
// drives libsnap through the maintainer-facing glue (integration/fleetsim_snap.hpp,
// compiled here against the reference headers): restore_job's materialization of
// the manifest onto one snap_ctx, then build_manifest's device section on the
// GPU. Built by oracle/Makefile into oracle/_ref/libfleetsim_glue.so; needs a B200
// at run time (snap_open), so only the GPU tests call it.
#include <cstring>
#include <memory>
#include <vector>

#include "fleetsim/oracle.hpp"
#include "fleetsim/runner.hpp"
#include "fleetsim/scenario.hpp"
#include "fleetsim/sched.hpp"
#include "fleetsim/trace.hpp"
#include "fleetsim_snap.hpp"

using namespace fleetsim;

extern "C" {

// out[k] = {s_g, device_upload (the manifest's), staged bytes by libsnap through the
// glue, restore ok (1/0)} for the first `cap` checkpoints; returns the count or -1.
int glue_manifest_run(const char* scenario_json, int device, uint64_t* out, int cap) {
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
    snap_ctx* ctx = nullptr;
    std::set<u64> seen;
    int count = 0, k = 0;
    const Time step = 5 * kUsec;
    for (Time h = step; k < cap; h += step) {
      const bool drained = eng.run(h);
      if (!sched.jobs().empty()) {
        auto& rec = sched.rec(sched.jobs().begin()->first);
        if (rec.ckpt_count > count && rec.last_manifest) {
          count = rec.ckpt_count;
          const auto& m = *rec.last_manifest;
          const u64 gpu_mem = sched.fleet().at(rec.placement.begin()->second).mem_bytes;
          const auto base = snapglue::gpu_bases(rec.placement, gpu_mem);
          const u64 staging_at = base.size() * gpu_mem;
          if (!ctx && snap_open(device, staging_at + (u64(64) << 20), &ctx) != SNAP_OK) return -1;
          u64 upload = 0;
          for (const auto& [d, b] : m.device_blobs)
            if (!seen.count(d)) upload += b;
          int ok = 1;
          try {
            snapglue::restore_device_state(m, store, rec.placement, base, staging_at, ctx);
          } catch (...) {
            ok = 0;
          }
          const auto sec = snapglue::snapshot_device_state(m, rec.placement, base, ctx);
          snapglue::check(snap_known_commit(ctx), ctx, "known_commit");
          out[4 * k + 0] = m.s_g;
          out[4 * k + 1] = upload;
          out[4 * k + 2] = sec.staged_bytes;
          out[4 * k + 3] = uint64_t(ok);
          ++k;
          for (const auto& ws : m.workers) {
            for (u64 p : ws.pages) seen.insert(p);
            for (const auto& f : ws.files)
              if (!f.deleted) seen.insert(f.digest);
          }
          for (const auto& [d, b] : m.device_blobs) seen.insert(d);
        }
      }
      if (drained || h > 3600 * kSecond) break;
    }
    if (ctx) snap_close(ctx);
    return k;
  } catch (...) {
    return -1;
  }
}

}  // extern "C"
