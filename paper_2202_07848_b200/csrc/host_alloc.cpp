// host_alloc.cpp — the device-proxy memory tracker: a two-ended allocator over
// the arena's rank region, same contract as mem::BidiAllocator
// (proj/include/fleetsim/alloc.hpp:17-62, proj/src/alloc.cpp:62-155):
//   * stable requests (params / optimizer state) are carved top-down, transient
//     ones (grads / activations) bottom-up, so the stable addresses are a pure
//     function of the stable request sequence — replicas of a DP job get
//     identical P/O addresses (test_alloc.cpp:44-80), which is what makes the
//     positional cross-rank dedup and the splice "already here" test work;
//   * 256-byte rounding; OOM = the cursors would cross (nullopt in the
//     reference, SNAP_ENOMEM here); freeing an unknown address is a fault;
//   * freed blocks go to per-end free lists with neighbour coalescing; the
//     stable end reuses the highest fitting block (carving its top), the
//     transient end the lowest fitting block (carving its bottom); a free
//     block touching its cursor retreats the cursor.
// Host metadata only: no device work happens here.
#include <map>
#include <vector>

#include "snap.h"

namespace {

uint64_t fnv_words(const std::vector<uint64_t>& w) {  // sim::digest_of_words
  uint64_t h = 14695981039346656037ull;
  for (uint64_t x : w)
    for (int b = 0; b < 8; ++b) {
      h ^= (x >> (8 * b)) & 0xff;
      h *= 1099511628211ull;
    }
  return h;
}

struct Tracker {
  uint64_t lo_bound, hi_bound;
  uint64_t t_cur, s_cur;  // transient cursor (first unused low byte), stable cursor (one past)
  uint64_t live_bytes = 0;
  std::map<uint64_t, uint64_t> lowfree, highfree;  // base -> size
  struct Live {
    uint64_t size;
    bool stable;
  };
  std::map<uint64_t, Live> live;

  Tracker(uint64_t lo, uint64_t hi) : lo_bound(lo), hi_bound(hi), t_cur(lo), s_cur(hi) {}

  static void add_free(std::map<uint64_t, uint64_t>& fl, uint64_t base, uint64_t size) {
    auto nx = fl.lower_bound(base);
    if (nx != fl.begin()) {
      auto pv = std::prev(nx);
      if (pv->first + pv->second == base) {  // merge with the left neighbour
        base = pv->first;
        size += pv->second;
        fl.erase(pv);
      }
    }
    if (nx != fl.end() && base + size == nx->first) {  // and with the right one
      size += nx->second;
      fl.erase(nx);
    }
    fl[base] = size;
  }

  bool carve_high(uint64_t bytes, uint64_t* out) {
    for (auto it = highfree.end(); it != highfree.begin();) {
      --it;
      if (it->second < bytes) continue;
      const uint64_t base = it->first, size = it->second;
      highfree.erase(it);
      if (size > bytes) highfree[base] = size - bytes;
      *out = base + size - bytes;
      return true;
    }
    return false;
  }

  bool carve_low(uint64_t bytes, uint64_t* out) {
    for (auto it = lowfree.begin(); it != lowfree.end(); ++it) {
      if (it->second < bytes) continue;
      const uint64_t base = it->first, size = it->second;
      lowfree.erase(it);
      if (size > bytes) lowfree[base + bytes] = size - bytes;
      *out = base;
      return true;
    }
    return false;
  }

  int alloc(uint64_t bytes, bool stable, uint64_t* out) {
    if (bytes == 0) return SNAP_EFAULT;
    bytes = (bytes + 255) / 256 * 256;
    uint64_t a = 0;
    if (stable) {
      if (!carve_high(bytes, &a)) {
        if (s_cur < t_cur + bytes) return SNAP_ENOMEM;
        s_cur -= bytes;
        a = s_cur;
      }
    } else {
      if (!carve_low(bytes, &a)) {
        if (t_cur + bytes > s_cur) return SNAP_ENOMEM;
        a = t_cur;
        t_cur += bytes;
      }
    }
    live[a] = {bytes, stable};
    live_bytes += bytes;
    *out = a;
    return SNAP_OK;
  }

  int release(uint64_t addr) {
    auto it = live.find(addr);
    if (it == live.end()) return SNAP_EFAULT;
    const Live l = it->second;
    live.erase(it);
    live_bytes -= l.size;
    if (l.stable) {
      add_free(highfree, addr, l.size);
      auto at = highfree.find(s_cur);
      if (at != highfree.end()) {
        s_cur += at->second;
        highfree.erase(at);
      }
    } else {
      add_free(lowfree, addr, l.size);
      if (!lowfree.empty()) {
        auto last = std::prev(lowfree.end());
        if (last->first + last->second == t_cur) {
          t_cur = last->first;
          lowfree.erase(last);
        }
      }
    }
    return SNAP_OK;
  }

  uint64_t stable_digest() const {
    std::vector<uint64_t> w{s_cur};
    for (const auto& [b, s] : highfree) {
      w.push_back(b);
      w.push_back(s);
    }
    for (const auto& [a, l] : live)
      if (l.stable) {
        w.push_back(a);
        w.push_back(l.size);
      }
    return fnv_words(w);
  }

  // snapshot layout (u64 words): t_cur, s_cur, nlow, nhigh, nlive,
  // (base,size)*nlow, (base,size)*nhigh, (addr,size,stable)*nlive
  std::vector<uint64_t> save() const {
    std::vector<uint64_t> w{t_cur, s_cur, lowfree.size(), highfree.size(), live.size()};
    for (const auto& [b, s] : lowfree) w.insert(w.end(), {b, s});
    for (const auto& [b, s] : highfree) w.insert(w.end(), {b, s});
    for (const auto& [a, l] : live) w.insert(w.end(), {a, l.size, uint64_t(l.stable)});
    return w;
  }

  int load(const uint64_t* w, uint64_t n) {
    if (n < 5) return SNAP_EINVAL;
    const uint64_t nl = w[2], nh = w[3], nv = w[4];
    if (n != 5 + 2 * nl + 2 * nh + 3 * nv) return SNAP_EINVAL;
    t_cur = w[0];
    s_cur = w[1];
    lowfree.clear();
    highfree.clear();
    live.clear();
    live_bytes = 0;
    const uint64_t* p = w + 5;
    for (uint64_t i = 0; i < nl; ++i, p += 2) lowfree[p[0]] = p[1];
    for (uint64_t i = 0; i < nh; ++i, p += 2) highfree[p[0]] = p[1];
    for (uint64_t i = 0; i < nv; ++i, p += 3) {
      live[p[0]] = {p[1], p[2] != 0};
      live_bytes += p[1];
    }
    return SNAP_OK;
  }
};

}  // namespace

extern "C" {

int snap_alloc_create(uint64_t low, uint64_t high, void** out) {
  if (!out || low % 256 || high % 256 || low >= high) return SNAP_EINVAL;
  *out = new Tracker(low, high);
  return SNAP_OK;
}

int snap_alloc_destroy(void* a) {
  delete static_cast<Tracker*>(a);
  return SNAP_OK;
}

int snap_alloc_alloc(void* a, uint64_t bytes, int stable, uint64_t* addr) {
  if (!a || !addr) return SNAP_EINVAL;
  return static_cast<Tracker*>(a)->alloc(bytes, stable != 0, addr);
}

int snap_alloc_free(void* a, uint64_t addr) {
  if (!a) return SNAP_EINVAL;
  return static_cast<Tracker*>(a)->release(addr);
}

uint64_t snap_alloc_stable_digest(void* a) { return static_cast<Tracker*>(a)->stable_digest(); }

int snap_alloc_cursors(void* a, uint64_t* transient_cursor, uint64_t* stable_cursor,
                       uint64_t* live_bytes) {
  if (!a) return SNAP_EINVAL;
  auto* t = static_cast<Tracker*>(a);
  if (transient_cursor) *transient_cursor = t->t_cur;
  if (stable_cursor) *stable_cursor = t->s_cur;
  if (live_bytes) *live_bytes = t->live_bytes;
  return SNAP_OK;
}

int snap_alloc_snapshot(void* a, uint64_t* words, uint64_t cap, uint64_t* n) {
  if (!a || !n) return SNAP_EINVAL;
  auto w = static_cast<Tracker*>(a)->save();
  *n = w.size();
  if (words) {
    if (cap < w.size()) return SNAP_EINVAL;
    std::copy(w.begin(), w.end(), words);
  }
  return SNAP_OK;
}

int snap_alloc_restore(void* a, const uint64_t* words, uint64_t n) {
  if (!a || !words) return SNAP_EINVAL;
  return static_cast<Tracker*>(a)->load(words, n);
}

}  // extern "C"
