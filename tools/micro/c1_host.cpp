// C1 snapshot / verified-restore per-call time from C++ (dev tool): the same
// loop as bench.py's c1 section without the Python call overhead.
//   g++ -O2 -std=c++17 -I include tools/micro/c1_host.cpp -o tools/micro/c1_host \
//       -Lpaper_2202_07848_b200 -lsnap -Wl,-rpath,$PWD/paper_2202_07848_b200
#include <chrono>
#include <cstdio>
#include <vector>

#include "snap.h"

#define CK(x)                                                            \
  do {                                                                   \
    int rc_ = (x);                                                       \
    if (rc_) {                                                           \
      std::printf("%s: %d %s\n", #x, rc_, snap_last_error(ctx));         \
      return 1;                                                          \
    }                                                                    \
  } while (0)

int main() {
  const uint64_t nbytes = 256ull << 20, nb = 4ull << 20;
  snap_ctx* ctx = nullptr;
  CK(snap_open(0, nbytes, &ctx));
  CK(snap_fill_mix64(ctx, 0, nbytes, 1, 0));
  std::vector<snap_buf> bufs;
  for (uint64_t i = 0; i < nbytes / nb; ++i) bufs.push_back({0, int32_t(i), i * nb, nb, 0, 0});
  snap_geom geom{4096, 65536};
  uint64_t nchunks = 0;
  CK(snap_set_buffers(ctx, bufs.data(), bufs.size(), &geom, &nchunks));
  for (int i = 0; i < 5; ++i) {
    CK(snap_snapshot(ctx));
    CK(snap_restore_self(ctx, 1));
  }
  CK(snap_sync(ctx));
  const int reps = 50;
  for (int round = 0; round < 3; ++round) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) CK(snap_snapshot(ctx));
    CK(snap_sync(ctx));
    auto t1 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) CK(snap_restore_self(ctx, 1));
    auto t2 = std::chrono::steady_clock::now();
    std::printf("snapshot %.1f us/call  restore(verify) %.1f us/call\n",
                std::chrono::duration<double, std::micro>(t1 - t0).count() / reps,
                std::chrono::duration<double, std::micro>(t2 - t1).count() / reps);
  }
  return snap_close(ctx);
}
