// The reference's device/digest unit tests (proj/tests/test_vdev.cpp:79-96,
// 171-179; test_simcore.cpp:107-117) restated against the B200 arena, plus the
// checkpoint/splice round trips through the C++ mirror. Needs a B200.
#include <filesystem>
#include <unistd.h>
#include <random>

#include "mini_test.hpp"
#include "snap.hpp"

using namespace snapb200;
using vdev::MemRange;

static u64 mix64(u64 x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

TEST_CASE("digest is a pure function of content") {
  vdev::Gpu g(0, 1 << 20);
  std::vector<u64> a(64), b(64);
  for (u64 i = 0; i < 64; ++i) a[i] = b[i] = mix64(i);
  g.write_words({0, 512}, a);
  g.write_words({4096, 512}, b);
  CHECK(g.digest({0, 512}) == g.digest({4096, 512}));
  b[63] ^= 1;
  g.write_words({4096, 512}, b);
  CHECK(!(g.digest({0, 512}) == g.digest({4096, 512})));
}

TEST_CASE("copy round trip preserves digests") {
  vdev::Gpu g(0, 1 << 20);
  std::vector<u64> content(64);
  for (u64 i = 0; i < 64; ++i) content[i] = mix64(i);
  g.write_words({0, 512}, content);
  auto d0 = g.digest({0, 512});
  auto host = g.words({0, 512});  // d2h, then h2d
  g.write_words({0, 512}, std::vector<u64>(64, 0));
  g.write_words({0, 512}, host);
  CHECK(g.digest({0, 512}) == d0);
  g.write_words({4096, 512}, host);  // d2d move to a different address
  CHECK(g.digest({4096, 512}) == d0);
}

TEST_CASE("modular integer reduction is order independent") {
  vdev::Gpu g(0, 1 << 20);
  std::mt19937_64 rng(5);
  std::vector<std::vector<u64>> v(4, std::vector<u64>(1024));
  for (auto& x : v)
    for (auto& w : x) w = rng();
  for (int r = 0; r < 4; ++r) g.write_words({u64(r) * 8192, 8192}, v[r]);
  coll::grad_sum(g, SNAP_U64, {0, 8192, 16384, 24576}, 32768, 1024);
  coll::grad_sum(g, SNAP_U64, {24576, 16384, 8192, 0}, 40960, 1024);
  CHECK(g.words({32768, 8192}) == g.words({40960, 8192}));
}

TEST_CASE("snapshot -> restore round trip is bit-exact") {
  vdev::Gpu g(0, 8 << 20);
  std::vector<u64> img((4 << 20) / 8);
  for (u64 i = 0; i < img.size(); ++i) img[i] = mix64(7 ^ i);
  g.write_words({0, 4 << 20}, img);
  ckpt::Snapshotter s(g);
  s.set_buffers({{0, 0, 0, 1 << 20, 0, 0}, {0, 1, 1 << 20, (3 << 20) - 768, 1, 0}});
  s.snapshot();
  CHECK(s.staged_bytes() == (4u << 20) - 768);
  g.write_words({0, 4 << 20}, std::vector<u64>(img.size(), 0));
  s.restore_self(/*verify=*/true);
  auto back = g.words({0, (4 << 20) - 768});
  CHECK(std::equal(back.begin(), back.end(), img.begin()));
}

TEST_CASE("splice: identical replicas move no bytes after the first switch") {
  vdev::Gpu g(0, 8 << 20);
  std::vector<u64> p((2 << 20) / 8);
  for (u64 i = 0; i < p.size(); ++i) p[i] = mix64(i);
  g.write_words({0, 2 << 20}, p);
  splice::Splicer sp(g, 16 << 20);
  std::vector<splice::RankBuf> bufs{{0, 0, 1 << 20, vdev::BufCat::Param, true, false},
                                    {1, 1 << 20, 1 << 20, vdev::BufCat::OptState, true, false}};
  for (int r = 0; r < 2; ++r) sp.set_rank_bufs(r, bufs);
  auto first = sp.switch_to(0, 1);
  auto second = sp.switch_to(1, 0);
  auto third = sp.switch_to(0, 1);
  CHECK(first.swap_out_bytes == (2u << 20));
  CHECK(second.swap_out_bytes == 0 && second.swap_in_bytes == 0);
  CHECK(third.swap_out_bytes == 0 && third.swap_in_bytes == 0);
  CHECK(third.resident_bytes == (2u << 20));
}

TEST_CASE("window tracker + persist/load through the C++ mirror") {
  vdev::Gpu g(0, 8 << 20);
  std::vector<u64> img((4 << 20) / 8);
  for (u64 i = 0; i < img.size(); ++i) img[i] = mix64(i ^ 77);
  g.write_words({0, 4 << 20}, img);
  std::vector<splice::RankBuf> bufs{{0, 0, 1 << 20, vdev::BufCat::Param, true, false},
                                    {1, 1 << 20, 2 << 20, vdev::BufCat::OptState, true, false},
                                    {2, 3 << 20, 1 << 20, vdev::BufCat::Grad, true, true}};
  splice::WindowTracker w(g);
  std::map<RankId, splice::ValidationRecord> recs;
  for (int r = 0; r < 2; ++r) {
    g.write_words({0, 4 << 20}, img);
    w.open(r, bufs);
    auto v = g.words({1 << 20, 256});
    v[3] ^= 0x55;  // the step touches the optimizer state only
    g.write_words({1 << 20, 256}, v);
    w.close(r, bufs, recs[r]);
  }
  CHECK(recs[0].mutations.size() == 1 && recs[0].mutations.count(1 << 20) == 1);
  CHECK(splice::validate_window(recs).pass);

  ckpt::Snapshotter s(g);
  s.set_buffers({{0, 0, 0, 1 << 20, 0, 0}, {0, 1, 1 << 20, 3 << 20, 1, 0}});
  s.snapshot();
  char tmpl[] = "/tmp/snap_cpp_XXXXXX";
  const std::string dir = mkdtemp(tmpl);
  auto st = s.persist(dir);
  CHECK(st.written == 64 && st.layout_chunks == 64);
  const auto before = g.words({0, 4 << 20});
  g.write_words({0, 4 << 20}, std::vector<u64>(img.size(), 0));
  auto ls = s.load(dir);
  CHECK(ls.layout_blobs == 64);
  const auto after = g.words({0, 4 << 20});
  CHECK(after == before);
  std::filesystem::remove_all(dir);
}

TEST_CASE("exact whole-range digest equals the reference FNV-1a") {
  vdev::Gpu g(0, 1 << 20);
  std::vector<u64> w(4096);
  for (u64 i = 0; i < w.size(); ++i) w[i] = mix64(i + 7);
  g.write_words({0, 32768}, w);
  u64 h = 14695981039346656037ull;  // sim.hpp:55-65 restated over the bytes
  for (u64 x : w)
    for (int k = 0; k < 8; ++k) {
      h ^= (x >> (8 * k)) & 0xff;
      h *= 0x100000001b3ull;
    }
  CHECK(g.digest_exact({0, 32768}).value == h);
}

TEST_CASE("splice: deferred result install reaches the inactive rank at its switch") {
  vdev::Gpu g(0, 8 << 20);
  splice::Splicer sp(g, 4 << 20);
  std::vector<splice::RankBuf> bufs = {{0, 0, 1 << 20, vdev::BufCat::Param, true, false},
                                       {1, 1 << 20, 64 << 10, vdev::BufCat::Grad, true, true}};
  sp.set_rank_bufs(0, bufs);
  sp.set_rank_bufs(1, bufs);
  std::vector<u64> res(8192);
  for (u64 i = 0; i < res.size(); ++i) res[i] = mix64(i ^ 0x77);
  g.write_words({4 << 20, 65536}, res);
  sp.switch_to(-1, 0);                                    // rank 0 active
  sp.install_result({0, 1}, {1 << 20, 1 << 20}, 4 << 20, 65536);
  CHECK(sp.pending_install_bytes(1) == 65536 && sp.pending_install_bytes(0) == 0);
  g.write_words({1 << 20, 65536}, std::vector<u64>(8192, 0));  // rank 0's next backward
  auto plan = sp.switch_to(0, 1);
  CHECK(plan.install_bytes == 65536);
  CHECK(g.words({1 << 20, 65536}) == res);
}

MINI_MAIN()
