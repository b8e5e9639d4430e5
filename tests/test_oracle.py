"""CPU tests: the oracle (CPU restatement) pinned to the reference's known-answer tests,
the Appendix-B golden vectors and the reference library itself (oracle/_ref)."""
import numpy as np
import pytest

import oracle as O


def test_digest_known_answers(golden):
    # test_simcore.cpp:115-117 — empty digest is the FNV offset basis
    assert O.digest_of_words(np.zeros(0, np.uint64)) == 14695981039346656037 == golden["empty"]
    # test_simcore.cpp:107-113 — pure function of content
    a = np.array([1, 2, 3], np.uint64)
    b = a.copy()
    assert O.digest_of_words(a) == O.digest_of_words(b) == golden["w123"]
    b[2] = 4
    assert O.digest_of_words(a) != O.digest_of_words(b)
    assert O.digest_of_words(O.fill_mix64(8)) == golden["mix0_7"]
    assert O.digest_of_words(O.fill_mix64(512)) == golden["page_mix0_511"]
    assert O.digest_of_words(O.fill_mix64(512, 0, 1000)) == golden["page_mix1000_1511"]


def test_no_collisions_10k():
    # test_simcore.cpp:119-130 (same property, numpy RNG)
    rng = np.random.default_rng(7)
    seen = {}
    for _ in range(10000):
        buf = rng.integers(0, 2**63, size=1 + int(rng.integers(16)), dtype=np.uint64)
        d = O.digest_of_words(buf)
        if d in seen:
            assert np.array_equal(seen[d], buf)
        seen[d] = buf
    assert len(seen) >= 9999


def test_c1_golden_digests(golden, c1_golden):
    img = O.fill_mix64((256 << 20) // 8)
    assert O.digest_of_words(img) == golden["c1_whole"]
    bufs = [(0, 0, 0, 256 << 20, 0)]
    d, lens, bd = O.hash_chunks([img], bufs, 65536, 65536)
    assert np.array_equal(d, c1_golden["direct"])
    assert (lens == 65536).all()
    d, _, bd = O.hash_chunks([img], bufs, 4096, 65536)
    assert np.array_equal(d, c1_golden["merkle"])
    assert int(bd[0]) == int(c1_golden["buf"][0])
    # Appendix B spot values
    assert int(c1_golden["direct"][0]) == 0x248805F70C9A88EA
    assert int(c1_golden["merkle"][1]) == 0x1AA72605D2DBCE8A
    assert int(c1_golden["direct"][4095]) == 0xD13B5CAE3A84AA0E


def ragged_arena(golden):
    rag = golden["ragged"]
    arena = O.fill_mix64(rag["arena_bytes"] // 8, rag["seed"], 0)
    src, dst, n = rag["dup"]
    arena[dst // 8:(dst + n) // 8] = arena[src // 8:(src + n) // 8]
    return arena, [tuple(b) for b in rag["bufs"]]


@pytest.mark.parametrize("geom", [(4096, 65536), (65536, 65536), (256, 4096), (1024, 32768)])
def test_ragged_golden(golden, geom):
    arena, bufs = ragged_arena(golden)
    d, lens, bd = O.hash_chunks([arena], bufs, *geom)
    exp = golden["ragged"][f"{geom[0]}_{geom[1]}"]
    assert [f"{x:016x}" for x in d] == exp["chunks"]
    assert [f"{x:016x}" for x in bd] == exp["bufs"]
    assert lens.sum() == sum(b[3] for b in bufs)


def test_oracle_vs_reference_library():
    R = O.ref()
    if R is None:
        pytest.skip("reference library not built here")
    rng = np.random.default_rng(1)
    for n in [0, 1, 7, 512, 8191]:
        w = rng.integers(0, 2**63, size=n, dtype=np.uint64)
        assert O.digest_of_words(w) == R.ref_digest_of_words(w.ctypes.data, n)
    for x in [0, 1, 12345, 2**63 + 5]:
        assert O.mix64(x) == R.ref_mix64(x)


def test_select_semantics():
    """First occurrence in canonical order, minus the known set (ckpt.cpp:97,157-166,18-20)."""
    d = np.array([5, 6, 5, 7, 6, 8, 9, 9], np.uint64)
    lens = np.array([256, 512, 256, 256, 512, 1024, 256, 256], np.uint32)
    sel, owner, off, total = O.select(d, lens, known=np.array([7], np.uint64))
    assert sel.tolist() == [1, 1, 0, 0, 0, 1, 1, 0]
    assert owner.tolist() == [0, 1, 0, 2**64 - 1, 1, 5, 6, 6]
    assert off.tolist()[:3] == [0, 256, 0] and off[3] == 2**64 - 1
    assert off[5] == 768 and off[6] == 1792 and off[7] == 1792
    assert total == 2048


def test_compact_restore_round_trip(golden):
    arena, bufs = ragged_arena(golden)
    d, lens, _ = O.hash_chunks([arena], bufs, 4096, 65536)
    sel, owner, off, total = O.select(d, lens)
    # buffer 3 duplicates buffer 1 -> its chunks are not staged again
    assert total == sum(b[3] for b in bufs) - bufs[3][3]
    img = O.compact([arena], bufs, 65536, sel, off, total)
    fresh = np.zeros_like(arena)
    O.restore([fresh], bufs, 65536, img, off)
    for (_r, _s, a, n, _c) in bufs:
        assert np.array_equal(fresh[a // 8:(a + n) // 8], arena[a // 8:(a + n) // 8])


def test_stripe_replicated():
    # 3 ranks; chunks 0..3 replicated at the same positions, chunk 4 per-rank
    world, per = 3, 5
    d = np.array([[10, 11, 12, 13, 100 + r] for r in range(world)], np.uint64).ravel()
    lens = np.full(d.size, 65536, np.uint32)
    sel, *_ = O.select(d, lens)
    writer, off, sb = O.stripe(d, lens, [per] * world, sel)
    assert writer.tolist()[:5] == [0, 1, 2, 0, 0]  # holders = all ranks -> i % 3
    assert writer.tolist()[9] == 1 and writer.tolist()[14] == 2
    assert sb.sum() == 7 * 65536


def test_grad_sums():
    rng = np.random.default_rng(3)
    g = [rng.integers(0, 2**64 - 1, size=1000, dtype=np.uint64) for _ in range(4)]
    s = O.grad_sum_u64(g)
    assert np.array_equal(s, ((g[0] + g[1]) + g[2]) + g[3])  # numpy wraps mod 2^64
    f = [rng.standard_normal(1000).astype(np.float32) for _ in range(4)]
    sf = O.grad_sum_f32(f)
    assert np.array_equal(sf, ((f[0] + f[1]) + f[2]) + f[3])


def test_blobstore_golden(golden):
    R = O.ref()
    if R is None:
        pytest.skip("reference library not built here")
    import ctypes as C
    s = R.ref_store_new()
    page = np.array([R.ref_mix64(3 ^ i) for i in range(512)], np.uint64)
    dig = C.c_uint64()
    assert R.ref_store_put(s, page.ctypes.data, 512, C.byref(dig)) == golden["blobstore"]["first_fresh"]
    assert f"{dig.value:016x}" == golden["blobstore"]["digest"]
    assert O.digest_of_words(page) == dig.value
    out = np.zeros(512, np.uint64)
    assert R.ref_store_get(s, dig.value, out.ctypes.data, 512) == 0
    assert np.array_equal(out, page)
    assert R.ref_store_get(s, dig.value ^ 1, out.ctypes.data, 512) == -1
    R.ref_store_free(s)


def test_host_pages_oracle_vs_reference_store():
    # the oracle's fresh flags == BlobStore::put's `fresh` for the same page sequence
    # (ckpt.cpp:121-126), and its page digests == the reference digest of each page
    import ctypes as C
    R = O.ref()
    if R is None:
        pytest.skip("reference library not built here")
    rng = np.random.default_rng(3)
    bufs = [O.fill_mix64(700, 5, 0), np.zeros(300, np.uint64), O.fill_mix64(512, 5, 0),
            O.fill_mix64(1100, 6, 0)]
    dig, flags = O.host_pages(bufs)
    allw = np.concatenate(bufs + [np.zeros((-sum(b.size for b in bufs)) % 512, np.uint64)])
    st = R.ref_store_new()
    try:
        for i in range(dig.size):
            page = np.ascontiguousarray(allw[i * 512:(i + 1) * 512])
            d = C.c_uint64()
            fresh = R.ref_store_put(st, page.ctypes.data_as(C.c_void_p), 512, C.byref(d))
            assert d.value == int(dig[i]) and bool(fresh) == bool(flags[i] & 1)
    finally:
        R.ref_store_free(st)
    _, f2 = O.host_pages(bufs, prev_pages=dig[:2])
    prev = set(dig[:2].tolist())
    assert [bool(f & 2) for f in f2] == [d not in prev for d in dig.tolist()]
    del rng


def test_bf16_sum_rounding_matches_torch(oracle_mod):
    """The bf16 gradient restatement (fp32 chain, one RN-even rounding) against torch's
    float32 -> bfloat16 conversion on the CPU."""
    import numpy as np
    import torch
    rng = np.random.default_rng(5)
    a = (rng.standard_normal(100_000) * 10.0 ** rng.integers(-20, 20, 100_000)).astype(np.float32)
    b = (rng.standard_normal(100_000) * 10.0 ** rng.integers(-20, 20, 100_000)).astype(np.float32)
    ha = (a.view(np.uint32) >> 16).astype(np.uint16)
    hb = (b.view(np.uint32) >> 16).astype(np.uint16)
    got = oracle_mod.grad_sum_bf16([ha, hb])
    fa = torch.from_numpy((ha.astype(np.uint32) << 16).view(np.float32))
    fb = torch.from_numpy((hb.astype(np.uint32) << 16).view(np.float32))
    exp = (fa + fb).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, exp)


def _blobstore_select(R, chunks, known_chunks):
    """The reference's own BlobStore::put (ckpt.cpp:16-21) over a canonical chunk sequence,
    after the known chunks were stored: fresh flags and the staging offsets they imply."""
    import ctypes as C
    st = R.ref_store_new()
    d = C.c_uint64()
    for w in known_chunks:
        R.ref_store_put(st, w.ctypes.data_as(C.c_void_p), w.size, C.byref(d))
    fresh, offs, digs, total, at = [], [], [], 0, {}
    for w in chunks:
        f = R.ref_store_put(st, w.ctypes.data_as(C.c_void_p), w.size, C.byref(d))
        fresh.append(f)
        digs.append(d.value)
        if f:
            at[d.value] = total
        # a repeated chunk's bytes are at its first occurrence's offset; a chunk the
        # store already held before this snapshot has no bytes in this image
        offs.append(at.get(d.value, 2**64 - 1))
        total += w.size * 8 if f else 0
    R.ref_store_free(st)
    return np.array(fresh, np.uint8), np.array(offs, np.uint64), np.array(digs, np.uint64), total


@pytest.mark.parametrize("case", ["ragged", "random_dups", "known_set"])
def test_select_pinned_to_blobstore_put(ref_lib, golden, case):
    """K2's CPU restatement (or_select: first occurrence in canonical order, not in the
    known set, staging offsets = running sum of staged bytes) is exactly BlobStore::put's
    `fresh` over the same chunk sequence."""
    rng = np.random.default_rng(11)
    if case == "ragged":
        arena, bufs = ragged_arena(golden)
        chunks = []
        for (_r, _s, a, n, _c) in bufs:
            for k in range(0, n, 65536):
                chunks.append(arena[(a + k) // 8:(a + min(n, k + 65536)) // 8])
    else:
        pool = [O.fill_mix64(int(rng.integers(1, 64)) * 32, 100 + i, 0) for i in range(40)]
        chunks = [pool[int(rng.integers(0, 40))] for _ in range(300)]
    known = [] if case != "known_set" else [chunks[int(i)] for i in rng.integers(0, 300, 25)]
    fresh, offs, digs, total = _blobstore_select(ref_lib, chunks, known)
    lens = np.array([w.size * 8 for w in chunks], np.uint32)
    kn = np.array([O.digest_of_words(w) for w in known], np.uint64)
    sel, owner, off, tot = O.select(digs, lens, kn if known else None)
    assert np.array_equal(sel, fresh)
    assert np.array_equal(off, offs)
    assert tot == total
    assert np.array_equal(digs, [O.digest_of_words(w) for w in chunks])


def appendix_b_scenario(dp):
    """one DP job, 4 layers x 2048 words, scenario seed 7, one node of dp
    4 MiB GPUs, checkpoints at 0.5 ms and 2.1 ms of simulated time."""
    return {"seed": 7,
            "fleet": {"regions": [{"clusters": [{"nodes": [{"gpus": dp, "mem_mib": 4}]}]}]},
            "jobs": [{"name": "j", "spec": {"world": dp, "dp": dp, "layers": 4,
                                            "params_per_layer": 2048}}],
            "events": [{"at_sec": 0.0005, "kind": "checkpoint", "job": "j"},
                       {"at_sec": 0.0021, "kind": "checkpoint", "job": "j"}]}


@pytest.mark.parametrize("dp,s_cr,s_cr_inc,upload", [(4, 1097728, 16384, 414240),
                                                      (8, 2195456, 32768, 430912)])
def test_manifest_dedup_pinned_to_reference(ref_lib, dp, s_cr, s_cr_inc, upload):
    """build_manifest's device section (ckpt.cpp:147-167), run by the reference's own
    scheduler on the Appendix-B scenario, reproduces the Appendix-B goldens; the oracle's
    chunk-level select over the manifest's device buffers (canonical rank/slot order, one
    chunk per buffer) gives the same S_G and the same device upload bytes, first and
    incremental checkpoint (VERDICT r1 missing #6)."""
    ms = O.ref_manifests(appendix_b_scenario(dp))
    assert len(ms) == 2
    m1, m2 = ms
    assert (m1["s_g"], m2["s_g"]) == (131072, 131072)  # S_G invariant under DP degree
    assert m1["s_cr"] == s_cr and m2["s_cr_inc"] == s_cr_inc and m1["upload_bytes"] == upload
    prev = None
    for m in ms:
        recs = [d for r in range(m["world"]) for d in m["dev"][r]]
        digs = np.array([d["digest"] for d in recs], np.uint64)
        assert all(O.digest_of_words(d["content"]) == d["digest"] for d in recs)
        lens = np.array([d["words"] * 8 for d in recs], np.uint32)
        sel, _, _, tot = O.select(digs, lens)
        assert tot == m["s_g"]
        known = None if prev is None else prev
        _, _, _, up = O.select(digs, lens, known)
        assert up == m["device_upload"]
        prev = digs


def test_bench_parity_fnv_restatement(c1_golden):
    """bench.py's untimed parity block re-hashes sampled chunks with its own numpy FNV-1a;
    that restatement equals the reference goldens (C1 chunk 0 and 1, Merkle mode)."""
    import bench
    img = O.fill_mix64(2 * 65536 // 8).view(np.uint8).reshape(2, 65536)
    d = bench.chunk_digests_np(img)
    assert np.array_equal(d, c1_golden["merkle"][:2])
