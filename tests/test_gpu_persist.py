"""GPU tests of the on-disk format: snap_persist writes the staged chunks
as BlobStore::persist does (ckpt.cpp:42-52, blobs/<2hex>/<16hex>), snap_load restores a
rank from the directory (restore_job materialization, ckpt.cpp:504-533) with the
BlobStore::get digest verification (ckpt.cpp:26-27)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

ARENA = 48 << 20


def layout(rng, arena_bytes, dup_every=5):
    """Random 256-B aligned buffers (ragged tails) + the host image with duplicated buffers."""
    img = O.fill_mix64(arena_bytes // 8, int(rng.integers(1, 1 << 30)), 0)
    bufs, addr = [], 0
    while True:
        nb = int(rng.integers(1, 900)) * 256
        if addr + nb > arena_bytes:
            break
        bufs.append((0, len(bufs), addr, nb, int(rng.integers(0, 5))))
        addr += nb + int(rng.integers(0, 4)) * 256
    # duplicate some buffers' content (cross-buffer dedup: one blob for both)
    for i in range(dup_every, len(bufs), dup_every):
        s, d = bufs[i - dup_every], bufs[i]
        n = min(s[3], d[3])
        img[d[2] // 8:(d[2] + n) // 8] = img[s[2] // 8:(s[2] + n) // 8]
    return img, bufs


def tree(root):
    return {os.path.relpath(os.path.join(dp, f), root): open(os.path.join(dp, f), "rb").read()
            for dp, _, fs in os.walk(root) for f in fs}


def blob_files(root):
    return {k: v for k, v in tree(root).items() if k.startswith("blobs/")}


def chunks_of(img, bufs, chunk):
    out = []
    for (_, _, a, n, _) in bufs:
        for o in range(0, n, chunk):
            out.append(img[(a + o) // 8:(a + min(n, o + chunk)) // 8])
    return out


def test_persist_files_identical_to_reference_blobstore(snap, ref_lib, tmp_path):
    # page == chunk: blob name = digest_of_words(content), so the reference BlobStore fed
    # the same chunks must persist the very same directory
    rng = np.random.default_rng(1)
    img, bufs = layout(rng, ARENA)
    with snap.Ctx(0, ARENA) as c:
        c.write(0, img)
        c.set_buffers(bufs, 65536, 65536)
        c.snapshot()
        st = c.persist(tmp_path / "ours")
    st_ref = ref_lib.ref_store_new()
    try:
        for w in chunks_of(img, bufs, 65536):
            w = np.ascontiguousarray(w)
            d = C.c_uint64()
            ref_lib.ref_store_put(st_ref, w.ctypes.data_as(C.c_void_p), w.size, C.byref(d))
        nref = ref_lib.ref_store_count(st_ref)
        assert ref_lib.ref_store_persist(st_ref, str(tmp_path / "ref").encode()) == 0
    finally:
        ref_lib.ref_store_free(st_ref)
    ours, ref = blob_files(tmp_path / "ours"), blob_files(tmp_path / "ref")
    assert len(ours) == nref == st["blobs"] == st["written"] and st["present"] == 0
    assert ours == ref
    # names: oracle digest of the content
    for k, v in ours.items():
        assert k == O.blob_rel_path(O.digest_of_words(np.frombuffer(v, np.uint64)))


@pytest.mark.parametrize("geom", [(4096, 65536), (256, 8192), (65536, 65536)])
def test_persist_load_round_trip(snap, tmp_path, geom):
    rng = np.random.default_rng(2 + geom[0])
    img, bufs = layout(rng, ARENA)
    d_dir = tmp_path / "ck"
    with snap.Ctx(0, ARENA) as c:
        c.write(0, img)
        c.set_buffers(bufs, *geom)
        c.snapshot()
        d, lens, bd = c.digests(buf_digests=True)
        _, _, _, sbytes, schunks = c.selection()
        st = c.persist(d_dir, threads=8)
        assert st["blobs"] == schunks == st["written"] and st["bytes"] == sum(
            len(v) for v in blob_files(d_dir).values())
        assert st["layout_chunks"] == c.nchunks and st["layout_blobs"] == len(set(d.tolist()))
        # blob contents = the oracle's chunk bytes
        od, olens, _ = O.hash_chunks([img], bufs, *geom)
        assert np.array_equal(d, od)
        files = blob_files(d_dir)
        for w, dg in zip(chunks_of(img, bufs, geom[1]), od):
            assert files[O.blob_rel_path(int(dg))] == w.tobytes()
        # manifest: device section with the reference's field names
        m = json.load(open(d_dir / "manifest.dev.0.json"))
        assert m["geometry"] == {"page_bytes": geom[0], "chunk_bytes": geom[1]}
        assert [(r["slot"], r["addr"], r["words"], r["cat"], r["digest"]) for r in m["dev"]] == [
            (b[1], b[2], b[3] // 8, b[4], int(x)) for b, x in zip(bufs, bd)]
        assert m["sizes"]["upload_bytes"] == st["bytes"]
    # a fresh context (zeroed arena) restores the image from the directory alone
    with snap.Ctx(0, ARENA) as c2:
        ls = c2.load(d_dir, threads=8)
        assert ls["blobs"] == st["layout_blobs"] and ls["layout_chunks"] == st["layout_chunks"]
        got = c2.read(0, ARENA).view(np.uint64)
        for (_, _, a, n, _) in bufs:
            assert np.array_equal(got[a // 8:(a + n) // 8], img[a // 8:(a + n) // 8])
        # the loaded layout is installed: hashing it reproduces the persisted digests
        c2.hash()
        d2, _ = c2.digests()
        assert np.array_equal(d2, d)


def test_incremental_persist_writes_only_dirty_chunks(snap, tmp_path):
    rng = np.random.default_rng(9)
    img, bufs = layout(rng, ARENA, dup_every=1000)
    with snap.Ctx(0, ARENA) as c:
        c.write(0, img)
        c.set_buffers(bufs)
        c.snapshot()
        st0 = c.persist(tmp_path)
        c.known_commit()
        d0, lens = c.digests()
        # dirty ~5 % of the chunks (xor into word 0, C4's mutation)
        starts = np.concatenate([[0], np.cumsum([(b[3] + 65535) // 65536 for b in bufs])])
        caddr = [b[2] + o for b in bufs for o in range(0, b[3], 65536)]
        dirty = sorted(set(int(x) for x in rng.choice(len(caddr), max(1, len(caddr) // 20),
                                                       replace=False)))
        c.xor_words([caddr[i] for i in dirty], 0x5A5A)
        img2 = img.copy()
        for i in dirty:
            img2[caddr[i] // 8] ^= np.uint64(0x5A5A)
        c.snapshot()
        st1 = c.persist(tmp_path)
        assert st1["written"] == st1["blobs"] == len(dirty) and st1["present"] == 0
        assert len(blob_files(tmp_path)) == st0["written"] + len(dirty)
        assert starts[-1] == c.nchunks
    # the newest layout restores from old + new blobs together
    with snap.Ctx(0, ARENA) as c2:
        c2.load(tmp_path)
        got = c2.read(0, ARENA).view(np.uint64)
        for (_, _, a, n, _) in bufs:
            assert np.array_equal(got[a // 8:(a + n) // 8], img2[a // 8:(a + n) // 8])


def test_persist_from_host_staging_and_repersist_skips(snap, tmp_path):
    nbytes = 96 << 20
    img = O.fill_mix64(nbytes // 8, 31, 0)
    bufs = [(0, 0, 0, 40 << 20, 0), (0, 1, 40 << 20, (30 << 20) + 512, 1),
            (0, 2, 80 << 20, 16 << 20, 2)]
    pin = snap.PinnedHost(nbytes)
    pin.array[:] = img.view(np.uint8)
    out = snap.PinnedHost(nbytes)
    with snap.Ctx(0, nbytes) as c:
        c.set_buffers(bufs)
        staged = c.snapshot_host(pin.ptr, 0, nbytes, out.ptr, nbytes)
        st = c.persist(tmp_path, host_ptr=out.ptr, host_bytes=staged)
        assert st["bytes"] == staged
        again = c.persist(tmp_path)  # device staging path, every blob already present
        assert again["written"] == 0 and again["present"] == st["blobs"]
    with snap.Ctx(0, nbytes) as c2:
        c2.load(tmp_path)
        got = c2.read(0, nbytes).view(np.uint64)
        for (_, _, a, n, _) in bufs:
            assert np.array_equal(got[a // 8:(a + n) // 8], img[a // 8:(a + n) // 8])


def test_load_detects_corrupt_truncated_and_missing_blobs(snap, tmp_path):
    rng = np.random.default_rng(4)
    img, bufs = layout(rng, 8 << 20)
    with snap.Ctx(0, 8 << 20) as c:
        c.write(0, img)
        c.set_buffers(bufs)
        c.snapshot()
        c.persist(tmp_path)
    files = sorted(p for p in blob_files(tmp_path))
    victim = tmp_path / files[len(files) // 2]
    good = victim.read_bytes()
    with snap.Ctx(0, 8 << 20) as c2:
        # flipped byte: restored, re-hashed, digest mismatch -> SimFault
        victim.write_bytes(bytes([good[0] ^ 1]) + good[1:])
        with pytest.raises(snap.SnapFault):
            c2.load(tmp_path)
        # without verification the corrupt bytes land (caller opted out)
        c2.load(tmp_path, verify=False)
        victim.write_bytes(good[:-8])  # truncated
        with pytest.raises(snap.SnapFault):
            c2.load(tmp_path)
        victim.unlink()  # missing
        with pytest.raises(snap.SnapFault, match="missing blob"):
            c2.load(tmp_path)
        victim.write_bytes(good)
        c2.load(tmp_path)
        # a damaged layout file is rejected before anything is written
        lp = tmp_path / "layout.0.snapl"
        raw = bytearray(lp.read_bytes())
        raw[60] ^= 0xFF
        lp.write_bytes(bytes(raw))
        with pytest.raises(snap.SnapError):
            c2.load(tmp_path)
        with pytest.raises(snap.SnapError):
            c2.load(tmp_path, rank=7)  # no such layout


def test_migrate_time_sliced_ranks_through_the_blob_store(snap, tmp_path):
    """restore_job on a new GPU for a 2-way time-sliced job (ckpt.cpp:504-533): the active
    rank is materialized in the arena (snap_load), the co-resident rank's chunks are
    seeded into the HBM chunk cache (snap_splice_load); switching then restores each
    rank's bytes exactly — P/O identical across the replicas stay resident, only the
    gradients move."""
    arena = 16 << 20
    po = [(0, 0, 0, 3 << 20, 0), (0, 1, 3 << 20, (2 << 20) + 768, 1)]   # identical replicas
    gbuf = (0, 2, 6 << 20, 1 << 20, 2)                                    # per-rank gradient
    state = {}

    def held(c, bufs):  # the bytes the rank's buffers hold (gaps are not state)
        return [c.read(b[2], b[3]) for b in bufs]

    def same(a, b):
        return all(np.array_equal(x, y) for x, y in zip(a, b))

    with snap.Ctx(0, arena) as src:
        for r in range(2):
            src.fill_mix64(0, 6 << 20, 42, 0)            # same P/O on both ranks
            src.fill_mix64(6 << 20, 1 << 20, 100 + r, 0)  # different G
            bufs = [(r,) + b[1:] for b in po] + [(r,) + gbuf[1:]]
            src.set_buffers(bufs)
            src.snapshot()
            src.persist(tmp_path, layout_rank=r)
            state[r] = (bufs, held(src, bufs))
    with snap.Ctx(0, arena) as dst:
        dst.splice_init(16 << 20)  # room for the seed + a worst-case swap-out
        ld = dst.load(tmp_path, rank=0)                  # active rank -> arena (verified)
        assert ld["layout_chunks"] > 0
        assert same(held(dst, state[0][0]), state[0][1])
        dst.splice_set_rank(0, state[0][0])
        seed = dst.splice_load(tmp_path, layout_rank=1, splice_rank=1)
        assert seed["layout_bufs"] == 3
        s01 = dst.splice_switch(0, 1)
        assert same(held(dst, state[1][0]), state[1][1])
        po_bytes = (3 << 20) + (2 << 20) + 768
        assert s01["resident_bytes"] == po_bytes and s01["swap_in_bytes"] == 1 << 20
        s10 = dst.splice_switch(1, 0)
        assert same(held(dst, state[0][0]), state[0][1])
        assert s10["swap_in_bytes"] == 1 << 20 and s10["resident_bytes"] == po_bytes
        # a missing blob of the co-resident rank is a fault, not silent garbage
        with snap.Ctx(0, arena) as probe:
            probe.load(tmp_path, rank=1)
            d1, _ = probe.digests()
        os.remove(tmp_path / O.blob_rel_path(int(d1[-1])))
        with pytest.raises(snap.SnapFault):
            dst.splice_load(tmp_path, layout_rank=1, splice_rank=2)
