"""Generates tests/golden/* from the REFERENCE library (oracle/_ref/libfleetsim_ref.so,
compiled from /root/reference/proj/src by oracle/Makefile). Only the reference's own
sim::digest_of_words / mix64 / BlobStore / BidiAllocator / DeviceLayout::carve are called
here, never the CPU restatement, so the fixtures pin the restatement and the CUDA path to
the reference. Re-run with `python tests/golden/make_golden.py` in a container that has
/root/reference; the outputs are committed.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

R = oracle.ref()
assert R is not None, "build oracle/_ref first (make -C oracle)"


def mixes(n, seed=0, base=0):
    return np.array([R.ref_mix64(seed ^ (base + i)) for i in range(n)], dtype=np.uint64)


def dw(words):
    w = np.ascontiguousarray(words, dtype=np.uint64)
    return int(R.ref_digest_of_words(w.ctypes.data, w.size))


def chunk_digests(arena, bufs, page_bytes, chunk_bytes):
    """Reference digests over the chunk grid: digest_of_words on every page span, then
    digest_of_words over the page digests (or the chunk span in direct mode)."""
    out, per_buf = [], []
    for (_r, _s, addr, nbytes, _c) in bufs:
        cd = []
        for off in range(0, nbytes, chunk_bytes):
            ln = min(chunk_bytes, nbytes - off)
            span = arena[(addr + off) // 8:(addr + off + ln) // 8]
            if page_bytes == chunk_bytes:
                cd.append(dw(span))
            else:
                pds = [dw(span[q // 8:(q + min(page_bytes, ln - q)) // 8])
                       for q in range(0, ln, page_bytes)]
                cd.append(dw(np.array(pds, dtype=np.uint64)))
        out += cd
        per_buf.append(dw(np.array(cd, dtype=np.uint64)))
    return out, per_buf


def main():
    g = {}
    # SURVEY.md Appendix B + test_simcore.cpp:107-117
    g["empty"] = dw(np.zeros(0, np.uint64))
    g["w123"] = dw(np.array([1, 2, 3], np.uint64))
    g["mix0_7"] = dw(mixes(8))
    g["page_mix0_511"] = dw(mixes(512))
    g["page_mix1000_1511"] = dw(mixes(512, 0, 1000))

    # C1 image words[i] = mix64(i), 256 MiB: full digest vectors (direct + merkle)
    n_words = (256 << 20) // 8
    img = np.empty(n_words, np.uint64)
    oracle.lib().or_fill_mix64(img.ctypes.data, n_words, 0, 0)
    assert int(img[12345]) == R.ref_mix64(12345)
    g["c1_whole"] = dw(img)
    c1 = [(0, 0, 0, 256 << 20, 0)]
    direct, _ = chunk_digests(img, c1, 65536, 65536)
    merkle, c1_buf = chunk_digests(img, c1, 4096, 65536)
    np.savez_compressed(os.path.join(HERE, "c1_digests.npz"),
                        direct=np.array(direct, np.uint64), merkle=np.array(merkle, np.uint64),
                        buf=np.array(c1_buf, np.uint64))

    # Ragged multi-buffer layout (256-B multiples, partial pages/chunks, duplicates):
    # content = mix64(7 ^ i) over a 4 MiB arena; buffer 3 duplicates buffer 1's bytes.
    arena_bytes = 4 << 20
    arena = np.empty(arena_bytes // 8, np.uint64)
    oracle.lib().or_fill_mix64(arena.ctypes.data, arena.size, 7, 0)
    bufs = [(0, 0, 0, 256, 0), (0, 1, 4096, 65536 + 4096 + 256, 1), (0, 2, 200704, 131072, 2),
            (0, 3, 524288, 65536 + 4096 + 256, 1), (0, 4, 1048576, 3 * 65536 + 768, 3),
            (0, 5, 2097152, 4096, 4)]
    arena[524288 // 8:(524288 + 65536 + 4096 + 256) // 8] = \
        arena[4096 // 8:(4096 + 65536 + 4096 + 256) // 8]
    rag = {"bufs": bufs, "seed": 7, "arena_bytes": arena_bytes,
           "dup": [4096, 524288, 65536 + 4096 + 256]}
    for pb, cb in [(4096, 65536), (65536, 65536), (256, 4096), (1024, 32768)]:
        d, bd = chunk_digests(arena, bufs, pb, cb)
        rag[f"{pb}_{cb}"] = {"chunks": [f"{x:016x}" for x in d], "bufs": [f"{x:016x}" for x in bd]}
    g["ragged"] = rag

    # BlobStore semantics (ckpt.cpp:16-29): fresh puts, dedup, digest-verified get.
    s = R.ref_store_new()
    dig = C.c_uint64()
    page = mixes(512, 3, 0)
    f1 = R.ref_store_put(s, page.ctypes.data, 512, C.byref(dig))
    d1 = dig.value
    f2 = R.ref_store_put(s, page.ctypes.data, 512, C.byref(dig))
    g["blobstore"] = {"first_fresh": f1, "second_fresh": f2, "digest": f"{d1:016x}",
                      "total_bytes": int(R.ref_store_total_bytes(s)),
                      "count": int(R.ref_store_count(s))}
    R.ref_store_free(s)

    # DeviceLayout::carve (splice.cpp:7-19)
    carve = []
    for mem, mb, sl in [(1 << 20, 65536, 0.02), (4 << 20, 1 << 20, 0.02), (256 << 20, 4096, 0.0),
                        (183359 << 20, 80 << 30, 0.02), (8192, 8192, 0.5)]:
        out = (C.c_uint64 * 3)()
        rc = R.ref_carve(mem, mb, sl, out)
        carve.append({"mem": mem, "max_buf": mb, "slack": sl, "rc": rc,
                      "out": list(out) if rc == 0 else None})
    g["carve"] = carve

    # BidiAllocator address sequence (alloc.cpp:62-108) for a scripted op list.
    a = R.ref_alloc_new(0, 1 << 20)
    rng = np.random.default_rng(11)
    ops, live = [], []
    addr = C.c_uint64()
    for i in range(300):
        if live and rng.random() < 0.4:
            k = int(rng.integers(len(live)))
            x = live.pop(k)
            rc = R.ref_alloc_free(a, x)
            ops.append(["free", x, rc])
        else:
            st = int(rng.random() < 0.5)
            nb = int(rng.integers(1, 9000))
            rc = R.ref_alloc_alloc(a, nb, st, C.byref(addr))
            ops.append(["alloc", nb, st, rc, addr.value if rc == 0 else None])
            if rc == 0:
                live.append(addr.value)
    tc, sc, lb = C.c_uint64(), C.c_uint64(), C.c_uint64()
    R.ref_alloc_cursors(a, C.byref(tc), C.byref(sc), C.byref(lb))
    g["alloc"] = {"ops": ops, "stable_digest": f"{R.ref_alloc_stable_digest(a):016x}",
                  "cursors": [tc.value, sc.value, lb.value]}
    R.ref_alloc_free_obj(a)

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
