"""oracle — TEST INFRASTRUCTURE ONLY.

ctypes bindings to
  * liboracle.so            the CPU restatement (snap_oracle.c), and
  * _ref/libfleetsim_ref.so the reference library itself, compiled from
                            /root/reference/proj/src by oracle/Makefile.

Only tests/, __graft_entry__.smoke() (as the checker) and bench.py's
cpu_baseline / --impl reference legs may import this package. The product
(paper_2202_07848_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None
_ref = None

U64P = C.POINTER(C.c_uint64)


class OrBuf(C.Structure):
    """or_buf / snap_buf: RankBuf/DevRec (splice.hpp:26-34, ckpt.hpp:64-71)."""

    _fields_ = [
        ("rank", C.c_uint32),
        ("slot", C.c_int32),
        ("addr", C.c_uint64),
        ("bytes", C.c_uint64),
        ("cat", C.c_int32),
        ("flags", C.c_uint32),
    ]


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.or_fnv1a.restype = C.c_uint64
        L.or_fnv1a.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.or_digest_of_words.restype = C.c_uint64
        L.or_digest_of_words.argtypes = [C.c_void_p, C.c_uint64]
        L.or_mix64.restype = C.c_uint64
        L.or_mix64.argtypes = [C.c_uint64]
        L.or_fill_mix64.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_num_chunks.restype = C.c_uint64
        L.or_num_chunks.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32]
        L.or_hash.restype = C.c_int
        L.or_hash.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.or_select.restype = C.c_uint64
        L.or_select.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_stripe.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_compact.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p,
                                 C.c_void_p, C.c_void_p]
        L.or_restore.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p,
                                 C.c_void_p]
        L.or_grad_sum_u64.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p]
        L.or_grad_sum_f32.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p]
        L.or_grad_sum_bf16.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p]
        _lib = L
    return _lib


def ref():
    """The reference library (None when it was never built here)."""
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libfleetsim_ref.so")
        if not os.path.exists(path):
            return None
        L = C.CDLL(path)
        L.ref_digest_of_words.restype = C.c_uint64
        L.ref_digest_of_words.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_digest_of_bytes.restype = C.c_uint64
        L.ref_digest_of_bytes.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_mix64.restype = C.c_uint64
        L.ref_mix64.argtypes = [C.c_uint64]
        L.ref_store_new.restype = C.c_void_p
        L.ref_store_free.argtypes = [C.c_void_p]
        L.ref_store_put.restype = C.c_int
        L.ref_store_put.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, U64P]
        L.ref_store_get.restype = C.c_int
        L.ref_store_get.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]
        L.ref_store_total_bytes.restype = C.c_uint64
        L.ref_store_total_bytes.argtypes = [C.c_void_p]
        L.ref_store_count.restype = C.c_uint64
        L.ref_store_count.argtypes = [C.c_void_p]
        L.ref_store_persist.restype = C.c_int
        L.ref_store_persist.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_validate_window.restype = C.c_int
        L.ref_validate_window.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_char_p, C.c_uint64]
        L.ref_blob_rel_path.restype = C.c_int
        L.ref_blob_rel_path.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64]
        L.ref_alloc_new.restype = C.c_void_p
        L.ref_alloc_new.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_alloc_free_obj.argtypes = [C.c_void_p]
        L.ref_alloc_alloc.restype = C.c_int
        L.ref_alloc_alloc.argtypes = [C.c_void_p, C.c_uint64, C.c_int, U64P]
        L.ref_alloc_free.restype = C.c_int
        L.ref_alloc_free.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_alloc_stable_digest.restype = C.c_uint64
        L.ref_alloc_stable_digest.argtypes = [C.c_void_p]
        L.ref_alloc_cursors.argtypes = [C.c_void_p, U64P, U64P, U64P]
        L.ref_carve.restype = C.c_int
        L.ref_carve.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_void_p]
        L.ref_snapshot_chunks.restype = C.c_uint64
        L.ref_snapshot_chunks.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_void_p]
        L.ref_restore_chunks.restype = C.c_int
        L.ref_restore_chunks.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_void_p]
        L.ref_grad_sum_u64.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p, C.c_int]
        L.ref_splice_new.restype = C.c_void_p
        L.ref_splice_new.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_splice_free.argtypes = [C.c_void_p]
        L.ref_splice_alloc.restype = C.c_int
        L.ref_splice_alloc.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                       C.c_int, C.c_int]
        L.ref_splice_write.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]
        L.ref_splice_read.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]
        L.ref_splice_switch.restype = C.c_int
        L.ref_splice_switch.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        L.ref_manifest_run.restype = C.c_void_p
        L.ref_manifest_run.argtypes = [C.c_char_p]
        L.ref_manifest_free.argtypes = [C.c_void_p]
        L.ref_manifest_count.restype = C.c_int
        L.ref_manifest_count.argtypes = [C.c_void_p]
        L.ref_manifest_stats.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.ref_manifest_ndev.restype = C.c_int
        L.ref_manifest_ndev.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_manifest_dev.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                       C.c_void_p]
        L.ref_splice_switch2.restype = C.c_int
        L.ref_splice_switch2.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        L.ref_splice_mark_pending.restype = C.c_int
        L.ref_splice_mark_pending.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_splice_install.restype = C.c_int
        L.ref_splice_install.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_uint64]
        _ref = L
    return _ref


# ----------------------------------------------------------------- helpers

def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def mix64(x: int) -> int:
    return lib().or_mix64(x)


def fill_mix64(nwords: int, seed: int = 0, base: int = 0) -> np.ndarray:
    out = np.empty(nwords, dtype=np.uint64)
    lib().or_fill_mix64(_p(out), nwords, seed, base)
    return out


def digest_of_words(words: np.ndarray) -> int:
    w = np.ascontiguousarray(words, dtype=np.uint64)
    return lib().or_digest_of_words(_p(w), w.size)


def digest_of_bytes(b: bytes) -> int:
    return lib().or_fnv1a(b, len(b), 14695981039346656037)


def blob_rel_path(digest: int) -> str:
    """BlobStore::blob_rel_path (ckpt.cpp:35-40): "blobs/" + first two hex digits of the
    zero-padded 16-digit lowercase hex digest + "/" + the 16 digits."""
    h = f"{digest:016x}"
    return f"blobs/{h[:2]}/{h}"


def persisted_tree(blobs):
    """BlobStore::persist (ckpt.cpp:42-52) of a set of blobs {digest: bytes}: the expected
    {relative path: content} of the directory (content = the blob's words, little endian)."""
    return {blob_rel_path(d): bytes(b) for d, b in blobs.items()}


def host_pages(host_bufs, prev_pages=None, known=()):
    """build_manifest host section (ckpt.cpp:59-68 paged_host_words, 116-130): concatenate
    the rank's host buffers, zero-pad to 512-word pages, digest_of_words per page; fresh =
    first occurrence and not in the store (`known`), inc = not in the previous page set
    (every page when there is no previous manifest). Pure numpy + the oracle digest."""
    allw = np.concatenate([np.asarray(b, np.uint64) for b in host_bufs] or
                          [np.zeros(0, np.uint64)])
    pad = (-allw.size) % 512
    allw = np.concatenate([allw, np.zeros(pad, np.uint64)])
    dig = np.array([digest_of_words(allw[o:o + 512]) for o in range(0, allw.size, 512)],
                   np.uint64)
    seen, known, prev = set(), set(int(k) for k in known), (
        None if prev_pages is None else set(int(p) for p in prev_pages))
    flags = np.zeros(dig.size, np.uint8)
    for i, d in enumerate(dig.tolist()):
        if d not in known and d not in seen:
            flags[i] |= 1
        seen.add(d)
        if prev is None or d not in prev:
            flags[i] |= 2
    return dig, flags


def bufs_array(bufs):
    """bufs: iterable of (rank, slot, addr, bytes, cat) tuples or dicts."""
    arr = (OrBuf * max(1, len(bufs)))()
    for i, b in enumerate(bufs):
        if isinstance(b, dict):
            b = (b.get("rank", 0), b.get("slot", i), b["addr"], b["bytes"], b.get("cat", 0))
        arr[i] = OrBuf(b[0], b[1], b[2], b[3], b[4] if len(b) > 4 else 0, 0)
    return arr


def num_chunks(bufs, chunk_bytes: int) -> int:
    return lib().or_num_chunks(bufs_array(bufs), len(bufs), chunk_bytes)


def _arena_ptrs(arenas):
    arenas = [np.ascontiguousarray(a).view(np.uint8) for a in arenas]
    ptrs = (C.c_void_p * len(arenas))(*[a.ctypes.data for a in arenas])
    return arenas, ptrs


def hash_chunks(arenas, bufs, page_bytes=4096, chunk_bytes=65536, nthreads=8):
    """Returns (chunk_digests u64[n], chunk_lens u32[n], buf_digests u64[nbufs])."""
    keep, ptrs = _arena_ptrs(arenas)
    n = num_chunks(bufs, chunk_bytes)
    d = np.zeros(max(n, 1), dtype=np.uint64)
    lens = np.zeros(max(n, 1), dtype=np.uint32)
    bd = np.zeros(max(len(bufs), 1), dtype=np.uint64)
    rc = lib().or_hash(ptrs, bufs_array(bufs), len(bufs), page_bytes, chunk_bytes, _p(d), _p(lens),
                       _p(bd), nthreads)
    assert rc == 0, "or_hash: bad page/chunk geometry"
    del keep
    return d[:n], lens[:n], bd[: len(bufs)]


def select(digests, lens, known=None):
    """Returns (sel u8[n], owner u64[n], offsets u64[n], total_bytes)."""
    d = np.ascontiguousarray(digests, dtype=np.uint64)
    ln = np.ascontiguousarray(lens, dtype=np.uint32)
    kn = np.ascontiguousarray(known if known is not None else np.zeros(0), dtype=np.uint64)
    n = d.size
    sel = np.zeros(max(n, 1), dtype=np.uint8)
    owner = np.zeros(max(n, 1), dtype=np.uint64)
    off = np.zeros(max(n, 1), dtype=np.uint64)
    total = lib().or_select(_p(d), _p(ln), n, _p(kn), kn.size, _p(sel), _p(owner), _p(off))
    return sel[:n], owner[:n], off[:n], int(total)


def stripe(digests, lens, n_per_rank, sel):
    d = np.ascontiguousarray(digests, dtype=np.uint64)
    ln = np.ascontiguousarray(lens, dtype=np.uint32)
    npr = np.ascontiguousarray(n_per_rank, dtype=np.uint64)
    s = np.ascontiguousarray(sel, dtype=np.uint8)
    n = d.size
    writer = np.zeros(max(n, 1), dtype=np.int32)
    off = np.zeros(max(n, 1), dtype=np.uint64)
    sb = np.zeros(len(npr), dtype=np.uint64)
    lib().or_stripe(_p(d), _p(ln), _p(npr), len(npr), _p(s), _p(writer), _p(off), _p(sb))
    return writer[:n], off[:n], sb


def compact(arenas, bufs, chunk_bytes, sel, offsets, total):
    keep, ptrs = _arena_ptrs(arenas)
    staging = np.zeros(max(int(total), 1), dtype=np.uint8)
    s = np.ascontiguousarray(sel, dtype=np.uint8)
    o = np.ascontiguousarray(offsets, dtype=np.uint64)
    lib().or_compact(ptrs, bufs_array(bufs), len(bufs), chunk_bytes, _p(s), _p(o), _p(staging))
    del keep
    return staging[: int(total)]


def restore(arenas, bufs, chunk_bytes, image, src_off):
    """Scatter image chunks into the (mutable numpy) arenas in place."""
    arenas = [a.view(np.uint8) for a in arenas]
    ptrs = (C.c_void_p * len(arenas))(*[a.ctypes.data for a in arenas])
    img = np.ascontiguousarray(image, dtype=np.uint8)
    so = np.ascontiguousarray(src_off, dtype=np.uint64)
    lib().or_restore(ptrs, bufs_array(bufs), len(bufs), chunk_bytes, _p(img), _p(so))


def grad_sum_u64(grads):
    gs = [np.ascontiguousarray(g, dtype=np.uint64) for g in grads]
    ptrs = (C.c_void_p * len(gs))(*[g.ctypes.data for g in gs])
    out = np.empty_like(gs[0])
    lib().or_grad_sum_u64(ptrs, len(gs), gs[0].size, _p(out))
    return out


def grad_sum_bf16(grads):
    """bf16 gradients as uint16 arrays: ascending-order fp32 chain, one bf16 rounding."""
    gs = [np.ascontiguousarray(g, dtype=np.uint16) for g in grads]
    ptrs = (C.c_void_p * len(gs))(*[g.ctypes.data for g in gs])
    out = np.empty_like(gs[0])
    lib().or_grad_sum_bf16(ptrs, len(gs), gs[0].size, _p(out))
    return out


def grad_sum_f32(grads):
    gs = [np.ascontiguousarray(g, dtype=np.float32) for g in grads]
    ptrs = (C.c_void_p * len(gs))(*[g.ctypes.data for g in gs])
    out = np.empty_like(gs[0])
    lib().or_grad_sum_f32(ptrs, len(gs), gs[0].size, _p(out))
    return out


def ref_manifests(scenario: dict):
    """Every checkpoint manifest of the first job of `scenario`, built by the reference's
    own scheduler + build_manifest (oracle/ref_shim.cpp ref_manifest_run): stats and, per
    rank, the DevRecs {slot, addr, words, cat, digest} with their content (u64 words)."""
    import json
    R = ref()
    h = R.ref_manifest_run(json.dumps(scenario).encode())
    if not h:
        raise RuntimeError("reference scenario run failed")
    try:
        out = []
        for k in range(R.ref_manifest_count(h)):
            st = np.zeros(8, np.uint64)
            R.ref_manifest_stats(h, k, _p(st))
            names = ["s_g", "s_cr", "s_cr_inc", "upload_bytes", "dump_d2h_max",
                     "total_blob_bytes", "device_upload", "world"]
            m = {n: int(v) for n, v in zip(names, st)}
            m["dev"] = []
            for r in range(m["world"]):
                recs = []
                for i in range(R.ref_manifest_ndev(h, k, r)):
                    rec = np.zeros(5, np.uint64)
                    R.ref_manifest_dev(h, k, r, i, _p(rec), None)
                    words = np.zeros(int(rec[2]), np.uint64)
                    R.ref_manifest_dev(h, k, r, i, _p(rec), _p(words))
                    recs.append({"slot": int(np.int64(rec[0])), "addr": int(rec[1]),
                                 "words": int(rec[2]), "cat": int(np.int64(rec[3])),
                                 "digest": int(rec[4]), "content": words})
                m["dev"].append(recs)
            out.append(m)
        return out
    finally:
        R.ref_manifest_free(h)
