"""paper_2202_07848_b200 — B200-native snapshot / dedup / restore / splice hot path.

Thin ctypes binding of the C ABI in include/snap.h (libsnap.so, built in-tree
by `make -C paper_2202_07848_b200`). There is no CPU fallback: importing works
anywhere, but every compute call goes through the sm_100a kernels and raises
SnapError when the library or a B200 is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SNAP_LIB_PATH: A/B tooling only (tools/ab_step.py), the default is the in-tree build
LIB_PATH = os.environ.get("SNAP_LIB_PATH") or os.path.join(HERE, "libsnap.so")

SNAP_OK, SNAP_EINVAL, SNAP_ENOMEM, SNAP_EFAULT, SNAP_ECUDA, SNAP_EINTERNAL = 0, -1, -2, -3, -4, -5
U64, F32, BF16 = 0, 1, 2

# vdev::BufCat (vdev.hpp:17)
PARAM, OPTSTATE, GRAD, ACTIVATION, SCRATCH = range(5)


class SnapError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{msg} (code {code})")
        self.code = code


class SnapFault(SnapError):
    """SNAP_EFAULT: the reference's SimFault (common.hpp:31-35)."""


class SnapBuf(C.Structure):
    """snap_buf = RankBuf/DevRec (splice.hpp:26-34, ckpt.hpp:64-71)."""

    _fields_ = [
        ("rank", C.c_uint32),
        ("slot", C.c_int32),
        ("addr", C.c_uint64),
        ("bytes", C.c_uint64),
        ("cat", C.c_int32),
        ("flags", C.c_uint32),
    ]


class SwitchStats(C.Structure):
    """snap_switch_stats: the switch_report trace fields (job.cpp:181-195)."""

    _fields_ = [("hashed_bytes", C.c_uint64), ("swap_out_bytes", C.c_uint64),
                ("swap_in_bytes", C.c_uint64), ("resident_bytes", C.c_uint64),
                ("cache_bytes", C.c_uint64), ("install_bytes", C.c_uint64),
                ("cache_free_bytes", C.c_uint64), ("reclaimed_bytes", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


BUF_REPLICATED, BUF_PRIVATE, BUF_PENDING = 1, 2, 4


class SnapGeom(C.Structure):
    _fields_ = [("page_bytes", C.c_uint32), ("chunk_bytes", C.c_uint32)]


_lib = None

class PersistStats(C.Structure):
    """snap_persist_stats: blob files of one persist/load call and the rank layout's sizes
    (Manifest sizes: upload_bytes, total_blob_bytes; ckpt.hpp:102-107)."""

    _fields_ = [("blobs", C.c_uint64), ("written", C.c_uint64), ("present", C.c_uint64),
                ("bytes", C.c_uint64), ("layout_chunks", C.c_uint64),
                ("layout_blobs", C.c_uint64), ("layout_bytes", C.c_uint64),
                ("layout_bufs", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class PagesStats(C.Structure):
    """snap_pages_stats: the host-page sizes of build_manifest (ckpt.cpp:122-130)."""

    _fields_ = [("pages", C.c_uint64), ("s_cr", C.c_uint64), ("s_cr_inc", C.c_uint64),
                ("upload_bytes", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


PAGE_FRESH, PAGE_INC = 1, 2


class SnapMutation(C.Structure):
    """snap_mutation: ValidationRecord::mutations entry (splice.hpp:50-53)."""

    _fields_ = [("addr", C.c_uint64), ("bytes", C.c_uint64), ("digest", C.c_uint64)]


class WindowRecord(C.Structure):
    """snap_window_record: one rank's ValidationRecord (splice.hpp:50-54)."""

    _fields_ = [("rank", C.c_int32), ("mutations", C.POINTER(SnapMutation)),
                ("n_mutations", C.c_uint64), ("d2h", C.POINTER(C.c_uint64)),
                ("n_d2h", C.c_uint64)]


_SIGS = {
    "snap_open": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]),
    "snap_close": (C.c_int, [C.c_void_p]),
    "snap_last_error": (C.c_char_p, [C.c_void_p]),
    "snap_strerror": (C.c_char_p, [C.c_int]),
    "snap_arena": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]),
    "snap_launch_count": (C.c_uint64, [C.c_void_p]),
    "snap_sync": (C.c_int, [C.c_void_p]),
    "snap_layout_carve": (C.c_int, [C.c_uint64, C.c_uint64, C.c_double, C.c_void_p]),
    "snap_write": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "snap_read": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "snap_fill_mix64": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]),
    "snap_xor_words": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64]),
    "snap_set_buffers": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                   C.POINTER(C.c_uint64)]),
    "snap_hash": (C.c_int, [C.c_void_p]),
    "snap_get_digests": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "snap_digest_ranges": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "snap_known_clear": (C.c_int, [C.c_void_p]),
    "snap_digest_whole": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "snap_known_add": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "snap_known_commit": (C.c_int, [C.c_void_p]),
    "snap_select": (C.c_int, [C.c_void_p]),
    "snap_get_selection": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "snap_compact": (C.c_int, [C.c_void_p]),
    "snap_snapshot": (C.c_int, [C.c_void_p]),
    "snap_staging": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]),
    "snap_read_staging": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
    "snap_restore": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int]),
    "snap_restore_self": (C.c_int, [C.c_void_p, C.c_int]),
    "snap_grad_sum": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint32, C.c_uint64,
                                C.c_uint64, C.c_int]),
    "snap_comm_unique_id": (C.c_int, [C.c_void_p]),
    "snap_comm_init": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "snap_comm_destroy": (C.c_int, [C.c_void_p]),
    "snap_allreduce": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64]),
    "snap_allreduce_ordered": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_uint32,
                                         C.c_uint64, C.c_uint64]),
    "snap_comm_init_local": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_char_p]),
    "snap_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(C.c_void_p)]),
    "snap_host_free": (C.c_int, [C.c_void_p]),
    "snap_snapshot_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                     C.c_uint64, C.POINTER(C.c_uint64), C.c_void_p]),
    "snap_host_pages": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                  C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                  C.POINTER(PagesStats)]),
    "snap_window_open": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]),
    "snap_window_close": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64,
                                    C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]),
    "snap_validate_window": (C.c_int, [C.c_void_p, C.c_uint64, C.c_char_p, C.c_uint64]),
    "snap_blob_rel_path": (C.c_int, [C.c_uint64, C.c_char_p, C.c_uint64]),
    "snap_persist": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_uint64, C.c_int,
                               C.POINTER(PersistStats)]),
    "snap_load": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_int,
                            C.POINTER(PersistStats)]),
    "snap_persist_rank": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_void_p, C.c_uint64,
                                    C.c_int, C.POINTER(PersistStats)]),
    "snap_splice_load": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(PersistStats)]),
    "snap_global_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "snap_get_global_digests": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "snap_get_shard": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint64)]),
    "snap_prof_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "snap_set_k1_variant": (C.c_int, [C.c_int]),
    "snap_last_k1_kernel": (C.c_char_p, []),
    "snap_prof_read": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_float),
                                 C.POINTER(C.c_uint64)]),
    "snap_alloc_create": (C.c_int, [C.c_uint64, C.c_uint64, C.POINTER(C.c_void_p)]),
    "snap_alloc_destroy": (C.c_int, [C.c_void_p]),
    "snap_alloc_alloc": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_uint64)]),
    "snap_alloc_free": (C.c_int, [C.c_void_p, C.c_uint64]),
    "snap_alloc_stable_digest": (C.c_uint64, [C.c_void_p]),
    "snap_alloc_cursors": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_uint64)]),
    "snap_alloc_snapshot": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64,
                                      C.POINTER(C.c_uint64)]),
    "snap_alloc_restore": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "snap_splice_init": (C.c_int, [C.c_void_p, C.c_uint64]),
    "snap_splice_init_slots": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32]),
    "snap_splice_install": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64,
                                      C.c_uint64]),
    "snap_splice_pending": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64)]),
    "snap_splice_set_rank": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_void_p]),
    "snap_splice_switch": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "snap_splice_recorded": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_uint64)]),
    "snap_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p]),
    "snap_ipc_import": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "snap_restore_shards": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "snap_timer_start": (C.c_int, [C.c_void_p]),
    "snap_timer_stop": (C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
}


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


def lib():
    """Loads libsnap.so; raises if it was never built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SnapError(SNAP_ECUDA, f"{LIB_PATH} missing: run `make -C {HERE}` "
                                        "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def validate_window(records):
    """splice::validate_window (splice.cpp:21-61). records: {rank: (mutations, d2h)} with
    mutations = [(addr, bytes, digest)] in address order and d2h = [(bytes, digest)].
    Returns (passed, reason)."""
    keep, arr = [], (WindowRecord * max(1, len(records)))()
    for i, (rank, (muts, d2h)) in enumerate(records.items()):
        m = (SnapMutation * max(1, len(muts)))(*[SnapMutation(*x) for x in muts])
        d = (C.c_uint64 * max(2, 2 * len(d2h)))(*[v for p in d2h for v in p])
        keep += [m, d]
        arr[i] = WindowRecord(rank, C.cast(m, C.POINTER(SnapMutation)), len(muts),
                              C.cast(d, C.POINTER(C.c_uint64)), len(d2h))
    reason = C.create_string_buffer(512)
    rc = lib().snap_validate_window(arr, len(records), reason, 512)
    if rc < 0:
        raise SnapError(rc, "snap_validate_window")
    return rc == 1, reason.value.decode()


def blob_rel_path(digest: int) -> str:
    """BlobStore::blob_rel_path (ckpt.cpp:35-40) as the product library computes it."""
    b = C.create_string_buffer(40)
    rc = lib().snap_blob_rel_path(C.c_uint64(digest), b, 40)
    if rc:
        raise SnapError(rc, "snap_blob_rel_path")
    return b.value.decode()


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def bufs_array(bufs):
    arr = (SnapBuf * max(1, len(bufs)))()
    for i, b in enumerate(bufs):
        if isinstance(b, dict):
            b = (b.get("rank", 0), b.get("slot", i), b["addr"], b["bytes"], b.get("cat", 0),
                 b.get("flags", 0))
        arr[i] = SnapBuf(b[0], b[1], b[2], b[3], b[4] if len(b) > 4 else 0,
                         b[5] if len(b) > 5 else 0)
    return arr


def layout_carve(mem_bytes, max_buffer_bytes, slack_fraction):
    """splice::DeviceLayout::carve (splice.cpp:7-19) -> (rank_region_end, scratch_base, scratch_bytes)."""
    out = (C.c_uint64 * 3)()
    rc = lib().snap_layout_carve(mem_bytes, max_buffer_bytes, slack_fraction, out)
    if rc != SNAP_OK:
        raise SnapError(rc, "device too small for layout")
    return tuple(out)


PROF_HASH, PROF_SELECT, PROF_COMPACT, PROF_RESTORE, PROF_GRAD, PROF_EXCHANGE, PROF_SWITCH = range(7)


class BidiAllocator:
    """mem::BidiAllocator (alloc.hpp:17-62): same method names and error behaviour —
    alloc() returns None on OOM (std::nullopt) and raises SnapFault on a zero size,
    free() raises SnapFault on an unknown address."""

    STABLE, TRANSIENT = 1, 0

    def __init__(self, low: int, high: int):
        self._L = lib()
        h = C.c_void_p()
        rc = self._L.snap_alloc_create(low, high, C.byref(h))
        if rc != SNAP_OK:
            raise SnapError(rc, "allocator region must be aligned and non-empty")
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self._L.snap_alloc_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def alloc(self, nbytes: int, stable: bool):
        a = C.c_uint64()
        rc = self._L.snap_alloc_alloc(self.h, nbytes, 1 if stable else 0, C.byref(a))
        if rc == SNAP_ENOMEM:
            return None
        if rc == SNAP_EFAULT:
            raise SnapFault(rc, "alloc: zero size")
        if rc != SNAP_OK:
            raise SnapError(rc, "alloc")
        return a.value

    def free(self, addr: int):
        rc = self._L.snap_alloc_free(self.h, addr)
        if rc == SNAP_EFAULT:
            raise SnapFault(rc, "free: unknown allocation")
        if rc != SNAP_OK:
            raise SnapError(rc, "free")

    def stable_state_digest(self) -> int:
        return int(self._L.snap_alloc_stable_digest(self.h))

    def cursors(self):
        t, s, l = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._L.snap_alloc_cursors(self.h, C.byref(t), C.byref(s), C.byref(l))
        return t.value, s.value, l.value

    def snapshot(self) -> np.ndarray:
        n = C.c_uint64()
        self._L.snap_alloc_snapshot(self.h, None, 0, C.byref(n))
        w = np.zeros(max(n.value, 1), np.uint64)
        rc = self._L.snap_alloc_snapshot(self.h, _p(w), w.size, C.byref(n))
        if rc != SNAP_OK:
            raise SnapError(rc, "snapshot")
        return w[: n.value]

    def restore(self, words: np.ndarray):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        rc = self._L.snap_alloc_restore(self.h, _p(w), w.size)
        if rc != SNAP_OK:
            raise SnapError(rc, "restore: malformed snapshot")


class PinnedHost:
    """Page-locked host buffer (snap_host_alloc) viewed as a numpy uint8 array."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        rc = lib().snap_host_alloc(nbytes, C.byref(p))
        if rc != SNAP_OK:
            raise SnapError(rc, f"snap_host_alloc({nbytes})")
        self.ptr = p.value
        self.nbytes = nbytes
        self.array = np.ctypeslib.as_array((C.c_uint8 * max(nbytes, 1)).from_address(self.ptr))[:nbytes]

    def free(self):
        if self.ptr:
            lib().snap_host_free(C.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Ctx:
    """One snap_ctx: the per-(job, GPU) device proxy (proxy.hpp:32-122)."""

    def __init__(self, device: int = 0, arena_bytes: int = 1 << 28):
        self._L = lib()
        h = C.c_void_p()
        rc = self._L.snap_open(device, arena_bytes, C.byref(h))
        if rc != SNAP_OK:
            raise SnapError(rc, f"snap_open(device={device}, arena={arena_bytes}): "
                                f"{self._L.snap_strerror(rc).decode()}")
        self.h = h
        self.arena_bytes = arena_bytes
        self.nchunks = 0
        self.nbufs = 0

    # -- plumbing
    def close(self):
        if self.h:
            self._L.snap_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _ck(self, rc, what):
        if rc != SNAP_OK:
            msg = f"{what}: {self._L.snap_last_error(self.h).decode()}"
            raise (SnapFault if rc == SNAP_EFAULT else SnapError)(rc, msg)

    @property
    def launches(self) -> int:
        return int(self._L.snap_launch_count(self.h))

    def arena_ptr(self) -> int:
        p = C.c_void_p()
        self._ck(self._L.snap_arena(self.h, C.byref(p), None), "snap_arena")
        return p.value

    def sync(self):
        self._ck(self._L.snap_sync(self.h), "snap_sync")

    def write(self, addr: int, data: np.ndarray):
        d = np.ascontiguousarray(data)
        self._ck(self._L.snap_write(self.h, addr, _p(d), d.nbytes), "snap_write")

    def read(self, addr: int, nbytes: int) -> np.ndarray:
        out = np.empty(nbytes, dtype=np.uint8)
        self._ck(self._L.snap_read(self.h, addr, _p(out), nbytes), "snap_read")
        return out

    def fill_mix64(self, addr: int, nbytes: int, seed: int = 0, base: int = 0):
        self._ck(self._L.snap_fill_mix64(self.h, addr, nbytes, seed, base), "snap_fill_mix64")

    def xor_words(self, addrs, value: int):
        a = np.ascontiguousarray(addrs, dtype=np.uint64)
        self._ck(self._L.snap_xor_words(self.h, _p(a), a.size, value), "snap_xor_words")

    # -- K1
    def set_buffers(self, bufs, page_bytes=4096, chunk_bytes=65536) -> int:
        arr = bufs_array(bufs)
        g = SnapGeom(page_bytes, chunk_bytes)
        n = C.c_uint64()
        self._ck(self._L.snap_set_buffers(self.h, arr, len(bufs), C.byref(g), C.byref(n)),
                 "snap_set_buffers")
        self.nchunks = n.value
        self.nbufs = len(bufs)
        return self.nchunks

    def hash(self):
        self._ck(self._L.snap_hash(self.h), "snap_hash")

    def digests(self, buf_digests=False):
        n = self.nchunks
        d = np.zeros(max(n, 1), dtype=np.uint64)
        lens = np.zeros(max(n, 1), dtype=np.uint32)
        bd = np.zeros(max(self.nbufs, 1), dtype=np.uint64)
        self._ck(self._L.snap_get_digests(self.h, _p(d), _p(lens), _p(bd) if buf_digests else None),
                 "snap_get_digests")
        if buf_digests:
            return d[:n], lens[:n], bd[: self.nbufs]
        return d[:n], lens[:n]

    # -- K2
    def digest_whole(self, bufs):
        """Gpu::digest value-equal to the reference (one FNV-1a chain per range)."""
        arr = bufs_array([b[:5] for b in bufs])
        out = np.zeros(max(len(bufs), 1), np.uint64)
        self._ck(self._L.snap_digest_whole(self.h, arr, len(bufs), _p(out)), "snap_digest_whole")
        return out[:len(bufs)]

    def known_clear(self):
        self._ck(self._L.snap_known_clear(self.h), "snap_known_clear")

    def known_add(self, digests):
        d = np.ascontiguousarray(digests, dtype=np.uint64)
        self._ck(self._L.snap_known_add(self.h, _p(d), d.size), "snap_known_add")

    def known_commit(self):
        self._ck(self._L.snap_known_commit(self.h), "snap_known_commit")

    def select(self):
        self._ck(self._L.snap_select(self.h), "snap_select")

    def selection(self):
        n = self.nchunks
        sel = np.zeros(max(n, 1), dtype=np.uint8)
        owner = np.zeros(max(n, 1), dtype=np.uint64)
        off = np.zeros(max(n, 1), dtype=np.uint64)
        sb, sc = C.c_uint64(), C.c_uint64()
        self._ck(self._L.snap_get_selection(self.h, _p(sel), _p(owner), _p(off), C.byref(sb),
                                            C.byref(sc)), "snap_get_selection")
        return sel[:n], owner[:n], off[:n], sb.value, sc.value

    # -- K3
    def compact(self):
        self._ck(self._L.snap_compact(self.h), "snap_compact")

    def snapshot(self):
        self._ck(self._L.snap_snapshot(self.h), "snap_snapshot")

    def staging_ptr(self):
        p, n = C.c_void_p(), C.c_uint64()
        self._ck(self._L.snap_staging(self.h, C.byref(p), C.byref(n)), "snap_staging")
        return p.value, n.value

    def read_staging(self, off: int, nbytes: int) -> np.ndarray:
        out = np.empty(nbytes, dtype=np.uint8)
        self._ck(self._L.snap_read_staging(self.h, off, _p(out), nbytes), "snap_read_staging")
        return out

    def snapshot_host(self, host_ptr: int, addr: int, nbytes: int, staging_ptr: int,
                      staging_cap: int, digests_out=None) -> int:
        sb = C.c_uint64()
        d = None if digests_out is None else digests_out
        self._ck(self._L.snap_snapshot_host(self.h, C.c_void_p(host_ptr), addr, nbytes,
                                            C.c_void_p(staging_ptr), staging_cap, C.byref(sb),
                                            _p(d) if d is not None else None),
                 "snap_snapshot_host")
        return sb.value

    # -- ranges / squash-window validation (window.cpp)
    def digest_ranges(self, bufs, page_bytes=4096, chunk_bytes=65536):
        """Gpu::digest (vdev.cpp:118) of each (rank, slot, addr, bytes, cat) range, on the
        auxiliary grid (the installed snapshot grid is untouched)."""
        arr = bufs_array(bufs)
        g = SnapGeom(page_bytes, chunk_bytes)
        out = np.zeros(max(1, len(bufs)), np.uint64)
        self._ck(self._L.snap_digest_ranges(self.h, arr, len(bufs), C.byref(g), _p(out)),
                 "snap_digest_ranges")
        return out[:len(bufs)]

    def host_pages(self, host_bufs, prev_pages=None):
        """build_manifest host section (ckpt.cpp:116-130) for one rank: host_bufs = list of
        uint64 arrays (slot order). Returns (page_digests, flags, stats)."""
        arrs = [np.ascontiguousarray(b, dtype=np.uint64) for b in host_bufs]
        ptrs = (C.c_void_p * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])
        words = np.array([a.size for a in arrs] or [0], np.uint64)
        npages = (int(words[:len(arrs)].sum()) * 8 + 4095) // 4096
        dig = np.zeros(max(1, npages), np.uint64)
        flags = np.zeros(max(1, npages), np.uint8)
        prev = None if prev_pages is None else np.ascontiguousarray(prev_pages, dtype=np.uint64)
        st = PagesStats()
        self._ck(self._L.snap_host_pages(self.h, ptrs, _p(words), len(arrs),
                                         _p(prev) if prev is not None and prev.size else None,
                                         0 if prev is None else prev.size, _p(dig), npages,
                                         _p(flags), C.byref(st)), "snap_host_pages")
        return dig[:npages], flags[:npages], st.as_dict()

    def window_open(self, rank: int, bufs):
        """do_window_open validation branch (worker.cpp:355-362)."""
        arr = bufs_array(bufs)
        self._ck(self._L.snap_window_open(self.h, rank, arr, len(bufs)), "snap_window_open")

    def window_close(self, rank: int, bufs):
        """do_window_close validation branch (worker.cpp:411-421): the mutation set
        [(addr, bytes, digest)] in address order."""
        arr = bufs_array(bufs)
        out = (SnapMutation * max(1, len(bufs)))()
        n = C.c_uint64()
        self._ck(self._L.snap_window_close(self.h, rank, arr, len(bufs), out, len(bufs),
                                           C.byref(n)), "snap_window_close")
        return [(out[i].addr, out[i].bytes, out[i].digest) for i in range(n.value)]

    # -- on-disk format (BlobStore::persist, ckpt.cpp:42-52; restore_job, ckpt.cpp:504-533)
    def persist(self, directory, host_ptr: int = 0, host_bytes: int = 0, threads: int = 0,
                layout_rank=None):
        """Writes the last snapshot's staged chunks as blobs/<2hex>/<16hex> plus the layout
        + manifest (id = layout_rank, default the communicator rank) under `directory`."""
        st = PersistStats()
        hp = C.c_void_p(host_ptr) if host_ptr else None
        if layout_rank is None:
            rc = self._L.snap_persist(self.h, os.fsencode(directory), hp, host_bytes, threads,
                                      C.byref(st))
        else:
            rc = self._L.snap_persist_rank(self.h, os.fsencode(directory), layout_rank, hp,
                                           host_bytes, threads, C.byref(st))
        self._ck(rc, "snap_persist")
        return st.as_dict()

    def splice_load(self, directory, layout_rank: int, splice_rank: int, threads: int = 0):
        """restore_job cache seeding: a co-resident rank's persisted layout becomes splice
        rank `splice_rank` and its chunks enter the HBM chunk cache."""
        st = PersistStats()
        self._ck(self._L.snap_splice_load(self.h, os.fsencode(directory), layout_rank,
                                          splice_rank, threads, C.byref(st)), "snap_splice_load")
        return st.as_dict()

    def load(self, directory, rank: int = 0, verify: bool = True, threads: int = 0):
        """Installs rank `rank`'s persisted layout and restores its bytes from the blob files
        (digest-verified when verify); returns the stats dict."""
        st = PersistStats()
        rc = self._L.snap_load(self.h, os.fsencode(directory), rank, 1 if verify else 0, threads,
                               C.byref(st))
        if st.layout_chunks or rc == SNAP_OK:  # the layout was installed (even if verify failed)
            self.nchunks, self.nbufs = st.layout_chunks, st.layout_bufs
        self._ck(rc, "snap_load")
        return st.as_dict()

    def global_info(self):
        n, m = C.c_uint64(), C.c_uint64()
        self._ck(self._L.snap_global_info(self.h, C.byref(n), C.byref(m)), "snap_global_info")
        return n.value, m.value

    def global_digests(self):
        n, _ = self.global_info()
        d = np.zeros(max(n, 1), np.uint64)
        ln = np.zeros(max(n, 1), np.uint32)
        self._ck(self._L.snap_get_global_digests(self.h, _p(d), _p(ln)), "snap_get_global_digests")
        return d[:n], ln[:n]

    def global_selection(self):
        """Selection over the global (allgathered) vector: sel, owner, offsets, bytes, chunks."""
        n, _ = self.global_info()
        sel = np.zeros(max(n, 1), dtype=np.uint8)
        owner = np.zeros(max(n, 1), dtype=np.uint64)
        off = np.zeros(max(n, 1), dtype=np.uint64)
        sb, sc = C.c_uint64(), C.c_uint64()
        self._ck(self._L.snap_get_selection(self.h, _p(sel), _p(owner), _p(off), C.byref(sb),
                                            C.byref(sc)), "snap_get_selection")
        return sel[:n], owner[:n], off[:n], sb.value, sc.value

    def shard(self):
        n, _ = self.global_info()
        w = np.zeros(max(n, 1), np.int32)
        so = np.zeros(max(n, 1), np.uint64)
        mb, mc = C.c_uint64(), C.c_uint64()
        self._ck(self._L.snap_get_shard(self.h, _p(w), _p(so), C.byref(mb), C.byref(mc)),
                 "snap_get_shard")
        return w[:n], so[:n], mb.value, mc.value

    # -- resize / reshard
    def ipc_export(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        self._ck(self._L.snap_ipc_export(self.h, buf), "snap_ipc_export")
        return bytes(buf)

    def ipc_import(self, handles: bytes, nranks: int):
        buf = (C.c_uint8 * len(handles)).from_buffer_copy(handles)
        self._ck(self._L.snap_ipc_import(self.h, nranks, buf), "snap_ipc_import")

    def restore_shards(self, src_rank: int, verify=True):
        self._ck(self._L.snap_restore_shards(self.h, src_rank, 1 if verify else 0),
                 "snap_restore_shards")

    def prof_enable(self, on=True):
        self._ck(self._L.snap_prof_enable(self.h, 1 if on else 0), "snap_prof_enable")

    def prof_read(self, kind):
        ms, n = C.c_float(), C.c_uint64()
        self._ck(self._L.snap_prof_read(self.h, kind, C.byref(ms), C.byref(n)), "snap_prof_read")
        return ms.value, n.value

    # -- K4
    def restore(self, image_ptr: int, image_bytes: int, src_off, expect=None, verify=True):
        so = np.ascontiguousarray(src_off, dtype=np.uint64)
        ex = None if expect is None else np.ascontiguousarray(expect, dtype=np.uint64)
        self._ck(self._L.snap_restore(self.h, C.c_void_p(image_ptr), image_bytes, _p(so),
                                      _p(ex) if ex is not None else None, 1 if verify else 0),
                 "snap_restore")

    def restore_self(self, verify=True):
        self._ck(self._L.snap_restore_self(self.h, 1 if verify else 0), "snap_restore_self")

    # -- splice (GpuLedger::plan_switch/execute_switch)
    def splice_init(self, cache_bytes: int, slot_bytes: int = 65536):
        self._ck(self._L.snap_splice_init_slots(self.h, cache_bytes, slot_bytes),
                 "snap_splice_init_slots")

    def splice_install(self, ranks, dst_addrs, src_addr: int, nbytes: int):
        """on_coll_complete install (job.cpp:206-222): active rank now, others queued."""
        r = np.ascontiguousarray(ranks, dtype=np.int32)
        d = np.ascontiguousarray(dst_addrs, dtype=np.uint64)
        self._ck(self._L.snap_splice_install(self.h, _p(r), _p(d), r.size, src_addr, nbytes),
                 "snap_splice_install")

    def splice_pending(self, rank: int):
        c, b = C.c_uint64(), C.c_uint64()
        self._ck(self._L.snap_splice_pending(self.h, rank, C.byref(c), C.byref(b)),
                 "snap_splice_pending")
        return c.value, b.value

    def splice_set_rank(self, rank: int, bufs, page_bytes=4096, chunk_bytes=65536):
        arr = bufs_array([b[:5] for b in bufs])
        for i, b in enumerate(bufs):
            if len(b) > 5:
                arr[i].flags = b[5]
        g = SnapGeom(page_bytes, chunk_bytes)
        self._ck(self._L.snap_splice_set_rank(self.h, rank, arr, len(bufs), C.byref(g)),
                 "snap_splice_set_rank")

    def splice_recorded(self, rank: int) -> np.ndarray:
        """The rank's recorded chunk digests (its last switch-out), buffer/chunk order."""
        n = C.c_uint64()
        self._ck(self._L.snap_splice_recorded(self.h, rank, None, C.byref(n)),
                 "snap_splice_recorded")
        out = np.zeros(max(n.value, 1), np.uint64)
        self._ck(self._L.snap_splice_recorded(self.h, rank, _p(out), C.byref(n)),
                 "snap_splice_recorded")
        return out[:n.value]

    def splice_switch(self, frm: int, to: int) -> dict:
        st = SwitchStats()
        self._ck(self._L.snap_splice_switch(self.h, frm, to, C.byref(st)), "snap_splice_switch")
        return st.as_dict()

    # -- K5
    def grad_sum(self, dtype, src_addrs, dst_addr, elems, accumulate=False):
        a = np.ascontiguousarray(src_addrs, dtype=np.uint64)
        self._ck(self._L.snap_grad_sum(self.h, dtype, _p(a), a.size, dst_addr, elems,
                                       1 if accumulate else 0), "snap_grad_sum")

    # -- NCCL
    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        rc = lib().snap_comm_unique_id(buf)
        if rc != SNAP_OK:
            raise SnapError(rc, "ncclGetUniqueId failed")
        return bytes(buf)

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self._ck(self._L.snap_comm_init(self.h, nranks, rank, buf), "snap_comm_init")

    def comm_init_local(self, nranks: int, rank: int, key: str):
        """In-process communicator (one ctx per thread; blocks until all ranks joined)."""
        self._ck(self._L.snap_comm_init_local(self.h, nranks, rank, key.encode()),
                 "snap_comm_init_local")

    def allreduce_ordered(self, dtype, keys, src_addrs, dst_addr: int, elems: int):
        """Fixed-order allreduce: sum of every GPU's sources in ascending key order."""
        k = np.ascontiguousarray(keys, dtype=np.uint32)
        a = np.ascontiguousarray(src_addrs, dtype=np.uint64)
        self._ck(self._L.snap_allreduce_ordered(self.h, dtype, _p(k), _p(a), k.size, dst_addr,
                                                elems), "snap_allreduce_ordered")

    def comm_destroy(self):
        self._ck(self._L.snap_comm_destroy(self.h), "snap_comm_destroy")

    def allreduce(self, dtype, addr, elems):
        self._ck(self._L.snap_allreduce(self.h, dtype, addr, elems), "snap_allreduce")

    # -- timing
    def timer_start(self):
        self._ck(self._L.snap_timer_start(self.h), "snap_timer_start")

    def timer_stop(self) -> float:
        ms = C.c_float()
        self._ck(self._L.snap_timer_stop(self.h, C.byref(ms)), "snap_timer_stop")
        return ms.value


def set_k1_variant(variant: int = -1) -> None:
    """K1 kernel policy for this process (snap_set_k1_variant): -1 default, 11 tensor-core
    FNV, 10 TMA loads, 9 cp.async; applies to grids installed afterwards."""
    rc = lib().snap_set_k1_variant(int(variant))
    if rc < 0:
        raise SnapError(rc, "snap_set_k1_variant")


def last_k1_kernel() -> str:
    """Name of the K1 kernel the most recent hash launch used (snap_last_k1_kernel)."""
    return lib().snap_last_k1_kernel().decode()
