"""The opt-in whole-buffer digest (snap_digest_whole) is VALUE-equal to the reference's
Gpu::digest (vdev.cpp:118 = digest_of_words over the range): the Appendix-B C1 golden
(256 MiB whole-image FNV-1a = 0x2cfcad222b47bd17, computed by linking the reference) and
ragged ranges against the oracle / the reference library."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def test_whole_c1_golden(snap, golden):
    nbytes = 256 << 20
    with snap.Ctx(0, nbytes) as c:
        c.fill_mix64(0, nbytes, 0, 0)  # words[i] = mix64(i)
        d = c.digest_whole([(0, 0, 0, nbytes, 0)])
        assert int(d[0]) == golden["c1_whole"] == 0x2CFCAD222B47BD17


def test_whole_ragged_vs_reference(snap):
    rng = np.random.default_rng(4)
    sizes = [256, 512, 65536, 65536 + 256, 3 * 65536 - 768, 1 << 20, (5 << 20) + 4096 + 256]
    addr, bufs = 0, []
    for i, n in enumerate(sizes):
        bufs.append((0, i, addr, n, i % 3))
        addr += (n + 65535) // 65536 * 65536 + 256 * i
    arena = (addr + 65535) // 65536 * 65536
    with snap.Ctx(0, arena) as c:
        host = rng.integers(0, 2**63, size=arena // 8, dtype=np.uint64)
        c.write(0, host)
        got = c.digest_whole(bufs)
        R = O.ref()
        for (_r, _s, a, n, _c), d in zip(bufs, got):
            w = host[a // 8:(a + n) // 8]
            assert int(d) == O.digest_of_words(w)
            if R is not None:
                assert int(d) == R.ref_digest_of_words(w.ctypes.data, w.size)
