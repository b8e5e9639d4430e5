"""GPU tests of the host-page snapshot (build_manifest host section,
ckpt.cpp:59-68 and 116-130): page digests, fresh (store) and incremental (previous
manifest) classification against the CPU oracle."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def host_state(seed, n=6):
    rng = np.random.default_rng(seed)
    bufs = []
    for i in range(n):
        w = int(rng.integers(0, 3000))
        kind = int(rng.integers(0, 3))
        if kind == 0:
            bufs.append(np.zeros(w, np.uint64))          # zero pages dedup within the rank
        else:
            bufs.append(O.fill_mix64(w, seed * 10 + kind, 0))  # kind repeats -> duplicates
    return bufs


@pytest.mark.parametrize("seed", range(5))
def test_host_pages_vs_oracle(snap, ctx, seed):
    bufs = host_state(seed)
    dig, flags, st = ctx.host_pages(bufs)
    od, of = O.host_pages(bufs)
    assert np.array_equal(dig, od) and np.array_equal(flags, of)
    assert st["pages"] == od.size and st["s_cr"] == od.size * 4096
    assert st["upload_bytes"] == int((of & 1).sum()) * 4096
    assert st["s_cr_inc"] == od.size * 4096  # no previous manifest: every page is new
    # second checkpoint: the store holds the first one's pages, prev = its page list
    ctx.known_add(dig)
    bufs2 = [b.copy() for b in bufs]
    for b in bufs2[::2]:
        if b.size:
            b[b.size // 2] ^= np.uint64(0xFEED)
    dig2, flags2, st2 = ctx.host_pages(bufs2, prev_pages=dig)
    od2, of2 = O.host_pages(bufs2, prev_pages=dig, known=dig)
    assert np.array_equal(dig2, od2) and np.array_equal(flags2, of2)
    assert st2["upload_bytes"] == int((of2 & 1).sum()) * 4096
    assert st2["s_cr_inc"] == int(((of2 & 2) != 0).sum()) * 4096
    ctx.known_clear()


def test_host_pages_edges(snap, ctx):
    # no host state -> no pages; a single word -> one zero-padded page
    assert ctx.host_pages([])[2]["pages"] == 0
    assert ctx.host_pages([np.zeros(0, np.uint64)])[2]["pages"] == 0
    d, f, st = ctx.host_pages([np.array([7], np.uint64)])
    od, of = O.host_pages([np.array([7], np.uint64)])
    assert st["pages"] == 1 and np.array_equal(d, od) and np.array_equal(f, of)
    # a page whose digest equals the table's empty key still classifies correctly is
    # covered by the K2 table tests; here: many identical pages -> one fresh
    many = [np.zeros(512 * 1000, np.uint64)]
    d, f, st = ctx.host_pages(many)
    assert st["upload_bytes"] == 4096 and (f & 1).sum() == 1 and f[0] & 1
    # the installed grid is untouched by the host-page pass
    ctx.fill_mix64(0, 1 << 20, 1, 0)
    ctx.set_buffers([(0, 0, 0, 1 << 20, 0)])
    ctx.snapshot()
    before, _ = ctx.digests()
    ctx.host_pages([O.fill_mix64(5000, 2, 0)])
    after, _ = ctx.digests()
    assert np.array_equal(before, after)
    ctx.restore_self(verify=True)
