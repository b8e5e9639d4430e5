"""GPU parity of the replica-splicing context switch (snap_splice_*) against the reference's
own GpuLedger + vdev::Gpu (oracle/_ref, with the App. A-1 stale-digest fix applied by
refreshing the outgoing rank's digests before each plan): identical swap-out bytes,
identical swap-in (+ d2d move) bytes, and bit-identical device content of the incoming
rank after every switch, over time-sliced DP ranks with evolving P/O state."""
import ctypes as C

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

KIB = 1 << 10
MIB = 1 << 20


def rank_layout():
    # identical stable addresses on every replica (BidiAllocator property); the grad buffer
    # is pending (consumed by the local accumulation) and never swapped
    return [(0, 0, 0, 1 * MIB, 0, 0), (0, 1, 1 * MIB, 300 * KIB, 0, 0),
            (0, 2, 2 * MIB, 2 * MIB + 768, 1, 0), (0, 3, 5 * MIB, 64 * KIB, 1, 0),
            (0, 4, 6 * MIB, 512 * KIB, 2, 4)]


def mutate(words_by_buf, b, value):
    """xor `value` into the first word of every 64 KiB chunk of buffer b (whole-buffer
    change, so buffer- and chunk-granular ledgers take the same decisions)."""
    w = words_by_buf[b]
    w[::8192] ^= np.uint64(value)


@pytest.mark.parametrize("mode", ["identical", "divergent"])
def test_splice_matches_reference_ledger(snap, mode):
    R = O.ref()
    if R is None:
        pytest.skip("reference library not built here")
    nranks, mem = 4, 16 * MIB
    lay = rank_layout()
    ref = R.ref_splice_new(mem, 8 * MIB)
    ctx = snap.Ctx(0, mem)
    ctx.splice_init(64 * MIB)
    for r in range(nranks):
        ctx.splice_set_rank(r, lay)
    # per-rank truth: identical initial P/O, per-rank grads
    truth = []
    for r in range(nranks):
        t = {}
        for (_, s, a, n, c, f) in lay:
            # distinct bytes per buffer, so buffer- and chunk-granular dedup coincide
            t[s] = O.fill_mix64(n // 8, 7 + 1000 * s if c != 2 else 100 + r, 0)
        truth.append(t)

    def write_rank(r):
        for (_, s, a, n, c, f) in lay:
            ctx.write(a, truth[r][s])
            R.ref_splice_write(ref, a, truth[r][s].ctypes.data, n // 8)

    def check_resident(r, tag):
        for (_, s, a, n, c, f) in lay:
            if f & 4:
                continue
            got = ctx.read(a, n).view(np.uint64)
            exp = np.zeros(n // 8, np.uint64)
            R.ref_splice_read(ref, a, exp.ctypes.data, n // 8)
            assert np.array_equal(exp, truth[r][s]), f"reference content wrong {tag} slot {s}"
            assert np.array_equal(got, truth[r][s]), f"B200 content wrong {tag} slot {s}"

    out = np.zeros(5, np.uint64)
    # first activations: rank r allocates while active, then is switched out
    for r in range(nranks):
        for (_, s, a, n, c, f) in lay:
            assert R.ref_splice_alloc(ref, r, s, a, n, c, 1 if f & 4 else 0) == 0
        write_rank(r)
        nxt = r + 1 if r + 1 < nranks else 0
        rc = R.ref_splice_switch(ref, r, nxt if r + 1 < nranks else 0, out.ctypes.data)
        assert rc == 0
        st = ctx.splice_switch(r, nxt if r + 1 < nranks else 0)
        assert st["swap_out_bytes"] == int(out[0]), (r, st, out)
    check_resident(0, "after warm-up")
    # time-sliced mini-batches: the active rank updates its P/O, then yields
    rng = np.random.default_rng(1)
    active = 0
    for step in range(12):
        for b in range(4):
            if mode == "identical":
                # DP replicas apply the same update per mini-batch (after the allreduce)
                if rng.random() < 0.5:
                    mutate(truth[active], b, 0x1000 + step * 16 + b)
            else:
                if rng.random() < 0.5:
                    mutate(truth[active], b, 0x9000 + step * 64 + active * 8 + b)
        for (_, s, a, n, c, f) in lay:
            if not f & 4:
                ctx.write(a, truth[active][s])
                R.ref_splice_write(ref, a, truth[active][s].ctypes.data, n // 8)
        nxt = (active + 1) % nranks
        assert R.ref_splice_switch(ref, active, nxt, out.ctypes.data) == 0
        st = ctx.splice_switch(active, nxt)
        assert st["swap_out_bytes"] == int(out[0]), (step, st, out)
        assert st["swap_in_bytes"] == int(out[1]) + int(out[2]), (step, st, out)
        assert st["hashed_bytes"] == sum(n for (_, _, _, n, _, f) in lay if not f & 4)
        check_resident(nxt, f"step {step}")
        active = nxt
    R.ref_splice_free(ref)
    ctx.close()


def test_splice_identical_replicas_swap_nothing(snap):
    """with identical P/O across replicas a switch moves no bytes after the
    first cycle (only the digest pass)."""
    lay = rank_layout()
    with snap.Ctx(0, 16 * MIB) as ctx:
        ctx.splice_init(32 * MIB)
        for r in range(4):
            ctx.splice_set_rank(r, lay)
        ctx.fill_mix64(0, 6 * MIB, 3, 0)
        stats = [ctx.splice_switch(r, (r + 1) % 4) for r in range(4)]
        stats += [ctx.splice_switch(r, (r + 1) % 4) for r in range(4)]
        assert stats[0]["swap_out_bytes"] > 0
        assert all(s["swap_out_bytes"] == 0 for s in stats[1:])
        assert all(s["swap_in_bytes"] == 0 for s in stats[4:])


def test_splice_cache_full_is_enomem(snap):
    lay = rank_layout()
    with snap.Ctx(0, 16 * MIB) as ctx:
        ctx.splice_init(2 * MIB)  # smaller than one rank's live state (3.4 MiB)
        ctx.splice_set_rank(0, lay)
        ctx.splice_set_rank(1, lay)
        with pytest.raises(snap.SnapError) as e:
            ctx.splice_switch(0, 1)
        assert e.value.code == snap.SNAP_ENOMEM
