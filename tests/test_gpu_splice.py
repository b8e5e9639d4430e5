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
        ctx.splice_init(2 * MIB)  # 32 slots: fewer than one rank's 55 distinct chunks
        ctx.fill_mix64(0, 8 * MIB, 17, 0)
        ctx.splice_set_rank(0, lay)
        ctx.splice_set_rank(1, lay)
        with pytest.raises(snap.SnapError) as e:
            ctx.splice_switch(0, 1)
        assert e.value.code == snap.SNAP_ENOMEM


@pytest.mark.parametrize("cache_replicas", [2.25])
def test_splice_long_run_bounded_cache_with_installs(snap, cache_replicas):
    """200 switches of 4 time-sliced DP ranks with per-mini-batch P/O updates and the spliced
    gradient path: every mini-batch the active rank applies the
    optimizer update to its P/O (identical across replicas, as after the DP allreduce),
    writes its own gradient, accumulates it (K5, u64 = the reference's arithmetic) and, as
    the local closer, installs the result into every rank's G slot: now for itself, queued
    for the inactive ranks (job.cpp:206-222) and applied at their next switch-in
    (job.cpp:164-171). The HBM chunk cache holds only 2.25 replicas, so it must reclaim the
    chunks no rank records any more; the reference's host cache grows without bound. Per
    switch: swap-out, swap-in (+d2d) and install bytes equal the reference GpuLedger's
    (driven by the reference shim's restatement of the job runtime's install queue), and
    the incoming rank's P/O and G are bit-identical on both sides."""
    R = O.ref()
    if R is None:
        pytest.skip("reference library not built here")
    nranks, mem = 4, 16 * MIB
    lay = rank_layout()
    stable = [b for b in lay if not b[5] & 4]
    gslot, gaddr, gbytes = 4, 6 * MIB, 512 * KIB
    acc = 8 * MIB
    slots_per_replica = sum((n + 65535) // 65536 for (_, _, _, n, _, _) in stable)
    ref = R.ref_splice_new(mem, 8 * MIB)
    ctx = snap.Ctx(0, mem)
    ctx.splice_init(int(cache_replicas * slots_per_replica) * 65536)
    for r in range(nranks):
        ctx.splice_set_rank(r, lay)
    po = {s: O.fill_mix64(n // 8, 7 + 1000 * s, 0) for (_, s, a, n, c, f) in stable}
    truth = [{s: w.copy() for s, w in po.items()} for _ in range(nranks)]
    gtruth = [None] * nranks
    out = np.zeros(6, np.uint64)

    def write_po(r):
        for (_, s, a, n, c, f) in stable:
            ctx.write(a, truth[r][s])
            R.ref_splice_write(ref, a, truth[r][s].ctypes.data, n // 8)

    def check_incoming(r, tag):
        for (_, s, a, n, c, f) in stable:
            got = ctx.read(a, n).view(np.uint64)
            exp = np.zeros(n // 8, np.uint64)
            R.ref_splice_read(ref, a, exp.ctypes.data, n // 8)
            assert np.array_equal(exp, truth[r][s]), f"reference P/O wrong {tag} slot {s}"
            assert np.array_equal(got, truth[r][s]), f"B200 P/O wrong {tag} slot {s}"
        if gtruth[r] is not None:
            got = ctx.read(gaddr, gbytes).view(np.uint64)
            exp = np.zeros(gbytes // 8, np.uint64)
            R.ref_splice_read(ref, gaddr, exp.ctypes.data, gbytes // 8)
            assert np.array_equal(exp, gtruth[r]), f"reference G install wrong {tag}"
            assert np.array_equal(got, gtruth[r]), f"B200 G install wrong {tag}"

    contrib = {}  # mini-batch -> gradients issued so far (K5 accumulation order)
    next_mb = [0] * nranks
    updates = {}
    rng = np.random.default_rng(3)

    def run_slice(a):
        """The active rank's program until it blocks on a DP allreduce: optimizer step of
        its next mini-batch (needs the previous result), backward, issue + K5 accumulate;
        the local closer installs the result everywhere and keeps running."""
        nonlocal gtruth
        while True:
            mb = next_mb[a]
            next_mb[a] += 1
            if mb > 0:
                if mb not in updates:
                    updates[mb] = [b for b in range(4) if rng.random() < 0.5]
                for b in updates[mb]:
                    # a mix64 value per (mini-batch, buffer): no run of the xors
                    # repeats, so a version never recurs (a recurring version that nobody
                    # recorded any more is saved again by the bounded cache, while the
                    # reference's unbounded host cache still holds it)
                    mutate(truth[a], b, O.lib().or_mix64(0x5EED0000 + mb * 16 + b))
            write_po(a)
            g = O.fill_mix64(gbytes // 8, 50_000 + 97 * mb + a, 0)
            ctx.write(gaddr, g)
            R.ref_splice_write(ref, gaddr, g.ctypes.data, gbytes // 8)
            assert R.ref_splice_mark_pending(ref, a, gslot) == 0
            first = mb not in contrib
            contrib.setdefault(mb, []).append(g)
            ctx.grad_sum(snap.U64, [gaddr], acc, gbytes // 8, accumulate=not first)
            if len(contrib[mb]) < nranks:
                return
            res = O.grad_sum_u64(contrib.pop(mb))
            for q in range(nranks):
                assert R.ref_splice_install(ref, q, gslot, res.ctypes.data, res.size) == 0
            ctx.splice_install(list(range(nranks)), [gaddr] * nranks, acc, gbytes)
            gtruth = [res.copy() for _ in range(nranks)]

    # first activations: allocate, run until the first DP wait, yield
    for r in range(nranks):
        for (_, s, a, n, c, f) in lay:
            assert R.ref_splice_alloc(ref, r, s, a, n, c, 1 if f & 4 else 0) == 0
        run_slice(r)
        nxt = (r + 1) % nranks
        assert R.ref_splice_switch2(ref, r, nxt, out.ctypes.data) == 0
        st = ctx.splice_switch(r, nxt)
        assert st["swap_out_bytes"] == int(out[0]), (r, st, out)
        assert st["install_bytes"] == int(out[5]), (r, st, out)
    check_incoming(0, "after warm-up")
    active, reclaimed, installs = 0, 0, 0
    for k in range(200):
        run_slice(active)
        nxt = (active + 1) % nranks
        assert R.ref_splice_switch2(ref, active, nxt, out.ctypes.data) == 0
        st = ctx.splice_switch(active, nxt)
        assert st["swap_out_bytes"] == int(out[0]), (k, st, out)
        assert st["swap_in_bytes"] == int(out[1]) + int(out[2]), (k, st, out)
        assert st["install_bytes"] == int(out[5]), (k, st, out)
        assert st["cache_bytes"] + st["cache_free_bytes"] <= \
            int(cache_replicas * slots_per_replica) * 65536
        reclaimed = st["reclaimed_bytes"]
        installs += int(out[5]) > 0
        check_incoming(nxt, f"switch {k}")
        active = nxt
    assert installs > 100, "deferred installs were not exercised"
    assert reclaimed > 0, "the bounded cache never reclaimed anything"
    # the reference's host cache only grew: far beyond what the B200 cache holds
    assert int(out[4]) > 2 * int(cache_replicas * slots_per_replica) * 65536
    R.ref_splice_free(ref)
    ctx.close()


def test_splice_install_immediate_without_splicing(snap):
    """A ctx without splicing (or rank < 0) installs immediately (single-rank GPU)."""
    with snap.Ctx(0, 4 * MIB) as ctx:
        src = O.fill_mix64(65536 // 8, 9, 0)
        ctx.write(0, src)
        ctx.splice_install([0, -1], [1 * MIB, 2 * MIB], 0, 65536)
        assert np.array_equal(ctx.read(1 * MIB, 65536), src.view(np.uint8))
        assert np.array_equal(ctx.read(2 * MIB, 65536), src.view(np.uint8))


def test_splice_recorded_digests_in_buffer_order(snap):
    """The splice grid hashes chunk-aligned buffers first (tensor-core task regularity);
    snap_splice_recorded still reports the digests in the caller's buffer/chunk order."""
    lay = rank_layout()
    with snap.Ctx(0, 16 * MIB) as ctx:
        ctx.splice_init(32 * MIB)
        ctx.fill_mix64(0, 8 * MIB, 23, 0)
        ctx.splice_set_rank(0, lay)
        ctx.splice_set_rank(1, lay)
        ctx.splice_switch(0, 1)
        got = ctx.splice_recorded(0)
        host = ctx.read(0, 8 * MIB)
        live = [b[:5] for b in lay if not b[5] & 4]
        exp, _, _ = O.hash_chunks([host], live)
        assert np.array_equal(got, exp)


def test_splice_slot_geometry(snap):
    """The chunk cache's slot size bounds the chunk size (64 KiB chunks do not fit 4 KiB
    slots); small slots with small chunks switch correctly (4 KiB chunks, 4 KiB slots)."""
    lay = rank_layout()
    with snap.Ctx(0, 16 * MIB) as ctx:
        ctx.splice_init(8 * MIB, slot_bytes=4096)
        with pytest.raises(snap.SnapError) as e:
            ctx.splice_set_rank(0, lay)  # default 64 KiB chunks
        assert e.value.code == snap.SNAP_EINVAL
        ctx.fill_mix64(0, 8 * MIB, 41, 0)
        ctx.splice_set_rank(0, lay, page_bytes=4096, chunk_bytes=4096)
        ctx.splice_set_rank(1, lay, page_bytes=4096, chunk_bytes=4096)
        before = ctx.read(0, 6 * MIB)
        ctx.splice_switch(0, 1)
        ctx.fill_mix64(0, 6 * MIB, 42, 0)  # rank 1's different P/O
        st = ctx.splice_switch(1, 0)
        after = ctx.read(0, 6 * MIB)
        for (_, s, a, n, c, f) in lay:
            if not f & 4:
                assert np.array_equal(after[a:a + n], before[a:a + n])
        assert st["swap_in_bytes"] > 0
