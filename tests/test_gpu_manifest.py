"""build_manifest's device section on the GPU against the reference's OWN manifests
(VERDICT r1 missing #6): the Appendix-B scenario (DP4 / DP8, 4 layers x 2048 words, seed 7,
checkpoints at 0.5 ms and 2.1 ms) is run by the reference's scheduler (oracle/_ref,
ref_manifest_run); its device buffers — every rank's DevRecs with their content — are then
snapshotted by libsnap:
  * one ctx holding every rank's buffers (canonical rank/slot order), and
  * one ctx per rank on the in-process communicator (identical addresses on every rank,
    cross-rank dedup over the exchanged digest vectors, striped shards).
One chunk per buffer (geometry 64 KiB / 64 KiB, buffers <= 64 KiB), so every chunk digest is
the reference's whole-buffer digest_of_words and must equal the DevRec digest; staged
bytes must equal S_G (first checkpoint) and the device part of upload_bytes (second,
incremental checkpoint against the first one's blobs); the staged image holds exactly the
first-occurrence buffers' bytes."""
import numpy as np
import pytest

import oracle as O
from _group import run_threads

pytestmark = pytest.mark.gpu

REGION = 4 << 20  # mem_mib of the scenario's GPUs


def scenario(dp):
    return {"seed": 7,
            "fleet": {"regions": [{"clusters": [{"nodes": [{"gpus": dp, "mem_mib": 4}]}]}]},
            "jobs": [{"name": "j", "spec": {"world": dp, "dp": dp, "layers": 4,
                                            "params_per_layer": 2048}}],
            "events": [{"at_sec": 0.0005, "kind": "checkpoint", "job": "j"},
                       {"at_sec": 0.0021, "kind": "checkpoint", "job": "j"}]}


@pytest.fixture(scope="module", params=[4, 8])
def manifests(request):
    if O.ref() is None:
        pytest.skip("reference library not built")
    ms = O.ref_manifests(scenario(request.param))
    assert len(ms) == 2 and ms[0]["s_g"] == 131072
    return ms


def test_manifest_one_ctx(snap, manifests):
    world = manifests[0]["world"]
    with snap.Ctx(0, world * REGION) as c:
        prev = None
        for k, m in enumerate(manifests):
            bufs, digs, first, seen = [], [], [], set()
            for r in range(world):
                for d in m["dev"][r]:
                    a = r * REGION + d["addr"]
                    c.write(a, d["content"])
                    bufs.append((r, d["slot"], a, d["words"] * 8, d["cat"]))
                    digs.append(d["digest"])
                    if d["digest"] not in seen and (prev is None or d["digest"] not in prev):
                        first.append(d["content"])
                    seen.add(d["digest"])
            c.set_buffers(bufs, 65536, 65536)
            c.snapshot()
            got, _ = c.digests()
            assert np.array_equal(got, np.array(digs, np.uint64)), "chunk digest != DevRec digest"
            _, _, _, staged, _ = c.selection()
            assert staged == (m["s_g"] if k == 0 else m["device_upload"]), (k, staged, m)
            img = c.read_staging(0, staged)
            assert np.array_equal(img, np.concatenate(first).view(np.uint8))
            c.known_commit()
            prev = set(digs)


def test_manifest_threads(snap, manifests):
    world = manifests[0]["world"]

    def run(g):
        ok = True
        with snap.Ctx(0, REGION) as c:
            g.comm_init(c)
            for k, m in enumerate(manifests):
                recs = m["dev"][g.rank]
                for d in recs:
                    c.write(d["addr"], d["content"])
                c.set_buffers([(g.rank, d["slot"], d["addr"], d["words"] * 8, d["cat"])
                               for d in recs], 65536, 65536)
                c.snapshot()
                got, _ = c.digests()
                ok &= np.array_equal(got, np.array([d["digest"] for d in recs], np.uint64))
                _, _, _, gbytes, _ = c.global_selection()
                _, _, mine, _ = c.shard()
                want = m["s_g"] if k == 0 else m["device_upload"]
                tot = sum(g.all_gather(mine))
                if gbytes != want or tot != want:
                    print(f"FAIL rank {g.rank} ckpt {k}: staged {gbytes} / shards {tot} vs {want}")
                    ok = False
                c.known_commit()
            c.comm_destroy()
        return ok

    assert all(run_threads(world, run))


def test_manifest_through_integration_glue(snap, manifests):
    """The maintainer-facing glue (integration/fleetsim_snap.hpp), compiled against the
    reference's headers into oracle/_ref/libfleetsim_glue.so: at every checkpoint of the
    reference scheduler, restore_job's materialization of the manifest onto a snap_ctx
    (one verified scatter pass) and build_manifest's device section through libsnap
    give the reference's S_G and device upload bytes."""
    import ctypes as C
    import json
    import os
    path = os.path.join(os.path.dirname(O.__file__), "_ref", "libfleetsim_glue.so")
    if not os.path.exists(path):
        pytest.skip("glue library not built")
    L = C.CDLL(path)
    L.glue_manifest_run.restype = C.c_int
    L.glue_manifest_run.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_int]
    out = np.zeros(4 * 4, np.uint64)
    n = L.glue_manifest_run(json.dumps(scenario(manifests[0]["world"])).encode(), 0,
                            out.ctypes.data, 4)
    assert n == 2
    rows = out.reshape(4, 4)[:n]
    assert rows[0][0] == 131072 and rows[0][2] == rows[0][0], rows      # S_G
    assert rows[1][2] == rows[1][1] == manifests[1]["device_upload"], rows  # upload
    assert (rows[:, 3] == 1).all(), "restore through the glue failed verification"
