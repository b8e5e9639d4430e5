"""C1 (256 MiB, 64 x 4 MiB buffers) snapshot and verified-restore time per K1 variant
(dev tool). python tools/c1_variants.py [variants...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_07848_b200 as snap  # noqa: E402


def main():
    variants = [int(x) for x in sys.argv[1:]] or [-1, 7, 8, 9]
    nbytes, nb = 256 << 20, 4 << 20
    bufs = [(0, i, i * nb, nb, 0) for i in range(nbytes // nb)]
    for v in variants:
        snap.set_k1_variant(v)
        with snap.Ctx(0, nbytes) as c:
            c.fill_mix64(0, nbytes, 1, 0)
            c.set_buffers(bufs)
            for _ in range(3):
                c.snapshot()
                c.restore_self(verify=True)
            res = {}
            for name, fn in (("snapshot", c.snapshot), ("restore", lambda: c.restore_self(True))):
                best = []
                for _ in range(3):
                    c.sync()
                    c.prof_enable(True)
                    c.timer_start()
                    for _ in range(10):
                        fn()
                    best.append(c.timer_stop() / 10)
                    kin = {k: c.prof_read(k) for k in range(6)}
                    c.prof_enable(False)
                res[name] = (min(best), {k: round(t / max(n, 1), 4) for k, (t, n) in kin.items() if n})
            print(f"variant {v:3d} {snap.last_k1_kernel():60s} snapshot {res['snapshot'][0]:.4f} ms "
                  f"{res['snapshot'][1]} | restore {res['restore'][0]:.4f} ms {res['restore'][1]}",
                  flush=True)
    snap.set_k1_variant(-1)


if __name__ == "__main__":
    main()
