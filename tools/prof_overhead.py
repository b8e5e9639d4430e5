import os, sys
sys.path.insert(0, '/root/repo')
import paper_2202_07848_b200 as snap
from bench import c2_layout, fill_rank
bufs, rep, per = c2_layout()
ctx = snap.Ctx(0, rep + per + (64 << 20))
fill_rank(ctx, 0, rep, per)
ctx.set_buffers(bufs)
for _ in range(5): ctx.snapshot()
for rnd in range(3):
    for prof in (False, True):
        ctx.sync(); ctx.prof_enable(prof)
        ctx.timer_start()
        for _ in range(100): ctx.snapshot()
        ms = ctx.timer_stop() / 100
        ctx.prof_enable(False)
        print("prof", prof, round(ms, 4))
