"""Small evaluations for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family, ragged shapes, both upload paths, nw groups > 4, and
production-kernel schedules with several items per CTA (cross-item staging),
a balanced tail launch and two band windows."""
import sys

sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem

ctx = GPPContext(0)
for dims, nw in (((5, 3, 40), 2), ((47, 2, 33), 3), ((9, 7, 300), 5), ((16, 8, 512), 3)):
    p = synth_problem(*dims, seed=1, nw=nw)
    ctx.evaluate_host(p, "rcp_sq", counts=True, slabs=3)
    for v in ("rcp_sq", "rcp", "div"):
        ctx.run(v, counts=True)
        ctx.run(v, counts=False)
    ctx.time("rcp_sq", 1)
# Production schedules: (40, 5, 40000) = 471 items -> one whole wave of 296
# CTAs plus a balanced tail; (600, 2, 40000) = two band windows at nw 3.
for dims, nw in (((40, 5, 40000), 3), ((600, 2, 40000), 3), ((7, 3, 90000), 2)):
    p = synth_problem(*dims, seed=1, nw=nw, check=False)
    ctx.upload(p, force=True)
    ctx.run("rcp_sq", counts=True)
    ctx.run("rcp_sq", counts=False)
print("sanitize run ok")
