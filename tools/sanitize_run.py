"""Small evaluations for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family (production sacc + slot finalize, counting
kernel, ladder / as-written kernels + their finalize, fused factored kernel,
device synthesis, variant terms), ragged shapes, nw groups > 3, the
pipelined evaluate over ig slabs from pageable (staging ring) and pinned
host arrays, production schedules with several items per CTA (cross-item
staging), a balanced tail launch, two band windows, an empty band shard and
the single-process group path.  GPP_COLUMN_UPLOAD=1 in the environment runs
the column-split wtilde / i_eps upload (the sharded e2e path) on one rank."""
import sys

sys.path.insert(0, ".")
import numpy as np

from paper_2008_11326_b200 import GPPContext, GPPProblem, synth_problem, variant_terms
from paper_2008_11326_b200._lib import check, load
from paper_2008_11326_b200.dist import MultiDeviceGPP

ctx = GPPContext(0)
for dims, nw in (((5, 3, 40), 2), ((47, 2, 33), 3), ((9, 7, 300), 5), ((16, 8, 512), 3)):
    p = synth_problem(*dims, seed=1, nw=nw)
    ctx.evaluate_host(p, "rcp_sq", counts=True, slabs=3)
    ctx.evaluate_host(p, "div", counts=False, slabs=2)
    for v in ("rcp_sq", "rcp", "div", "rcp_sq/split", "rcp_sq/iw", "rcp_sq/seed"):
        ctx.run(v, counts=True)
        ctx.run(v, counts=False)
    for v in ("rcp_sq", "rcp", "div"):
        ctx.run_factored(v, counts=True)
    ctx.time("rcp_sq", 1)
variant_terms(synth_problem(8, 5, 64, seed=2, nw=3), "rcp_sq")
# Production schedules: (40, 5, 40000) = one whole wave of 296 CTAs plus a
# balanced tail; (600, 2, 40000) = two band windows at nw 3; pageable and
# pinned sources through the staging ring / direct DMA.
lib = load()
for dims, nw in (((40, 5, 40000), 3), ((600, 2, 40000), 3), ((7, 3, 90000), 2)):
    p = synth_problem(*dims, seed=1, nw=nw, check=False)
    q = GPPProblem(*dims, p.wtilde.copy(order="F"), p.i_eps.copy(order="F"),
                   p.aqsntemp.copy(order="F"), p.aqsmtemp.copy(order="F"), p.wx.copy())
    ctx.evaluate_host(q, "rcp_sq", counts=False)           # pageable: staging ring
    for a in (q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp):
        check(lib.gpp_host_register(a.ctypes.data, a.nbytes))
    ctx.evaluate_host(q, "rcp_sq", counts=True)            # pinned: direct
    for a in (q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp):
        lib.gpp_host_unregister(a.ctypes.data)
    ctx.upload(p, force=True)
    ctx.run("rcp_sq", counts=True)
    ctx.run("rcp_sq", counts=False)
    ctx.synth(*dims, seed=1, nw=nw, band_range=(1, dims[0] - 1))
    ctx.run("rcp_sq", counts=False)
# Empty band shard (more ranks than bands).
p = synth_problem(6, 5, 700, seed=2, nw=3, check=False)
ctx.upload(p, (3, 3), force=True)
ctx.run("rcp_sq", counts=True)
ctx.evaluate_host(p, "rcp_sq", band_range=(6, 6), counts=True)
ctx.close()
# Single-process group path on one device.
g = MultiDeviceGPP([0])
g.synth(40, 5, 40000, seed=1, nw=3)
g.run("rcp_sq", counts=True)
g.time("rcp_sq", 2)
g.evaluate(synth_problem(40, 5, 40000, seed=1, nw=3, check=False), "rcp_sq")
g.close()
print("sanitize run ok")
