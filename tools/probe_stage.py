"""Pageable e2e (paper size nw 3, the public seam) against the staging ring's
shape: GPP_STAGE_SLOTS x GPP_STAGE_MB and packing threads, one process per
setting (the settings are read once).  Median of three rounds of 10 calls."""
import os, statistics, subprocess, sys

CODE = r'''
import os, statistics, sys, time
sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPProblem, evaluate_variant, synth_problem
p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
q = GPPProblem(p.nbands, p.ngpown, p.ncouls, p.wtilde.copy(order="F"), p.i_eps.copy(order="F"),
               p.aqsntemp.copy(order="F"), p.aqsmtemp.copy(order="F"), p.wx.copy())
for _ in range(30):
    evaluate_variant(q, "rcp_sq")
r = []
for _ in range(3):
    t0 = time.perf_counter()
    for _ in range(10):
        evaluate_variant(q, "rcp_sq")
    r.append((time.perf_counter() - t0) / 10 * 1e3)
print(os.environ.get("GPP_STAGE_SLOTS", "4"), "x", os.environ.get("GPP_STAGE_MB", "8"), "MB, threads",
      os.environ.get("GPP_HOST_THREADS", "8"), f"{statistics.median(r):.3f} ms", flush=True)
'''
for slots, mb, th in [tuple(map(int, x.split(','))) for x in (sys.argv[1:] or ['4,8,8', '8,4,8', '4,4,8', '8,2,8', '6,4,8', '4,6,8', '3,8,8', '6,6,8', '12,2,8'])]:
    subprocess.run([sys.executable, "-c", CODE],
                   env=dict(os.environ, GPP_STAGE_SLOTS=str(slots), GPP_STAGE_MB=str(mb), GPP_HOST_THREADS=str(th)))
