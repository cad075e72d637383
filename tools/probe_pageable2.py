"""Pageable e2e breakdown: slab schedules, staging size (GPP_STAGE_MB) --
paper size nw 3; prints ms per evaluate_host call."""
import os, sys, time
sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, GPPProblem, synth_problem

p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
q = GPPProblem(p.nbands, p.ngpown, p.ncouls, p.wtilde.copy(order="F"), p.i_eps.copy(order="F"),
               p.aqsntemp.copy(order="F"), p.aqsmtemp.copy(order="F"), p.wx.copy())
ctx = GPPContext(0)


def timeit(fn, n=6):
    for _ in range(2):
        fn()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        best = min(best, (time.perf_counter() - t0) / n * 1e3)
    return best


tag = f"stage {os.environ.get('GPP_STAGE_MB', '8')} MB threads {os.environ.get('GPP_HOST_THREADS', 'dflt')} omp_wait {os.environ.get('OMP_WAIT_POLICY', 'dflt')}"
print(tag, f"upload {timeit(lambda: ctx.upload(q, force=True)):7.3f}", flush=True)
for slabs in (0, 1, 4, 16, 32, 64):
    print(tag, f"slabs {slabs:3d} {timeit(lambda: ctx.evaluate_host(q, 'rcp_sq', slabs=slabs)):7.3f}", flush=True)
