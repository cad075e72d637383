"""Pageable e2e (library staging ring) for explicit ig-slab lists, paper size nw 3."""
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
    for _ in range(4):
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        best = min(best, (time.perf_counter() - t0) / n * 1e3)
    return best


tag = f"stage {os.environ.get('GPP_STAGE_MB', '8')} MB threads {os.environ.get('GPP_HOST_THREADS', 'dflt')}"
print(tag, f"upload {timeit(lambda: ctx.upload(q, force=True)):7.3f}", flush=True)
lists = [None, [32, 32, 32, 16, 8, 4, 2, 2], [40, 32, 24, 16, 8, 4, 2, 2], [48, 32, 24, 12, 6, 3, 2, 1],
         [64, 32, 16, 8, 4, 2, 2], [24, 24, 24, 20, 16, 10, 6, 2, 2], [16, 16, 16, 16, 14, 12, 10, 8, 6, 5, 4, 3, 2]]
for sizes in lists:
    if sizes:
        assert sum(sizes) == 128, sizes
        os.environ["GPP_SLABS"] = ",".join(map(str, sizes))
    else:
        os.environ.pop("GPP_SLABS", None)
    print(tag, f"{timeit(lambda: ctx.evaluate_host(q, 'rcp_sq')):7.3f}", sizes or "default", flush=True)
