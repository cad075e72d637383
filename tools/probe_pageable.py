"""End-to-end evaluate (host arrays -> result, paper size nw 3) from pageable
numpy arrays (library staging ring) vs page-locked arrays, and the bare H2D.
GPP_HOST_THREADS sets the packing threads (default: cores, at most 16)."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2008_11326_b200 import GPPContext, GPPProblem, evaluate_variant, synth_problem
from paper_2008_11326_b200._lib import check, load

p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
# writeable copies: the public evaluate_variant re-uploads them on every call
q = GPPProblem(p.nbands, p.ngpown, p.ncouls, p.wtilde.copy(order="F"), p.i_eps.copy(order="F"),
               p.aqsntemp.copy(order="F"), p.aqsmtemp.copy(order="F"), p.wx.copy())
print("cpus", os.cpu_count(), "threads", os.environ.get("GPP_HOST_THREADS", "default"), flush=True)


def timeit(fn, n=8):
    for _ in range(2):
        fn()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        best = min(best, (time.perf_counter() - t0) / n * 1e3)
    return best


ref = evaluate_variant(p, "rcp_sq")
got = evaluate_variant(q, "rcp_sq")
assert np.array_equal(ref.achtemp, got.achtemp) and np.array_equal(ref.asxtemp, got.asxtemp)
print(f"pageable evaluate_variant (public seam) {timeit(lambda: evaluate_variant(q, 'rcp_sq')):7.3f} ms", flush=True)
ctx = GPPContext(0)
print(f"pageable upload alone                   {timeit(lambda: ctx.upload(q, force=True)):7.3f} ms", flush=True)
lib = load()
for a in (q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp):
    check(lib.gpp_host_register(a.ctypes.data, a.nbytes))
print(f"pinned evaluate_variant                 {timeit(lambda: evaluate_variant(q, 'rcp_sq')):7.3f} ms", flush=True)
print(f"pinned upload alone                     {timeit(lambda: ctx.upload(q, force=True)):7.3f} ms", flush=True)
for a in (q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp):
    lib.gpp_host_unregister(a.ctypes.data)
