"""Repeated end-to-end measurements (paper size nw 3) in one process:
pageable through the public seam and pinned, alternating, to see the spread.
GPP_HOST_THREADS / OMP_* from the environment."""
import os, sys, time
sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPProblem, evaluate_variant, synth_problem
from paper_2008_11326_b200._lib import check, load

p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
q = GPPProblem(p.nbands, p.ngpown, p.ncouls, p.wtilde.copy(order="F"), p.i_eps.copy(order="F"),
               p.aqsntemp.copy(order="F"), p.aqsmtemp.copy(order="F"), p.wx.copy())
lib = load()


def run(k=20):
    for _ in range(2):
        evaluate_variant(q, "rcp_sq")
    t0 = time.perf_counter()
    for _ in range(k):
        evaluate_variant(q, "rcp_sq")
    return (time.perf_counter() - t0) / k * 1e3


tag = f"threads={os.environ.get('GPP_HOST_THREADS', 'default')} omp_wait={os.environ.get('OMP_WAIT_POLICY', 'default')}"
for rep in range(3):
    pg = run()
    for a in (q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp):
        check(lib.gpp_host_register(a.ctypes.data, a.nbytes))
    pn = run()
    for a in (q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp):
        lib.gpp_host_unregister(a.ctypes.data)
    print(tag, f"rep {rep}: pageable {pg:.3f} ms  pinned {pn:.3f} ms", flush=True)
