import os, sys, time
sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPProblem, evaluate_variant, synth_problem
from paper_2008_11326_b200._lib import check, load
p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
q = GPPProblem(p.nbands, p.ngpown, p.ncouls, p.wtilde.copy(order="F"), p.i_eps.copy(order="F"),
               p.aqsntemp.copy(order="F"), p.aqsmtemp.copy(order="F"), p.wx.copy())
lib = load()
def run(k=20):
    t0 = time.perf_counter()
    for _ in range(k): evaluate_variant(q, "rcp_sq")
    return (time.perf_counter() - t0) / k * 1e3
for rep in range(6):
    print("pageable only, rep", rep, f"{run():.3f}", flush=True)
for a in (q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp):
    check(lib.gpp_host_register(a.ctypes.data, a.nbytes))
print("pinned", f"{run():.3f}", flush=True)
for a in (q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp):
    lib.gpp_host_unregister(a.ctypes.data)
for rep in range(3):
    print("pageable after register/unregister, rep", rep, f"{run():.3f}", flush=True)
