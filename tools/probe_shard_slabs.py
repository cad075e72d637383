import json, os, sys, time
sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, GPPProblem, synth_problem
from paper_2008_11326_b200._lib import check, load
from paper_2008_11326_b200.dist import band_range
n = int(os.environ.get("GPP_COLUMN_SIM", "1"))
p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
br = band_range(512, n, 0)
ctx = GPPContext(0)
lib = load()
for a in (p.wtilde, p.i_eps, p.aqsntemp, p.aqsmtemp):
    check(lib.gpp_host_register(a.ctypes.data, a.nbytes))
for slabs in (0, 1, 2, 4, 8, 16, 32):
    for _ in range(3): ctx.evaluate_host(p, "rcp_sq", band_range=br, slabs=slabs)
    t0 = time.perf_counter(); dms = []
    for _ in range(10): dms.append(ctx.evaluate_host(p, "rcp_sq", band_range=br, slabs=slabs)[2])
    wall = (time.perf_counter() - t0) / 10 * 1e3
    print(n, slabs, f"wall {wall:.3f} device {min(dms):.3f}", flush=True)
t0 = time.perf_counter()
for _ in range(10): ctx.upload(p, br, force=True)
print(n, "upload", (time.perf_counter() - t0) / 10 * 1e3)
