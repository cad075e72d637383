"""e2e time for explicit ig-slab lists (GPP_SLABS), paper size nw 3."""
import os, sys, time
sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem
from paper_2008_11326_b200._lib import check, load

p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
lib = load()
for a in (p.wtilde, p.i_eps, p.aqsntemp, p.aqsmtemp):
    check(lib.gpp_host_register(a.ctypes.data, a.nbytes))
ctx = GPPContext(0)
ctx.upload(p, force=True)
ctx.run("rcp_sq", counts=False)
t0 = time.perf_counter()
for _ in range(10):
    ctx.upload(p, force=True)
print(f"upload alone {(time.perf_counter() - t0) / 10 * 1e3:7.3f} ms", flush=True)
lists = [None, [22, 22, 18, 15, 12, 10, 8, 6, 5, 4, 3, 2, 1], [40, 30, 22, 16, 10, 6, 3, 1],
         [48, 36, 24, 12, 6, 2], [64, 32, 16, 8, 4, 2, 1, 1], [30, 30, 25, 20, 12, 8, 3],
         [36, 30, 24, 16, 10, 6, 4, 2], [28, 26, 22, 18, 14, 10, 6, 3, 1], [44, 34, 24, 14, 8, 3, 1]]
for sizes in lists:
    if sizes:
        assert sum(sizes) == 128, sizes
        os.environ["GPP_SLABS"] = ",".join(map(str, sizes))
    else:
        os.environ.pop("GPP_SLABS", None)
    for _ in range(3):
        ctx.evaluate_host(p, "rcp_sq")
    best = 1e9
    for _ in range(6):
        t0 = time.perf_counter()
        for _ in range(4):
            ctx.evaluate_host(p, "rcp_sq")
        best = min(best, (time.perf_counter() - t0) / 4 * 1e3)
    print(f"wall {best:7.3f} ms  {sizes or 'default'}", flush=True)
