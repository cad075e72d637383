"""End-to-end (host arrays -> result) timing vs ig-slab count (paper size)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem
from paper_2008_11326_b200._lib import check, load

p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
lib = load()
arrs = [p.wtilde, p.i_eps, p.aqsntemp, p.aqsmtemp]
for a in arrs:
    check(lib.gpp_host_register(a.ctypes.data, a.nbytes))
ctx = GPPContext(0)
ctx.upload(p, force=True)
ctx.run("rcp_sq", counts=False)
for _ in range(2):
    ctx.upload(p, force=True)
t0 = time.perf_counter()
for _ in range(10):
    ctx.upload(p, force=True)
print(f"upload alone            {(time.perf_counter() - t0) / 10 * 1e3:7.2f} ms")
t0 = time.perf_counter()
for _ in range(10):
    ctx.upload(p, force=True)
    ctx.run("rcp_sq", counts=False)
print(f"upload + run            {(time.perf_counter() - t0) / 10 * 1e3:7.2f} ms")
for slabs in (1, 2, 4, 8, 16, 32):
    ctx.evaluate_host(p, "rcp_sq", slabs=slabs)
    t0 = time.perf_counter()
    for _ in range(10):
        r, _, ms = ctx.evaluate_host(p, "rcp_sq", slabs=slabs)
    print(f"evaluate_host slabs={slabs:3d} {(time.perf_counter() - t0) / 10 * 1e3:7.2f} ms (device {ms:.2f} ms)")
