"""End-to-end (host arrays -> result) time vs the ig-slab schedule at paper
size: uniform counts and explicit block lists (GPP_SLABS)."""
import os
import sys
import time

sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem
from paper_2008_11326_b200._lib import check, load


def taper(n, m, r, last=1):
    out, s = [], last
    while sum(out) < n:
        out.append(min(m, s))
        s = max(s + 1, -(-s * r // 1))
    out[-1] -= sum(out) - n
    return [int(x) for x in reversed(out) if x > 0]


p = synth_problem(512, 66, 32768, seed=1, nw=int(os.environ.get("NW", "3")), check=False)
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
n = 128
cases = [("default", 0, None)] + [("uniform", k, None) for k in (8, 16, 32)]
if os.environ.get("SHORT"):
    cases = cases[:3]
for m in (() if os.environ.get("SHORT") else (16, 24, 128)):
    for r in (1.15, 1.2, 1.25):
        cases.append(("taper", 0, taper(n, m, r)))
for kind, k, sizes in cases:
    if sizes:
        os.environ["GPP_SLABS"] = ",".join(map(str, sizes))
    else:
        os.environ.pop("GPP_SLABS", None)
    for _ in range(2):
        ctx.evaluate_host(p, "rcp_sq", slabs=k)
    best, devs = 1e9, []
    for _ in range(5):
        t0 = time.perf_counter()
        for _ in range(4):
            _, _, ms = ctx.evaluate_host(p, "rcp_sq", slabs=k)
            devs.append(ms)
        best = min(best, (time.perf_counter() - t0) / 4 * 1e3)
    print(f"{kind:8s} {k:3d} wall {best:7.3f} ms  device {min(devs):7.3f} ms  {sizes or ''}",
          flush=True)
