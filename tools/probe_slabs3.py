"""e2e time of the pipelined evaluate for ig-slab lists (GPP_SLABS) over the
canonical item schedule, paper size nw 3 (pinned host arrays)."""
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


def even(per, tail):
    rev, s = ([tail] if tail else []), tail
    while s < 128:
        rev.append(min(per, 128 - s)); s += rev[-1]
    return rev[::-1]


lists = [None] + [even(per, t) for per in (4, 6, 8, 10, 12, 16) for t in (0, 1, 2, 3)]
lists += [[16, 16, 16, 16, 14, 12, 10, 8, 6, 5, 4, 3, 2], [20, 18, 16, 14, 12, 10, 9, 8, 7, 6, 4, 2, 2]]
for sizes in lists:
    if sizes:
        assert sum(sizes) == 128, sizes
        os.environ["GPP_SLABS"] = ",".join(map(str, sizes))
    else:
        os.environ.pop("GPP_SLABS", None)
    for _ in range(3):
        ctx.evaluate_host(p, "rcp_sq")
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        for _ in range(4):
            ctx.evaluate_host(p, "rcp_sq")
        best = min(best, (time.perf_counter() - t0) / 4 * 1e3)
    print(f"wall {best:7.3f} ms  {sizes or 'default'}", flush=True)
