"""e2e (paper size nw 3) for explicit slab lists (GPP_SLABS), pinned and
pageable inputs, median of three rounds of 8 calls each."""
import os, statistics, sys, time
sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, GPPProblem, synth_problem
from paper_2008_11326_b200._lib import check, load

p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
q = GPPProblem(p.nbands, p.ngpown, p.ncouls, p.wtilde.copy(order="F"), p.i_eps.copy(order="F"),
               p.aqsntemp.copy(order="F"), p.aqsmtemp.copy(order="F"), p.wx.copy())
ctx = GPPContext(0)
lib = load()


def med(fn):
    for _ in range(4):
        fn()
    r = []
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(8):
            fn()
        r.append((time.perf_counter() - t0) / 8 * 1e3)
    return statistics.median(r)


def even(per, last):
    rev, s = [last], last
    while s < 128:
        rev.append(min(per, 128 - s)); s += rev[-1]
    return rev[::-1]


def grow(last, step, per=6):
    rev, s, k = [last], last, 1
    while s < 128:
        rev.append(min(k * step, 128 - s)); s += rev[-1]; k += 1
    return rev[::-1]


lists = [None, grow(2, 6), grow(1, 6), grow(3, 6), grow(2, 3), grow(2, 9), grow(4, 6), grow(6, 6)]
for mode in ("pageable", "pinned"):
    if mode == "pinned":
        for a in (q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp):
            check(lib.gpp_host_register(a.ctypes.data, a.nbytes))
    for sizes in lists:
        if sizes:
            os.environ["GPP_SLABS"] = ",".join(map(str, sizes))
        else:
            os.environ.pop("GPP_SLABS", None)
        print(mode, f"{med(lambda: ctx.evaluate_host(q, 'rcp_sq')):7.3f}", sizes or "default", flush=True)
