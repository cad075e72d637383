"""Projection of the band-sharded end-to-end step at N GPUs from ONE GPU
(every box this round has one): rank 0's work of an N-way shard -- its
aqsntemp / aqsmtemp band shard, its 1/N of the wtilde / i_eps columns (the
column-split upload, GPP_COLUMN_SIM=N), the pipelined evaluation -- timed
through gpp_evaluate_host from pageable and from pinned host arrays.  The
NCCL broadcast of the other (N-1)/N columns over NVLink and the allreduce
are not included (reported separately as an estimate).  Prints one JSON
line per N.  Run:  for n in 1 2 4 8; do GPP_COLUMN_SIM=$n python tools/probe_shard_e2e.py; done
"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, GPPProblem, synth_problem
from paper_2008_11326_b200._lib import check, load
from paper_2008_11326_b200.dist import band_range

n = int(os.environ.get("GPP_COLUMN_SIM", "1"))
p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
q = GPPProblem(p.nbands, p.ngpown, p.ncouls, p.wtilde.copy(order="F"), p.i_eps.copy(order="F"),
               p.aqsntemp.copy(order="F"), p.aqsmtemp.copy(order="F"), p.wx.copy())
br = band_range(512, n, 0)
ctx = GPPContext(0)


def timeit(fn, k=10):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(k):
            fn()
        best = min(best, (time.perf_counter() - t0) / k * 1e3)
    return best


page = timeit(lambda: ctx.evaluate_host(q, "rcp_sq", band_range=br))
lib = load()
for a in (q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp):
    check(lib.gpp_host_register(a.ctypes.data, a.nbytes))
pin = timeit(lambda: ctx.evaluate_host(q, "rcp_sq", band_range=br))
ctx.upload(q, br, force=True)
tot, main = ctx.time("rcp_sq", 20)
h2d = 2 * 16 * 32768 * 66 // n + 16 * 32768 * (br[1] - br[0]) + 16 * 66 * (br[1] - br[0])
bcast = 2 * 16 * 32768 * 66 * (n - 1) / n
print(json.dumps({"N": n, "rank0_bands": br, "h2d_bytes_rank0": h2d, "e2e_ms_pageable": round(page, 3),
                  "e2e_ms_pinned": round(pin, 3), "compute_ms": round(tot / 20, 3),
                  "nvlink_broadcast_bytes_in": int(bcast),
                  "nvlink_broadcast_ms_est_at_600GBps": round(bcast / 600e9 * 1e3, 3)}), flush=True)
