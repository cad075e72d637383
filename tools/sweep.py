"""BASELINE configs[4]: igp/ig aspect-ratio sweep on one B200 (nbands 512,
nw 3, seed 1), plus the per-GPU shard of the weak-scaled config
(4096, 528, 65536) over 8 GPUs = (512, 528, 65536).

Prints one JSON line per point: device time of the production kernel
(CUDA events, mean of `iters` after warm-up), algorithmic TFLOP/s, fraction
of the live DFMA peak, and the kernel's launch shape.
"""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, fp64_peak, synth_problem
from paper_2008_11326_b200.counters import algorithmic_flops

NGPOWN = (16, 33, 66, 132, 264, 528)
NCOULS = (8192, 16384, 32768, 65536)
peak, _ = fp64_peak(0, 300_000)
print(json.dumps({"fp64_peak_tflops": peak}), flush=True)
ctx = GPPContext(0)
points = [(512, g, c) for c in NCOULS for g in NGPOWN]
for nb, ng, nc in points:
    t0 = time.perf_counter()
    p = synth_problem(nb, ng, nc, seed=1, nw=3, check=False)
    synth_s = time.perf_counter() - t0
    ctx.upload(p, force=True)
    _, (near, far), _ = ctx.run("rcp_sq", counts=True)
    iters = max(3, min(50, int(2e10 / (nb * ng * nc))))
    ctx.time("rcp_sq", 2)
    tot, main = ctx.time("rcp_sq", iters)
    ms = main / iters
    fl = algorithmic_flops(nb, ng, nc, 3, near, far)
    tf = fl / (ms * 1e-3) / 1e12
    print(json.dumps({"dims": [nb, ng, nc], "nw": 3, "seed": 1, "kernel_ms": round(ms, 4),
                      "alg_tflops": round(tf, 3), "frac_peak": round(tf / peak, 4),
                      "far_frac": round(far / (3 * nb * ng * nc), 4), "info": ctx.kernel_info("rcp_sq"),
                      "synth_s": round(synth_s, 1)}), flush=True)
    del p
