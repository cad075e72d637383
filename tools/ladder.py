"""The paper's version ladder (v0..v8) re-derived on B200.

For each reference version (rooflab/gpp/runner.py:75-115) run the B200
kernel that implements its step (runner.B200_KERNEL) on one workload and
report device time and the version's algorithmic FLOP rate (the reference's
own per-version counters, kernel.py:191-212).  With --ncu, every version is
launched exactly once after one counting launch, for

    ncu --metrics <list> -k regex:"gpp_main_kernel|gpp_sacc_kernel" -s 1 -c 9 python tools/ladder.py --ncu

whose CSV tools/ncu_to_rooflab.py turns into the reference's metrics format.
"""
import argparse
import json
import sys

sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem
from paper_2008_11326_b200.counters import BranchStats, counters_from_stats, total_flops
from paper_2008_11326_b200.runner import B200_KERNEL, VERSIONS

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=3, default=[512, 66, 32768])
ap.add_argument("--nw", type=int, default=3)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--ncu", action="store_true")
a = ap.parse_args()

p = synth_problem(*a.dims, seed=a.seed, nw=a.nw, check=False)
ctx = GPPContext(0)
ctx.upload(p)
_, (near, far), _ = ctx.run("rcp_sq", counts=True)
nb, ng, nc = a.dims
tuples = nb * ng * nc
stats = BranchStats(a.nw * tuples, near, far)
for name, spec in VERSIONS.items():
    kernel = B200_KERNEL[name]
    cnt = counters_from_stats(spec.variant, stats, tuples * (a.nw if spec.t_per_instance else 1),
                              spec.far_takes_sqrt)
    if a.ncu:
        ctx.time(kernel, 1)
        print(json.dumps({"version": name, "kernel": kernel}), flush=True)
        continue
    ctx.time(kernel, 2)
    tot, main = ctx.time(kernel, a.iters)
    ms = main / a.iters
    info = ctx.kernel_info(kernel)
    print(json.dumps({
        "version": name, "kernel": kernel, "dims": a.dims, "nw": a.nw, "seed": a.seed,
        "kernel_ms": round(ms, 4), "alg_flops": total_flops(cnt),
        "alg_tflops": round(total_flops(cnt) / (ms * 1e-3) / 1e12, 3),
        "registers_per_thread": info["registers_per_thread"],
        "threads_per_block": info["threads_per_block"],
        "warps_per_sm": info["blocks_per_sm"] * info["threads_per_block"] // 32,
        "description": spec.description}), flush=True)
