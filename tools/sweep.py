"""BASELINE configs[4]: igp/ig aspect-ratio sweep on one B200 (nbands 512,
nw 3, seed 1), plus the per-GPU shard of the weak-scaled config
(4096, 528, 65536) over 8 GPUs = (512, 528, 65536).

Prints one JSON line per point: device time of the production kernel (CUDA
events, mean of `iters` after warm-up), the ncu-counted FP64 FLOPs of one
evaluation of THIS build (live ncu capture, bench.ncu_capture) and the
executed TFLOP/s they give, the reference's algorithmic (effective) rate,
both as fractions of the live DFMA peak, FP64-pipe activity, and the
kernel's launch shape.  Inputs are drawn on the device (gpp_synth).

    python tools/sweep.py [--no-ncu]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2008_11326_b200 import GPPContext, fp64_peak  # noqa: E402
from paper_2008_11326_b200.counters import algorithmic_flops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--no-ncu", action="store_true")
a = ap.parse_args()
NGPOWN = (16, 33, 66, 132, 264, 528)
NCOULS = (8192, 16384, 32768, 65536)
peak, _ = fp64_peak(0, 300_000)
print(json.dumps({"fp64_peak_tflops": peak, "lib_sha256": bench.lib_sha256()}), flush=True)
ctx = GPPContext(0)
for nc in NCOULS:
    for ng in NGPOWN:
        nb = 512
        ctx.synth(nb, ng, nc, seed=1, nw=3)
        _, (near, far), _ = ctx.run("rcp_sq", counts=True)
        iters = max(5, min(50, int(2e10 / (nb * ng * nc))))
        ctx.time("rcp_sq", 3)
        tot, main = ctx.time("rcp_sq", iters)
        ms, step_ms = main / iters, tot / iters
        fl = algorithmic_flops(nb, ng, nc, 3, near, far)
        rec = {"dims": [nb, ng, nc], "nw": 3, "seed": 1, "kernel_ms": round(ms, 4),
               "step_ms": round(step_ms, 4), "alg_tflops": round(fl / (ms * 1e-3) / 1e12, 3),
               "alg_frac_peak": round(fl / (ms * 1e-3) / 1e12 / peak, 4),
               "far_frac": round(far / (3 * nb * ng * nc), 4), "info": ctx.kernel_info("rcp_sq")}
        if not a.no_ncu:
            cap = bench.ncu_capture(argparse.Namespace(workload="paper", dims=[nb, ng, nc], nw=3, seed=1,
                                                       variant="rcp_sq", gpus=1))
            if cap and "error" not in cap:
                ex = cap["executed_flops_main"] / (ms * 1e-3) / 1e12
                rec.update({"executed_flops": cap["executed_flops_main"], "ncu_tflops": round(ex, 3),
                            "ncu_frac_peak": round(ex / peak, 4),
                            "fp64_pipe_pct": round(cap["fp64_pipe_pct"], 2),
                            "fma_ratio": round(cap["fma_ratio"], 4),
                            "dram_bytes": cap["dram_bytes_main"]})
            else:
                rec["ncu_error"] = (cap or {}).get("error")
        print(json.dumps(rec), flush=True)
