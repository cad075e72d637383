"""Time of the factored path (gpp_run_factored: one fused kernel, band GEMM
on DMMA + branch terms) at the paper size and the weak size, with its error
against the per-instance kernel."""
import sys
import statistics

sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext
from paper_2008_11326_b200.problem import max_rel_error

ctx = GPPContext(0)
for dims, seed, nw in (((512, 66, 32768), 1, 3), ((512, 66, 32768), 1, 2), ((4096, 528, 65536), 42, 3)):
    ctx.synth(*dims, seed=seed, nw=nw)
    ref = ctx.run("rcp_sq", counts=False)[0]
    for v in ("rcp_sq", "div"):
        ctx.run_factored(v, counts=False)
        ms = [ctx.run_factored(v, counts=False)[2] for _ in range(7)]
        got = ctx.run_factored(v, counts=False)[0]
        nb, ng, nc = dims
        print(dims, "nw", nw, v, f"{statistics.median(ms):.3f} ms",
              f"GEMM {8 * nb * ng * nc / (statistics.median(ms) * 1e-3) / 1e12:.1f} TFLOP/s-equiv",
              f"err vs per-instance {max_rel_error(got, ref):.2e}", flush=True)
