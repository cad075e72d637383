"""Production-kernel time at the paper size for several frequency counts."""
import sys
sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem
from paper_2008_11326_b200.counters import algorithmic_flops

ctx = GPPContext(0)
for nw in [int(x) for x in (sys.argv[1:] or ["2", "3", "4", "5", "6"])]:
    p = synth_problem(512, 66, 32768, seed=1, nw=nw, check=False)
    ctx.upload(p, force=True)
    _, (n, f), _ = ctx.run("rcp_sq")
    ctx.time("rcp_sq", 2)
    tot, main = ctx.time("rcp_sq", 10)
    fl = algorithmic_flops(512, 66, 32768, nw, n, f)
    print(f"nw={nw}: {tot / 10:.3f} ms/eval, {fl / (tot / 10 * 1e-3) / 1e12:.2f} TFLOP/s", flush=True)
