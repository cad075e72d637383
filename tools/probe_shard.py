"""Per-GPU step time of the N-way band shard of the paper problem (strong
scaling projection without the collective): nbands/N bands on one B200."""
import sys

sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem
from paper_2008_11326_b200.counters import algorithmic_flops

p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
ctx = GPPContext(0)
base = None
for n in (1, 2, 4, 8):
    b1 = 512 // n
    ctx.upload(p, (0, b1), force=True)
    ctx.time("rcp_sq", 3)
    tot, main = ctx.time("rcp_sq", 50)
    ms = tot / 50
    if base is None:
        base = ms
    info = ctx.kernel_info("rcp_sq")
    print(f"N={n}: shard {b1} bands  step {ms:.4f} ms  (ideal {base / n:.4f})  efficiency {base / n / ms:.3f}  {info}", flush=True)
