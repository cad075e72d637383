"""Production-kernel time (nw 3) at a few (nbands, ngpown, ncouls) points."""
import sys
sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem
from paper_2008_11326_b200.counters import algorithmic_flops

pts = [(512, 66, 32768), (512, 528, 8192), (512, 16, 8192), (512, 33, 65536), (512, 264, 32768)]
ctx = GPPContext(0)
for dims in pts:
    p = synth_problem(*dims, seed=1, nw=3, check=False)
    ctx.upload(p, force=True)
    _, (n, f), _ = ctx.run("rcp_sq")
    ctx.time("rcp_sq", 2)
    it = max(3, min(30, int(2e10 / (dims[0] * dims[1] * dims[2]))))
    tot, _ = ctx.time("rcp_sq", it)
    fl = algorithmic_flops(*dims, 3, n, f)
    print(f"{dims}: {tot / it:.4f} ms  {fl / (tot / it * 1e-3) / 1e12:.2f} TF/s  chunk {ctx.kernel_info('rcp_sq')['band_chunk']}", flush=True)
