"""Quick device probe: FP64 peak, kernel timing at the paper size."""
import sys, time, json
sys.path.insert(0, '.')
from paper_2008_11326_b200 import GPPContext, synth_problem, fp64_peak
from paper_2008_11326_b200.counters import algorithmic_flops

for it in (20000, 200000):
    tf, ms = fp64_peak(0, it)
    print(f"fp64 peak iters={it}: {tf:.2f} TFLOP/s in {ms:.1f} ms", flush=True)
for nw in (3, 2):
    t = time.time(); p = synth_problem(512, 66, 32768, seed=1, nw=nw); print('synth', time.time()-t, flush=True)
    ctx = GPPContext(0)
    t = time.time(); ctx.upload(p); print('upload', time.time()-t, flush=True)
    for v in ('rcp_sq', 'rcp', 'div'):
        r, (n, f), ms = ctx.run(v)
        info = ctx.kernel_info(v)
        tot, main = ctx.time(v, 10)
        fl = algorithmic_flops(512, 66, 32768, nw, n, f)
        print(f"nw={nw} {v}: run {ms:.3f} ms; timed total {tot/10:.3f} main {main/10:.3f} ms/iter; "
              f"alg {fl/(main/10*1e-3)/1e12:.2f} TFLOP/s; near {n} far {f}; {info}", flush=True)
    ctx.close()
