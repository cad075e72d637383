"""Per-item overhead: production-kernel time of a band shard under forced
band chunks (GPP_TUNE=",,<bchunk>"), one subprocess per chunk."""
import os
import subprocess
import sys

CODE = r'''
import sys; sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem
nb = int(sys.argv[1])
p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
ctx = GPPContext(0); ctx.upload(p, (0, nb))
ctx.run("rcp_sq"); ctx.time("rcp_sq", 3)
tot, main = ctx.time("rcp_sq", 20)
print(f"  bands {nb} chunk {ctx.kernel_info('rcp_sq')['band_chunk']}: {tot / 20:.4f} ms", flush=True)
'''
for nb, chunks in ((64, (64, 32, 16, 8)), (512, (256, 128, 64, 32))):
    for bc in chunks:
        for tail in ("1", "0"):
            env = dict(os.environ, GPP_TUNE=f"0,0,{bc}", GPP_BALANCED_TAIL=tail)
            print(f"tail={tail}", end="", flush=True)
            subprocess.run([sys.executable, "-c", CODE, str(nb)], env=env)
