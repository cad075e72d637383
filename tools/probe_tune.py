"""Time the fast kernel at the paper size under several GPP_TUNE settings."""
import os
import subprocess
import sys

CODE = r'''
import sys; sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem
from paper_2008_11326_b200.counters import algorithmic_flops
nw = int(sys.argv[1])
p = synth_problem(512, 66, 32768, seed=1, nw=nw, check=False)
ctx = GPPContext(0); ctx.upload(p)
r, (n, f), ms = ctx.run("rcp_sq")
info = ctx.kernel_info("rcp_sq")
ctx.time("rcp_sq", 3)
tot, main = ctx.time("rcp_sq", 20)
fl = algorithmic_flops(512, 66, 32768, nw, n, f)
print(f"  nw={nw} main {main/20:.3f} ms  {fl/(main/20*1e-3)/1e12:.2f} TF/s  {info}  ach0={r.achtemp[0]:.12e}", flush=True)
'''
for tune in sys.argv[1:] or ["", "2,2", "1,2", "1,3", "2,3", "3,3"]:
    env = dict(os.environ, GPP_TUNE=tune)
    print("GPP_TUNE=" + tune, flush=True)
    for nw in (3, 2):
        subprocess.run([sys.executable, "-c", CODE, str(nw)], env=env)
