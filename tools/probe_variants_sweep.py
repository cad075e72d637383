"""Aspect-ratio sweep timings (main kernel ms, device synthesis) for
alternative library builds: python tools/probe_variants_sweep.py lib1 lib2 ..."""
import os
import subprocess
import sys

CODE = r'''
import os, sys; sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext
nw = int(os.environ.get("NW", "3"))
c = GPPContext(0)
out = []
for nc in (8192, 16384, 32768, 65536):
    for ng in (16, 33, 66, 132, 264, 528):
        c.synth(512, ng, nc, seed=1, nw=nw)
        it = max(5, min(40, int(2e10 / (512 * ng * nc))))
        c.time("rcp_sq", 2)
        tot, main = c.time("rcp_sq", it)
        out.append(main / it)
print("nw", nw, sys.argv[1].split("/")[-1], " ".join(f"{x:.4f}" for x in out), flush=True)
'''
for lib in sys.argv[1:]:
    subprocess.run([sys.executable, "-c", CODE, lib], env=dict(os.environ, GPP_B200_LIB=lib))
