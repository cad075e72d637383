"""Paper-size timing of alternative library builds (GPP_B200_LIB per
subprocess): main-kernel ms and the result's error against the golden
reference output.  usage: python tools/probe_variants.py lib1.so lib2.so ..."""
import os
import subprocess
import sys

CODE = r'''
import json, sys; sys.path.insert(0, ".")
import numpy as np
from paper_2008_11326_b200 import GPPContext
from paper_2008_11326_b200.problem import GPPResult, max_rel_error
c = GPPContext(0)
import os
nw = int(os.environ.get("NW", "3"))
c.synth(512, 66, 32768, seed=1, nw=nw)
r = c.run("rcp_sq", counts=False)[0]
info = c.kernel_info("rcp_sq")
c.time("rcp_sq", 3)
tot, main = c.time("rcp_sq", 20)
case = next((x for x in json.load(open("tests/golden/gpp_big.json"))["cases"]
             if x["dims"] == [512, 66, 32768] and x["seed"] == 1 and x["nw"] == nw), None)
want = None
if case:
    ev = case["evaluate_variant"]["rcp_sq"]
    want = GPPResult(np.array([complex(*z) for z in ev["achtemp"]]), np.array([complex(*z) for z in ev["asxtemp"]]))
c.synth(512, 66, 32768, seed=1, nw=nw, band_range=(0, 64))
c.time("rcp_sq", 3)
t8, m8 = c.time("rcp_sq", 20)
print(f"nw {nw} {sys.argv[1]:40s} main {main / 20:.4f} ms  shard/8 {m8 / 20:.4f} ms  err {max_rel_error(r, want) if want else float("nan"):.2e}  {info}", flush=True)
'''
for rnd in range(2):
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, "-c", CODE, lib], env=dict(os.environ, GPP_B200_LIB=lib))
