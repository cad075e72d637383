"""Minimal driver for ncu: one warm-up and one profiled evaluation.

usage: python tools/profile_run.py [nbands ngpown ncouls] [--nw 3] [--seed 1] [--variant rcp_sq] [--reps 2]
"""
import argparse
import sys

sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem

ap = argparse.ArgumentParser()
ap.add_argument("dims", nargs="*", type=int, default=[512, 66, 32768])
ap.add_argument("--nw", type=int, default=3)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--variant", default="rcp_sq")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
p = synth_problem(*a.dims, seed=a.seed, nw=a.nw, check=False)
ctx = GPPContext(0)
ctx.upload(p)
# The production (uncounted) kernel, as evaluate_variant and bench.py run it
# (run with GPP_BALANCED_TAIL=0 so that one launch covers the whole problem):
# profile with -k regex:gpp_sacc_kernel -s 1 -c 1 to capture the second launch.
tot, main = ctx.time(a.variant, a.reps)
print(a.variant, a.dims, "nw", a.nw, f"{main / a.reps:.3f} ms per launch")
