"""time the reference's literal loop-nest oracle
reference_result (rooflab/gpp/problem.py:179-208) and its production CPU
path evaluate_variant (kernel.py:98-114) on this host, tiny and paper sizes,
with the unmodified rooflab from baseline/_ref.  One JSON line per case.

    python tools/cpu_reference_result.py > profiles/r02_cpu_reference_result.json
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import rooflab.gpp as g  # noqa: E402
import rooflab.gpp.kernel as rk  # noqa: E402
import rooflab.gpp.problem as rp  # noqa: E402
import rooflab.gpp.runner as rr  # noqa: E402

print(json.dumps({"host": bench.host_info(), "rooflab": g.__file__}), flush=True)
for dims, seed, nw in (((32, 8, 512), 42, 2), ((512, 66, 32768), 1, 2), ((512, 66, 32768), 1, 3)):
    rp.NW = rk.NW = rr.NW = nw
    p = g.synth_problem(*dims, seed=seed)
    rec = {"dims": dims, "seed": seed, "nw": nw}
    t0 = time.perf_counter()
    r = g.reference_result(p)
    rec["reference_result_s"] = round(time.perf_counter() - t0, 3)
    best = min((lambda t0: (g.evaluate_variant(p, "rcp_sq"), time.perf_counter() - t0)[1])(time.perf_counter())
               for _ in range(3))
    rec["evaluate_variant_best_of_3_s"] = round(best, 4)
    art = g.run_version(p, "v8")
    rec["run_version_v8_elapsed_s"] = round(art.elapsed_s, 4)
    rec["achtemp0"] = [r.achtemp[0].real, r.achtemp[0].imag]
    print(json.dumps(rec), flush=True)
