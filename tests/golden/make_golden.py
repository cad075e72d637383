"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [--big]

It imports ``rooflab`` read-only and records, per case:
  * sha256 of every synthesized array (pins our synth_problem to theirs),
  * ``reference_result`` (problem.py:179-208) where it finishes in seconds,
  * ``evaluate_variant`` for div / rcp / rcp_sq (kernel.py:98-114),
  * ``branch_stats`` per variant (kernel.py:130-137),
  * ``run_version`` counters for v0..v8 (kernel.py:191-212, runner.py:249-286).
nw=3 cases patch NW=3 into rooflab.gpp.problem, .kernel and .runner, the
three modules that import it by value (SURVEY.md Table R).
``--big`` adds the paper size (512, 66, 32768) and the weak-scaled size
(4096, 528, 65536); the weak case needs ~18 GB of RAM and ~1 minute.
``--append weak-nw3`` adds the weak size at nw = 3 (the bench default) to an
existing gpp_big.json.  ``--append sweep`` adds every point of the igp/ig
aspect-ratio sweep (BASELINE.json configs[4]: nbands 512, ngpown in
SWEEP_NGPOWN x ncouls in SWEEP_NCOULS, seed 1, nw 3) that gpp_big.json does
not hold yet.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import shutil
import time
from contextlib import contextmanager
from pathlib import Path

import numpy as np

import rooflab.gpp as gpp
import rooflab.gpp.kernel as gkernel
import rooflab.gpp.problem as gproblem
import rooflab.gpp.runner as grunner

HERE = Path(__file__).resolve().parent

SMALL_DIMS = [(1, 1, 1), (5, 3, 40), (47, 2, 33), (8, 8, 64), (32, 8, 512), (64, 64, 512)]
SEEDS = [1, 42, 7]
SWEEP_NGPOWN = (16, 33, 66, 132, 264, 528)
SWEEP_NCOULS = (8192, 16384, 32768, 65536)


@contextmanager
def patched_nw(nw: int):
    saved = (gproblem.NW, gkernel.NW, grunner.NW)
    gproblem.NW = gkernel.NW = grunner.NW = nw
    try:
        yield
    finally:
        gproblem.NW, gkernel.NW, grunner.NW = saved


def _sha(arr: np.ndarray) -> str:
    return hashlib.sha256(np.asarray(arr).tobytes(order="F")).hexdigest()


def _cplx(z) -> list[list[float]]:
    return [[float(v.real), float(v.imag)] for v in z]


def make_case(dims, seed, nw, with_reference: bool, versions: bool = True) -> dict:
    with patched_nw(nw):
        t0 = time.perf_counter()
        p = gpp.synth_problem(*dims, seed=seed)
        case = {
            "dims": list(dims),
            "seed": seed,
            "nw": nw,
            "sha256": {
                name: _sha(getattr(p, name))
                for name in ("wtilde", "i_eps", "aqsntemp", "aqsmtemp", "wx")
            },
            "wx": [float(v) for v in p.wx],
        }
        if with_reference:
            ref = gpp.reference_result(p)
            case["reference_result"] = {"achtemp": _cplx(ref.achtemp), "asxtemp": _cplx(ref.asxtemp)}
        case["evaluate_variant"] = {}
        case["branch_stats"] = {}
        for variant in ("div", "rcp", "rcp_sq"):
            if not versions and variant != "rcp_sq":
                continue
            r = gpp.evaluate_variant(p, variant)
            case["evaluate_variant"][variant] = {"achtemp": _cplx(r.achtemp), "asxtemp": _cplx(r.asxtemp)}
            s = gpp.branch_stats(p, variant)
            case["branch_stats"][variant] = [s.instances, s.near, s.far]
        if versions:
            case["counters"] = {
                name: gpp.run_version(p, name).counters.to_dict() for name in gpp.VERSION_NAMES
            }
        else:
            case["counters"] = {"v8": gpp.run_version(p, "v8").counters.to_dict()}
        case["gen_seconds"] = round(time.perf_counter() - t0, 2)
    print(f"case {dims} seed {seed} nw {nw}: {case['gen_seconds']} s", flush=True)
    return case


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--append", choices=("weak-nw3", "sweep"),
                    help="append one big case to the existing gpp_big.json and stop")
    args = ap.parse_args()

    if args.append == "sweep":
        path = HERE / "gpp_big.json"
        big = json.loads(path.read_text())
        have = {(tuple(c["dims"]), c["seed"], c["nw"]) for c in big["cases"]}
        for ngpown in SWEEP_NGPOWN:
            for ncouls in SWEEP_NCOULS:
                key = ((512, ngpown, ncouls), 1, 3)
                if key in have:
                    continue
                big["cases"].append(make_case(key[0], 1, 3, with_reference=False, versions=False))
                path.write_text(json.dumps(big, indent=1) + "\n")  # checkpoint per point
        return

    if args.append == "weak-nw3":
        # The bench's weak workload at its default frequency count (nw 3).
        path = HERE / "gpp_big.json"
        big = json.loads(path.read_text())
        big["cases"] = [c for c in big["cases"]
                        if not (c["dims"] == [4096, 528, 65536] and c["seed"] == 42 and c["nw"] == 3)]
        big["cases"].append(make_case((4096, 528, 65536), 42, 3, with_reference=False, versions=False))
        path.write_text(json.dumps(big, indent=1) + "\n")
        return

    cases = []
    for dims in SMALL_DIMS:
        for seed in SEEDS:
            for nw in (2, 3):
                cases.append(make_case(dims, seed, nw, with_reference=True))
    (HERE / "gpp_small.json").write_text(json.dumps({"cases": cases}, indent=1) + "\n")

    # Bundled KAT from the reference, copied verbatim as a fixture.
    shutil.copy(gproblem.bundled_golden_path(), HERE / "gpp-golden-seed42-64x64x512.json")

    # Hand-picked counter KATs (test_gpp.py:112-130) recomputed through the reference.
    stats = gkernel.BranchStats(instances=60, near=50, far=8)
    kats = []
    for variant, t_products, far_sqrt in (("div", 30, False), ("rcp", 30, False),
                                          ("rcp_sq", 30, True), ("rcp_sq", 60, True)):
        for contraction in (True, False):
            c = gkernel.counters_from_stats(variant, stats, t_products, far_sqrt, contraction)
            kats.append({"variant": variant, "t_products": t_products, "far_sqrt": far_sqrt,
                         "contraction": contraction, "counters": c.to_dict()})
    (HERE / "counter_kats.json").write_text(json.dumps(kats, indent=1) + "\n")

    if args.big:
        big = []
        big.append(make_case((512, 66, 32768), 1, 2, with_reference=True, versions=False))
        for seed, nw in ((42, 2), (1, 3), (42, 3)):
            big.append(make_case((512, 66, 32768), seed, nw, with_reference=False, versions=False))
        for ngpown, ncouls in ((16, 8192), (528, 8192), (33, 65536)):
            big.append(make_case((512, ngpown, ncouls), 1, 3, with_reference=False, versions=False))
        big.append(make_case((4096, 528, 65536), 42, 2, with_reference=False, versions=False))
        (HERE / "gpp_big.json").write_text(json.dumps({"cases": big}, indent=1) + "\n")


if __name__ == "__main__":
    main()
