"""`gpp-run` on the B200 path: mirror of the reference's caller of the hot
path, rooflab/cli.py:126-186 (and its exit-code contract, cli.py:1-8 and
324-347: 0 success, 1 expected failure -- diverging result, RooflabError,
OSError -- 2 usage).

    python -m paper_2008_11326_b200 gpp-run --dims 512 66 32768 --seed 1 --nw 3

Synthesizes the problem, evaluates the literal nest (``reference_result``, the
``div`` formulation per instance on the GPU), runs the requested versions
through ``run_sweep`` (their B200 kernels), checks every result against the
reference within ``--rtol`` and optionally writes the KernelMetrics records
(metrics.py:131-217) to ``--out/metrics.json``.  The reference's element
traces and cache simulation (``--trace``, ``--simulate``) model hardware this
path measures with ncu; asking for them is a usage error.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
from pathlib import Path

from .counters import total_flops
from .errors import RooflabError
from .kernel import reference_result
from .problem import DEFAULT_DIMS, max_rel_error, synth_problem
from .runner import VERSION_NAMES, VERSIONS, emit_metrics, run_sweep


def _atomic_write_text(path: Path, text: str) -> None:
    """Write-then-rename (the reference's helper, cli.py:38-48)."""
    path.parent.mkdir(parents=True, exist_ok=True)
    fd, tmp = tempfile.mkstemp(dir=path.parent, prefix=path.name + ".", suffix=".tmp")
    try:
        with os.fdopen(fd, "w", encoding="utf-8") as fh:
            fh.write(text)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def cmd_gpp_run(args, parser: argparse.ArgumentParser) -> int:
    if min(args.dims) <= 0:
        parser.error("--dims values must all be positive")
    if args.trace or args.simulate:
        parser.error("--trace / --simulate model the cache hierarchy in rooflab; "
                     "the B200 path is profiled with ncu (tools/ncu_to_rooflab.py)")
    if args.versions == "all":
        names = list(VERSION_NAMES)
    else:
        names = [v.strip() for v in args.versions.split(",") if v.strip()]
        for name in names:
            if name not in VERSIONS:
                parser.error(f"unknown version {name!r}")
    nbands, ngpown, ncouls = args.dims
    problem = synth_problem(nbands, ngpown, ncouls, seed=args.seed, nw=args.nw)
    reference = reference_result(problem, device=args.device)
    artifacts = run_sweep(problem, names, device=args.device)
    system = args.system or f"synthetic-{nbands}x{ngpown}x{ncouls}-seed{args.seed}"
    records, worst = [], 0.0
    for art in artifacts:
        err = max_rel_error(art.result, reference)
        worst = max(worst, err)
        print(f"{art.version}: flops {total_flops(art.counters, args.div_weight):.6g} "
              f"near {art.stats.near} far {art.stats.far} rel-err {err:.3e} "
              f"kernel {art.kernel_s * 1e3:.3f} ms ({art.kernel})")
        records.append(emit_metrics(art, system=system))
    if worst > args.rtol:
        print(f"error: version results diverge from the reference beyond rtol {args.rtol:g} "
              f"(worst {worst:.3e})", file=sys.stderr)
        return 1
    print(f"all {len(artifacts)} versions within rtol {args.rtol:g} of reference")
    if args.out:
        out = Path(args.out) / "metrics.json"
        _atomic_write_text(out, json.dumps(records, indent=2) + "\n")
        print(f"wrote {out}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2008_11326_b200",
                                     description="GPP self-energy kernel on B200 (rooflab drop-in).")
    sub = parser.add_subparsers(dest="command", required=True)
    p_run = sub.add_parser("gpp-run", help="run the kernel versions on the GPU")
    p_run.add_argument("--dims", type=int, nargs=3, default=list(DEFAULT_DIMS),
                       metavar=("NBANDS", "NGPOWN", "NCOULS"))
    p_run.add_argument("--seed", type=int, default=42)
    p_run.add_argument("--nw", type=int, default=2, help="frequencies (the reference's NW)")
    p_run.add_argument("--versions", default="all", help="comma list or 'all'")
    p_run.add_argument("--out", default=None, help="directory for metrics.json")
    p_run.add_argument("--system", default=None, help="system label for metrics records")
    p_run.add_argument("--rtol", type=float, default=1e-10)
    p_run.add_argument("--div-weight", type=float, default=1.0)
    p_run.add_argument("--device", type=int, default=0)
    p_run.add_argument("--trace", action="store_true", help=argparse.SUPPRESS)
    p_run.add_argument("--simulate", default=None, help=argparse.SUPPRESS)
    return parser


def main(argv: list[str] | None = None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    try:
        if args.command == "gpp-run":
            return cmd_gpp_run(args, parser)
        parser.error(f"unknown command {args.command!r}")
    except RooflabError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    return 2


if __name__ == "__main__":
    sys.exit(main())
