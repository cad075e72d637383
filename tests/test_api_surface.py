"""The drop-in's public names: every name rooflab.gpp exports
(rooflab/gpp/__init__.py:8-48) exists here, trace helpers raise DomainError
(out of scope on B200), and the bundled known-answer file is the reference's.
CPU only."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

import paper_2008_11326_b200 as gpp
from conftest import GOLDEN

REF = Path("/root/reference/pkg/src")
# rooflab/gpp/__init__.py:8-48, for boxes without the reference.
REFERENCE_NAMES = {
    "BranchStats", "VariantTerms", "branch_stats", "complex_reciprocal", "counters_from_stats",
    "evaluate_variant", "primitive_table", "variant_terms", "BOUNDARY_MARGIN", "DEFAULT_DIMS",
    "LIMIT_ONE", "LIMIT_TWO", "NW", "SWEEP_DIMS", "TOL_ZERO", "GPPProblem", "GPPResult",
    "bundled_golden_path", "load_golden", "max_rel_error", "reference_result", "save_golden",
    "synth_problem", "ARRAY_NAMES", "VERSION_NAMES", "VERSIONS", "RunArtifacts", "VersionSpec",
    "block_sizes", "build_trace", "emit_metrics", "run_sweep", "run_version", "tuple_order",
    "version_spec",
}


def test_every_reference_name_exists():
    assert REFERENCE_NAMES - set(dir(gpp)) == set()


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted (GPU box)")
def test_reference_public_names_match_the_list():
    code = "import rooflab.gpp as g; print(' '.join(sorted(g.__all__)))"
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         env={**os.environ, "PYTHONPATH": str(REF), "PYTHONDONTWRITEBYTECODE": "1"})
    assert out.returncode == 0, out.stderr
    names = {n for n in out.stdout.split() if not n.startswith(("gpp", "kernel", "problem", "runner"))}
    assert names - set(dir(gpp)) == set()


def test_trace_helpers_raise_domain_error():
    for fn, args in ((gpp.build_trace, ("v8", 2, 2, 2)), (gpp.tuple_order, ("v8", 2, 2, 2)),
                     (gpp.block_sizes, (2, 2))):
        with pytest.raises(gpp.DomainError):
            fn(*args)
    assert gpp.ARRAY_NAMES == {0: "wtilde", 1: "i_eps", 2: "aqsntemp", 3: "aqsmtemp"}


def test_bundled_golden_is_the_reference_kat():
    path = gpp.bundled_golden_path()
    assert json.loads(path.read_text()) == json.loads((GOLDEN / "gpp-golden-seed42-64x64x512.json").read_text())
    dims, seed, result = gpp.load_golden(path)
    assert tuple(dims) == (64, 64, 512) and seed == 42
