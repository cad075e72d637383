"""bench.py's reference arm runs on the CPU (the reference's algorithm on
host cores) and prints one JSON line with the driver contract's keys.  CPU
only; the GPU arm's line is checked on the GPU box by running bench.py."""
import json
import subprocess
import sys

from pathlib import Path

from conftest import ROOT

KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def test_reference_arm_prints_contract_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "TFLOP/s"
    assert d["higher_is_better"] is True and d["n_gpus"] == 1
    # the unmodified reference when baseline/_ref holds it, else the oracle port
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["cpu_model"] and d["cpu_baseline"]["OPENBLAS_NUM_THREADS"]
    assert d["numerator"]["flops_per_step"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("paper")


def test_live_capture_record_reads_through_the_reference_importer(tmp_path):
    """bench.py writes its live ncu capture in the reference's profiler-CSV
    columns (rooflab/metrics.py:228-237); the reference's own
    import_profiler_csv reads it back (when the reference is mounted)."""
    import importlib
    import os

    import pytest

    sys.path.insert(0, str(ROOT))
    bench = importlib.import_module("bench")
    rec = {"label": "gpp_sacc_kernel (512, 66, 32768) nw3 x1 shards", "runtime": 4.13e-3,
           "counters": {"dadd": 3529506816, "dmul": 15644884992, "dfma": 38859177984, "ddiv": 0, "dother": 0},
           "bytes": {"l1": 1.0e11, "l2": 2.0e10, "hbm": 4.4e8}, "system": "B200"}
    path = tmp_path / "cap.csv"
    bench.rooflab_csv(rec, path)
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "rooflab").is_dir():
        ref = Path("/root/reference/pkg/src")
    if not (ref / "rooflab").is_dir():
        pytest.skip("reference not available")
    code = ("import sys; from rooflab.metrics import import_profiler_csv, total_flops; "
            f"r = import_profiler_csv({str(path)!r})[0]; "
            "print(r.label, r.runtime, total_flops(r.counters), r.bytes.hbm)")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         env={**os.environ, "PYTHONPATH": str(ref), "PYTHONDONTWRITEBYTECODE": "1"})
    assert out.returncode == 0, out.stderr[-2000:]
    fields = out.stdout.split()
    assert float(fields[-3]) == rec["runtime"]
    assert float(fields[-2]) == 2 * 38859177984 + 15644884992 + 3529506816
    assert float(fields[-1]) == rec["bytes"]["hbm"]
