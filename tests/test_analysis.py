"""The ncu -> rooflab analysis pipeline, CPU only.

The committed B200 ladder counters (profiles/r01_b200_ladder.*) and machine
file must be readable by the unmodified reference's own loaders when the
reference is available (this container); the converter is checked on a
hand-written ncu CSV everywhere.
"""
import csv
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import ROOT

REF = Path("/root/reference/pkg/src")


def _write_ncu_csv(path):
    rows = [["ID", "Process ID", "Process Name", "Host Name", "Kernel Name", "Context", "Stream",
             "Block Size", "Grid Size", "Device", "CC", "Section Name", "Metric Name", "Metric Unit",
             "Metric Value"]]
    vals = {"gpu__time_duration.sum": ("ms", "2.5"),
            "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": ("inst", "10"),
            "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": ("inst", "20"),
            "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": ("inst", "30"),
            "l1tex__t_bytes.sum": ("Mbyte", "4"), "lts__t_bytes.sum": ("Mbyte", "2"),
            "dram__bytes.sum": ("Kbyte", "1"), "launch__registers_per_thread": ("register/thread", "128"),
            "launch__block_size": ("", "256"), "sm__warps_active.avg.per_cycle_active": ("warp", "15.6")}
    for lid in ("0", "1"):
        for name, (unit, v) in vals.items():
            rows.append([lid, "1", "python", "h", "gpp_main_kernel", "1", "7", "", "", "0", "10.0",
                         "Command line profiler metrics", name, unit, v])
    with open(path, "w", newline="") as fh:
        csv.writer(fh).writerows(rows)


def test_converter_units_and_records(tmp_path):
    _write_ncu_csv(tmp_path / "n.csv")
    (tmp_path / "l.jsonl").write_text('{"version": "v0", "kernel": "div"}\n{"version": "v8", "kernel": "rcp_sq"}\n')
    subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_to_rooflab.py"), str(tmp_path / "n.csv"),
                    str(tmp_path / "l.jsonl"), str(tmp_path / "out")], check=True, capture_output=True)
    recs = json.loads((tmp_path / "out.metrics.json").read_text())
    assert [r["label"] for r in recs] == ["v0", "v8"]
    assert recs[0]["runtime"] == pytest.approx(2.5e-3)
    assert recs[0]["counters"] == {"dadd": 10, "dmul": 20, "dfma": 30, "ddiv": 0, "dother": 0}
    assert recs[0]["bytes"] == {"l1": 4e6, "l2": 2e6, "hbm": 1e3}
    assert recs[1]["achieved_warps_per_sm"] == 16 and recs[1]["registers_per_thread"] == 128


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted (GPU box)")
def test_reference_reads_committed_b200_analysis_files():
    code = f"""
import sys; sys.path.insert(0, {str(REF)!r})
from rooflab.machine import load_machine
from rooflab.metrics import import_profiler_csv, load_metrics
from rooflab.roofline import trajectory
m = load_machine({str(ROOT / 'profiles' / 'b200.machine')!r})
csv_recs = import_profiler_csv({str(ROOT / 'profiles' / 'r01_b200_ladder.ncu.csv')!r})
recs = load_metrics({str(ROOT / 'profiles' / 'r01_b200_ladder.metrics.json')!r})
assert [r.label for r in csv_recs] == [r.label for r in recs] == ['v%d' % i for i in range(9)]
rep = trajectory(recs, m)
e = rep.sequences[0].entries
assert e[-1].fraction_of_peak < 1.0 and e[-1].runtime < e[0].runtime
print('ok', m.name, round(e[-1].fraction_of_peak, 3))
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         env={**os.environ, "PYTHONDONTWRITEBYTECODE": "1"})
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("ok")
