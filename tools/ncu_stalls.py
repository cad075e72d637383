"""Summarise an ncu report: key SOL/scheduler metrics, stall reasons, top stalled SASS.

usage: python tools/ncu_stalls.py <report.ncu-rep> [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "dram__bytes_read.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
for k, uu, vv in zip(h, u, v):
    if k in want or (k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")):
        try:
            if float(vv.replace(",", "")) == 0:
                continue
        except ValueError:
            pass
        print(f"{k:90s} {vv} {uu}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hh = src[1]
rows = [dict(zip(hh, r)) for r in src[2:]]
agg = collections.Counter()
for d in rows:
    for c in hh:
        if c.startswith("stall") and c.endswith("(Not Issued)"):
            agg[c] += float(d[c] or 0)
print("not-issued stall samples:", ", ".join(f"{k.split(' ')[0]}={int(n)}" for k, n in agg.most_common(8)))
rows.sort(key=lambda d: -float(d["Warp Stall Sampling (Not-issued Samples)"] or 0))
for d in rows[:top]:
    reasons = sorted(((float(d[c] or 0), c.split(" ")[0]) for c in hh if c.startswith("stall") and c.endswith("(Not Issued)")), reverse=True)[:2]
    print(f"  {d['Address'][-5:]} {d['Warp Stall Sampling (Not-issued Samples)']:>7} {d['Source'][:60]:60s} {reasons}")
