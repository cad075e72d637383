"""Summarise an `ncu --set full` capture of the main GPP kernel into profiles/.

usage: python tools/ncu_summarize.py <report.ncu-rep> <out-stem> [--json profiles/ncu_summary.json]
       [--algorithmic-flops F]

Writes <out-stem>.txt (speed-of-light, pipes, scheduler, stall reasons,
memory traffic, FP64 instruction mix, top stalled SASS) and, with --json,
the per-launch numbers bench.py reports next to its live measurement:
dram bytes, ncu-counted FP64 FLOPs (2*dfma + dmul + dadd, the reference's
metric names rooflab/metrics.py:229-238) and the executed FMA ratio.
"""
import argparse
import csv
import io
import json
import subprocess
from pathlib import Path


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, check=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("stem")
    ap.add_argument("--json")
    ap.add_argument("--algorithmic-flops", type=float)
    ap.add_argument("--note", default="")
    ap.add_argument("--workload", default="512,66,32768,3,1",
                    help="nbands,ngpown,ncouls,nw,seed of the capture (tools/profile_run.py defaults)")
    a = ap.parse_args()

    raw = list(csv.reader(io.StringIO(ncu(a.report, "--page", "raw", "--csv"))))
    h, u, v = raw[0], raw[1], raw[2]
    d = {k: (vv, uu) for k, uu, vv in zip(h, u, v)}

    def num(k):
        try:
            return float(d[k][0].replace(",", ""))
        except (KeyError, ValueError):
            return None

    keys = [
        "Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    ]
    lines = [f"ncu --set full --clock-control none summary of {Path(a.report).name}", a.note, ""]
    for k in keys:
        if k in d:
            lines.append(f"{k:70s} {d[k][0]} {d[k][1]}")
    lines.append("")
    lines.append("warp stall reasons (cycles per issued instruction):")
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            val = num(k)
            if val and val > 0.005:
                lines.append(f"  {k.split('stalled_')[1].split('_per_issue')[0]:28s} {val:.3f}")

    dfma = num("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum") or 0
    dmul = num("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum") or 0
    dadd = num("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum") or 0
    flops = 2 * dfma + dmul + dadd
    dur_ms = num("gpu__time_duration.sum")
    unit = d.get("gpu__time_duration.sum", ("", "ms"))[1]
    dur_s = dur_ms * (1e-3 if unit == "ms" else 1e-6 if unit == "us" else 1e-9)
    rd = num("dram__bytes_read.sum")
    wr = num("dram__bytes_write.sum")
    rd_unit = d.get("dram__bytes_read.sum", ("", "byte"))[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(rd_unit, 1)
    wr_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d.get("dram__bytes_write.sum", ("", "byte"))[1], 1)
    traffic = (rd or 0) * scale + (wr or 0) * wr_scale
    fma_ratio = dfma / (dfma + dmul + dadd) if dfma else None
    lines.append("")
    lines.append(f"ncu-counted FP64 FLOPs per launch (2*dfma+dmul+dadd): {flops:.6e}")
    lines.append(f"executed FMA ratio dfma/(dfma+dmul+dadd): {fma_ratio:.4f}" if fma_ratio else "")
    lines.append(f"ncu-counted FP64 rate: {flops / dur_s / 1e12:.2f} TFLOP/s over {dur_ms} {unit}")
    if a.algorithmic_flops:
        lines.append(f"algorithmic FLOPs (reference analytic model): {a.algorithmic_flops:.6e} -> "
                     f"{a.algorithmic_flops / dur_s / 1e12:.2f} TFLOP/s; executed/algorithmic = "
                     f"{flops / a.algorithmic_flops:.3f}")
    lines.append(f"DRAM traffic per launch: {traffic / 1e6:.1f} MB")

    src = list(csv.reader(io.StringIO(ncu(a.report, "--page", "source", "--csv", "--print-source", "sass"))))
    hh = src[1]
    rows = [dict(zip(hh, r)) for r in src[2:]]
    rows.sort(key=lambda r: -float(r.get("Warp Stall Sampling (Not-issued Samples)") or 0))
    lines.append("")
    lines.append("top stalled SASS (not-issued samples, top reasons):")
    for r in rows[:15]:
        reasons = sorted(((float(r[c] or 0), c.split(" ")[0]) for c in hh
                          if c.startswith("stall") and c.endswith("(Not Issued)")), reverse=True)[:2]
        lines.append(f"  {r['Warp Stall Sampling (Not-issued Samples)']:>7} {r['Source'][:64]:64s} "
                     + ", ".join(f"{n}={int(x)}" for x, n in reasons))
    Path(a.stem + ".txt").write_text("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))
    if a.json:
        summary = {
            "source": f"{Path(a.report).name} (ncu --set full --clock-control none)",
            "kernel": d.get("Kernel Name", ("", ""))[0],
            "duration_ms_under_ncu": dur_s * 1e3,
            "dram_bytes_per_launch": traffic,
            "executed_flops_per_launch": flops,
            "fma_ratio": fma_ratio,
            "executed_over_algorithmic": (flops / a.algorithmic_flops) if a.algorithmic_flops else None,
            "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        }
        nb, ng, nc, nw, seed = (int(x) for x in a.workload.split(","))
        summary["workload"] = {"dims": [nb, ng, nc], "nw": nw, "seed": seed, "variant": "rcp_sq"}
        Path(a.json).write_text(json.dumps(summary, indent=1) + "\n")


if __name__ == "__main__":
    main()
