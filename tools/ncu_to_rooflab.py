"""ncu counters -> the reference's analysis formats.

Input: the CSV that `ncu --metrics ... --csv --log-file F` writes (one row per
(launch, metric)), plus the launch labels in launch order (e.g. the JSON lines
tools/ladder.py --ncu prints).  Output:

  <stem>.ncu.csv       columns of rooflab.metrics.DEFAULT_PROFILER_MAPPING
                       (metrics.py:229-238), runtime in seconds, so
                       rooflab.metrics.import_profiler_csv(path) reads it as is;
  <stem>.metrics.json  rooflab KernelMetrics records (metrics.py:110-217), the
                       input of `rooflab analyze` / roofline.trajectory.

Pure stdlib: the reference itself is not needed to write these files.
"""
import argparse
import csv
import json
from collections import OrderedDict

METRICS = {
    "runtime": "gpu__time_duration.sum",
    "dadd": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "dmul": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "dfma": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "l1": "l1tex__t_bytes.sum",
    "l2": "lts__t_bytes.sum",
    "hbm": "dram__bytes.sum",
    "regs": "launch__registers_per_thread",
    "tpb": "launch__block_size",
    "warps": "sm__warps_active.avg.per_cycle_active",
}
UNIT = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    launches = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        rec = launches.setdefault(d["ID"], {"kernel": d["Kernel Name"]})
        val = float(d["Metric Value"].replace(",", ""))
        rec[d["Metric Name"]] = val * UNIT.get(d["Metric Unit"], 1.0)
    return list(launches.values())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("ncu_csv")
    ap.add_argument("labels", help="JSON lines with a 'version' key, one per launch, in order")
    ap.add_argument("stem")
    ap.add_argument("--system", default="B200")
    a = ap.parse_args()
    labels = [json.loads(l) for l in open(a.labels) if l.strip().startswith("{")]
    labels = [l for l in labels if "version" in l]
    launches = read_launches(a.ncu_csv)
    if len(launches) != len(labels):
        raise SystemExit(f"{len(launches)} launches but {len(labels)} labels")
    cols = ["Kernel Name"] + [METRICS[k] for k in ("runtime", "dadd", "dmul", "dfma", "l1", "l2", "hbm")]
    with open(a.stem + ".ncu.csv", "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(cols + ["kernel"])
        for lab, rec in zip(labels, launches):
            w.writerow([lab["version"]] + [rec.get(c, 0.0) for c in cols[1:]] + [lab.get("kernel", "")])
    records = []
    for lab, rec in zip(labels, launches):
        records.append({
            "label": lab["version"],
            "runtime": rec[METRICS["runtime"]],
            "counters": {"dadd": int(rec[METRICS["dadd"]]), "dmul": int(rec[METRICS["dmul"]]),
                         "dfma": int(rec[METRICS["dfma"]]), "ddiv": 0, "dother": 0},
            "bytes": {"l1": rec[METRICS["l1"]], "l2": rec[METRICS["l2"]], "hbm": rec[METRICS["hbm"]]},
            "system": a.system,
            "registers_per_thread": int(rec[METRICS["regs"]]),
            "threads_per_block": int(rec[METRICS["tpb"]]),
            "achieved_warps_per_sm": int(round(rec[METRICS["warps"]])),
        })
    json.dump(records, open(a.stem + ".metrics.json", "w"), indent=2)
    print(f"wrote {a.stem}.ncu.csv and {a.stem}.metrics.json ({len(records)} records)")


if __name__ == "__main__":
    main()
