"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of a
bench.py command: per-kernel launch counts and times, and each kernel's share
of the timed step (all launches except the untimed counting launch, the FP64
peak microbenchmark and the e2e/synthesis helpers).

usage: python tools/launch_summary.py <launches.csv> "<command that was profiled>"
"""
import csv
import sys
from collections import OrderedDict


def main():
    path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = OrderedDict()
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        v = float(r[iv].replace(",", ""))
        v = v / 1e6 if r[iu] in ("ns", "nsecond") else (v / 1e3 if r[iu] in ("us", "usecond") else v)
        per.setdefault(r[ik], []).append(v)
    print("ncu --metrics gpu__time_duration.sum --clock-control none launch list of:")
    print(f"  {cmd}")
    print("per-launch times are cold-cache and serialised: compare SHARES, not absolutes.\n")
    for k, v in per.items():
        print(f"{len(v):5d} launches {sum(v):10.3f} ms total {sum(v)/len(v):10.4f} ms/launch  {k[:110]}")
    step = {k: sum(v) for k, v in per.items()
            if ("sacc" in k and ", 0>" in k) or "finalize" in k}
    tot = sum(step.values())
    print()
    for k, v in step.items():
        print(f"share of the timed step: {100 * v / tot:6.1f}%  {k[:80]}")


if __name__ == "__main__":
    main()
