"""Sustained throughput: the production kernel back to back for ~60 s at the
paper size (nw 3), one line per ~5 s window with the time per evaluation,
the ncu-counted rate (executed FLOPs of one evaluation from
profiles/ncu_summary.json) and the analytic (effective) rate, and the SM
clock / power / throttle reasons nvidia-smi reports meanwhile."""
import json
import subprocess
import sys
import time

sys.path.insert(0, ".")
from paper_2008_11326_b200 import GPPContext, synth_problem
from paper_2008_11326_b200.counters import algorithmic_flops

p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
ctx = GPPContext(0)
ctx.upload(p)
_, (n, f), _ = ctx.run("rcp_sq")
fl = algorithmic_flops(512, 66, 32768, 3, n, f)
ex = json.load(open("profiles/ncu_summary.json"))["workloads"]["paper/nw3/seed1/rcp_sq/shards1"]["executed_flops_all"]
Q = "clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,temperature.gpu"
t_end = time.time() + float(sys.argv[1] if len(sys.argv) > 1 else 60)
while time.time() < t_end:
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={Q}", "--format=csv,noheader", "-lms", "500"],
                           stdout=subprocess.PIPE, text=True)
    tot, _ = ctx.time("rcp_sq", 1200)  # ~5 s
    smi.terminate()
    rows = [r.split(", ") for r in smi.communicate()[0].strip().splitlines() if r]
    clk = sorted(int(r[0].split()[0]) for r in rows) if rows else [0]
    pw = max(float(r[1].split()[0]) for r in rows) if rows else 0.0
    reasons = sorted({k for r in rows for k, v in zip(("sw_power_cap", "hw_slowdown", "sw_thermal", "temp"), r[2:]) if v.strip() == "Active"})
    temp = max(int(r[5]) for r in rows) if rows else 0
    print(f"{tot / 1200:.4f} ms/eval  {ex / (tot / 1200 * 1e-3) / 1e12:.2f} TFLOP/s ncu-counted  "
          f"{fl / (tot / 1200 * 1e-3) / 1e12:.2f} effective  sm {clk[len(clk) // 2]} MHz  "
          f"power<= {pw:.0f} W  temp<= {temp} C  reasons {reasons or '-'}", flush=True)
