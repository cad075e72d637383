"""Write profiles/ncu_summary.json: ncu-counted FP64 FLOPs (2*dfma + dmul +
dadd), DRAM bytes and FP64-pipe activity of one evaluation of each bench
workload by THIS build, stamped with the build's device-code hash.

bench.py measures these live in every run (a child process under ncu after
the timed region); this file is the fallback it uses only when the hash
matches, and the numerator of the CPU reference arm (same FLOPs per step as
the GPU line, so the driver's ratio is a time ratio).  Run on a GPU box:

    python tools/ncu_commit.py [--shards 1 2 4 8] [--nw 3 2]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shards", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--nw", type=int, nargs="+", default=[3, 2])
ap.add_argument("--workload", default="paper")
a = ap.parse_args()

out = {"source": "tools/ncu_commit.py: ncu --metrics (FP64 op counts, DRAM bytes, FP64 pipe) "
                 "--clock-control none, one evaluation per band shard",
       "lib_sha256": bench.lib_sha256(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
       "workloads": {}}
for nw in a.nw:
    for shards in a.shards:
        args = argparse.Namespace(workload=a.workload, nw=nw, seed=1, variant="rcp_sq", gpus=shards)
        cap = bench.ncu_capture(args)
        if not cap or "error" in cap:
            print("failed", nw, shards, cap, flush=True)
            continue
        key = f"{a.workload}/nw{nw}/seed1/rcp_sq/shards{shards}"
        out["workloads"][key] = {k: v for k, v in cap.items() if k not in ("source", "lib_sha256")}
        print(key, json.dumps(out["workloads"][key]), flush=True)
(ROOT / "profiles" / "ncu_summary.json").write_text(json.dumps(out, indent=1) + "\n")
