#!/usr/bin/env python
"""GPP self-energy bench on B200: one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (BASELINE.json configs[1]): the paper size (nbands, ngpown, ncouls) =
(512, 66, 32768) with 3 frequencies, synth_problem seed 1 (3.5 % far-branch
instances; seed 42 never takes the far branch).  At N GPUs the
band (n1) loop is sharded (strong scaling, BASELINE configs[2]) and the
partials are combined by one NCCL allreduce inside the library -- one
process per GPU under torchrun, or, without torchrun, one process driving N
devices (gpp_comm_init_all + gpp_time_group).

A step = one full evaluation of the reduction (production kernel + slot
finalize (+ allreduce)), inputs resident in HBM (338 MB > the 126 MB L2, so
every step streams them from HBM; no flush needed).

Metric (BASELINE.json): "GPP FP64 TFLOP/s (ncu-counted)".  `value` = FP64
FLOPs the kernels EXECUTE per step (2*dfma + dmul + dadd, ncu's
smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum -- the
reference's profiler column names, rooflab/metrics.py:228-237), counted by
a live ncu capture of this build in a child process after the timed region,
summed over all GPUs' shards, / device time (CUDA events, max over ranks).
The reference's analytic count (rooflab/gpp/kernel.py:191-212) / the same
time is `effective_tflops` beside it: the kernel executes ~65 % of those
FLOPs (per-instance algebra), so that rate is not a roofline
figure.  `e2e` = the same numerator per step through the
public API (evaluate_variant on pageable numpy arrays: H2D of every input,
the evaluation and the D2H of the result).  The reference arm uses the same
numerator, so the driver's ratio of the two lines is a pure time ratio.
"""

from __future__ import annotations

import argparse
import csv
import hashlib
import io
import json
import os
import platform
import statistics
import struct
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GPP FP64 TFLOP/s (ncu-counted) per B200 & % of FP64 peak; 1/2/4/8-GPU time"
WORKLOADS = {
    "paper": (512, 66, 32768),
    "tiny": (32, 8, 512),
    "weak": (4096, 528, 65536),
}
LIB = ROOT / "paper_2008_11326_b200" / "lib" / "libgpp_b200.so"
NCU_SUMMARY = ROOT / "profiles" / "ncu_summary.json"
NCU_METRICS = (
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__time_duration.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_bytes.sum",
    "lts__t_bytes.sum",
    "dram__bytes.sum",
)
# The reference's profiler-CSV columns (rooflab/metrics.py:228-237,
# DEFAULT_PROFILER_MAPPING): the live capture is also written in that form.
ROOFLAB_COLUMNS = {
    "label": "Kernel Name", "runtime": "gpu__time_duration.sum",
    "dadd": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "dmul": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "dfma": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "l1": "l1tex__t_bytes.sum", "l2": "lts__t_bytes.sum", "hbm": "dram__bytes.sum",
}


def rooflab_csv(record: dict, path: Path) -> None:
    """One evaluation's production-kernel counters as a CSV that the
    reference's import_profiler_csv reads with its default mapping
    (runtime in seconds: runtime_scale=1)."""
    cols = list(ROOFLAB_COLUMNS.values())
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(cols)
        c, b = record["counters"], record["bytes"]
        w.writerow([record["label"], record["runtime"], c["dadd"], c["dmul"], c["dfma"],
                    b["l1"], b["l2"], b["hbm"]])


def parse_args():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="paper")
    ap.add_argument("--dims", type=int, nargs=3, default=None, metavar=("NBANDS", "NGPOWN", "NCOULS"),
                    help="explicit (nbands, ngpown, ncouls) instead of --workload (sweep points)")
    ap.add_argument("--nw", type=int, default=3)
    ap.add_argument("--seed", type=int, default=None,
                    help="synth_problem seed (default: 1; 42 for the weak workload, whose "
                         "reference output tests/golden/gpp_big.json holds)")
    ap.add_argument("--variant", choices=("rcp_sq", "rcp", "div"), default="rcp_sq")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ncu", action="store_true", help="skip the live ncu capture")
    ap.add_argument("--ncu-child", action="store_true", help=argparse.SUPPRESS)
    a = ap.parse_args()
    if a.seed is None:
        a.seed = 42 if a.workload == "weak" else 1
    return a


def dims_of(args) -> tuple[int, int, int]:
    dims = getattr(args, "dims", None)
    return tuple(dims) if dims else WORKLOADS[args.workload]


def lib_sha256() -> str | None:
    """sha256 of the library's device code as SASS (`cuobjdump -sass`, minus
    the source-path lines): the sm_100a kernels ncu counts, the same for every
    build of the same sources.  (The .nv_fatbin bytes are no build
    fingerprint: -lineinfo's DWARF line table records the sources' mtimes.)
    Falls back to the .nv_fatbin section when cuobjdump is missing."""
    try:
        out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, timeout=120)
        if out.returncode == 0 and out.stdout:
            # drop the "identifier = <source path>" lines: the build directory
            body = b"\n".join(l for l in out.stdout.splitlines() if not l.startswith(b"identifier"))
            return "sass:" + hashlib.sha256(body).hexdigest()
    except (OSError, subprocess.TimeoutExpired):
        pass
    try:
        b = LIB.read_bytes()
        shoff, = struct.unpack_from("<Q", b, 0x28)
        shentsize, shnum, shstrndx = struct.unpack_from("<HHH", b, 0x3A)
        secs = [struct.unpack_from("<IIQQQQIIQQ", b, shoff + i * shentsize) for i in range(shnum)]
        stro = secs[shstrndx][4]
        for sec in secs:
            name = b[stro + sec[0]: b.index(b"\0", stro + sec[0])]
            if name == b".nv_fatbin":
                return "fatbin:" + hashlib.sha256(b[sec[4]: sec[4] + sec[5]]).hexdigest()
        return None
    except (OSError, struct.error, ValueError, IndexError):
        return None


_LIB_SHA = None


def lib_sha256_cached() -> str | None:
    global _LIB_SHA
    if _LIB_SHA is None:
        _LIB_SHA = lib_sha256()
    return _LIB_SHA


# ----------------------------------------------------------------------------
# distributed plumbing
# ----------------------------------------------------------------------------
class Dist:
    """torchrun (WORLD_SIZE set): one process per GPU over NCCL.  Otherwise
    one process; --gpus N > 1 then drives N local devices itself."""

    def __init__(self, gpus: int):
        self.torchrun = "WORLD_SIZE" in os.environ
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        if self.torchrun and self.world != gpus:
            raise SystemExit(f"--gpus {gpus} but WORLD_SIZE={self.world}")
        self.gpus = gpus
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist

            torch.cuda.set_device(self.local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local_rank))
            self.pg = dist

    @property
    def single_process_group(self) -> bool:
        return not self.torchrun and self.gpus > 1

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------------------
# clocks sampler: NVML every 5 ms during the timed region (nvidia-smi fallback)
# ----------------------------------------------------------------------------
def nvml_devices(n: int) -> list[int]:
    """NVML indices of the first n CUDA devices (CUDA_VISIBLE_DEVICES order
    when it lists plain indices)."""
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    ids = [x.strip() for x in cvd.split(",") if x.strip()]
    if ids and all(x.isdigit() for x in ids):
        return [int(x) for x in ids[:n]]
    return list(range(n))


class Clocks:
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, devices):
        self.devices = list(devices)
        self.rows = []
        self.stop_ev = threading.Event()
        self.thread = None
        self.err = None

    def start(self):
        if not self.devices:
            return
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handles = [pynvml.nvmlDeviceGetHandleByIndex(d) for d in self.devices]
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nvml
        while not self.stop_ev.is_set():
            for h in self.handles:
                try:
                    self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                      nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
                                      nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                      nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
                except Exception:  # noqa: BLE001
                    pass
            time.sleep(0.005)

    def stop(self) -> dict | None:
        if not self.devices:
            return None
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no samples"]}
        self.stop_ev.set()
        self.thread.join(timeout=2)
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for r in self.rows for k, bit in self.REASONS.items() if r[3] & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(r[1] for r in self.rows) if self.rows else None,
                "power_w_max": max(r[2] for r in self.rows) if self.rows else None,
                "samples": len(self.rows), "sampler": "nvml 5 ms", "reasons": reasons}


# ----------------------------------------------------------------------------
# host description (cpu_baseline)
# ----------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def host_info() -> dict:
    return {"cpu_model": cpu_model(), "cpu_count": os.cpu_count(), "blas_threads": blas_threads(),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS", "unset (all cores)")}


# ----------------------------------------------------------------------------
# the reference CPU path: the unmodified rooflab from baseline/_ref when it is
# there (kind "reference"), else the oracle restatement (kind "port")
# ----------------------------------------------------------------------------
class CpuReference:
    """Whole-problem evaluations of the reference's production CPU path,
    evaluate_variant(p, "rcp_sq") -- what rooflab's run_version(p, "v8")
    times (runner.py:258-260)."""

    def __init__(self, dims, seed, nw):
        ref = ROOT / "baseline" / "_ref"
        self.kind = "port"
        if (ref / "rooflab").is_dir():
            sys.path.insert(0, str(ref))
            try:
                import rooflab.gpp as rgpp
                import rooflab.gpp.kernel as rk
                import rooflab.gpp.problem as rp
                import rooflab.gpp.runner as rr

                # nw != 2: the reference's NW constant, imported by value into
                # three modules (SURVEY.md Table R) -- patched at run time,
                # the installed source is untouched.
                rp.NW = rk.NW = rr.NW = nw
                self.kind = "reference"
                self.mod = rgpp
                self.what = "rooflab (unmodified, baseline/_ref) evaluate_variant(p, 'rcp_sq')"
                self.p = rgpp.synth_problem(*dims, seed=seed)
            except Exception as e:  # noqa: BLE001 -- fall back to the port
                self.kind = "port"
                self.why = f"baseline/_ref import failed: {e}"
        if self.kind == "port":
            from oracle import gpp_oracle as orc
            from paper_2008_11326_b200 import synth_problem

            self.mod = orc
            self.what = "oracle/gpp_oracle.py evaluate_variant(p, 'rcp_sq') (restatement of kernel.py:98-114)"
            self.p = synth_problem(*dims, seed=seed, nw=nw, check=False)

    def evaluate(self):
        return self.mod.evaluate_variant(self.p, "rcp_sq")

    def time(self, steps: int, warmup: int) -> list[float]:
        for _ in range(warmup):
            self.evaluate()
        out = []
        for _ in range(steps):
            t0 = time.perf_counter()
            self.evaluate()
            out.append(time.perf_counter() - t0)
        return out

    def reference_result_seconds(self, dims, seed, nw) -> float | None:
        """The literal loop-nest oracle (problem.py:179-208) at a small size."""
        if self.kind != "reference":
            return None
        p = self.mod.synth_problem(*dims, seed=seed)
        t0 = time.perf_counter()
        self.mod.reference_result(p)
        return time.perf_counter() - t0


# ----------------------------------------------------------------------------
# executed FP64 FLOPs: live ncu capture of this build (child process)
# ----------------------------------------------------------------------------
def ncu_child(args):
    """Under ncu: every band shard of the workload once (device synthesis,
    the production kernel as the timed region runs it)."""
    from paper_2008_11326_b200 import GPPContext
    from paper_2008_11326_b200.dist import band_range

    nb, ng, nc = dims_of(args)
    ctx = GPPContext(0)
    for r in range(args.gpus):
        ctx.synth(nb, ng, nc, seed=args.seed, nw=args.nw, band_range=band_range(nb, args.gpus, r))
        ctx.run(args.variant, counts=False)
        print(f"shard {r}", flush=True)
    ctx.close()


def ncu_capture(args, timeout_s: float = 420.0) -> dict | None:
    """Run ncu on the child; per shard: executed FP64 FLOPs, DRAM bytes,
    FP64-pipe activity of the production kernel launches."""
    out = Path(os.environ.get("GPP_NCU_DIR", "/tmp")) / f"gpp_ncu_{os.getpid()}.csv"
    cmd = ["ncu", "--metrics", ",".join(NCU_METRICS), "--clock-control", "none",
           "-k", "regex:gpp_sacc_kernel|gpp_slot_finalize|gpp_main_kernel|gpp_finalize",
           "--page", "raw", "--csv", "--print-units", "base", "--log-file", str(out),
           sys.executable, str(ROOT / "bench.py"), "--ncu-child", "--workload", args.workload,
           "--nw", str(args.nw), "--seed", str(args.seed), "--variant", args.variant,
           "--gpus", str(args.gpus), "--dims", *map(str, dims_of(args))]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = env.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0]
    t0 = time.perf_counter()
    try:
        proc = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s, env=env)
    except (OSError, subprocess.TimeoutExpired) as e:
        return {"error": f"ncu failed: {e}"}
    if proc.returncode != 0 or not out.exists():
        return {"error": f"ncu rc={proc.returncode}: {(proc.stderr or proc.stdout)[-300:]}"}
    text = out.read_text()
    if not os.environ.get("GPP_NCU_KEEP"):
        out.unlink(missing_ok=True)
    # The log also holds ncu's own "==PROF==" lines: the table starts at the
    # header row ("ID", ...), then one row of units, then one row per launch.
    rows = [r for r in csv.reader(io.StringIO(text)) if r]
    start = next((i for i, r in enumerate(rows) if r[0] == "ID"), None)
    if start is None:
        return {"error": f"ncu produced no table: {text[-300:]}"}
    hdr = rows[start]
    data = [r for r in rows[start + 2:] if len(r) == len(hdr) and r[0].isdigit()]
    col = {k: i for i, k in enumerate(hdr)}

    def val(r, k):
        try:
            return float(r[col[k]].replace(",", ""))
        except (KeyError, ValueError):
            return 0.0

    main, fin = [], []
    for r in data:
        (main if "gpp_sacc_kernel" in r[col["Kernel Name"]] or "gpp_main_kernel" in r[col["Kernel Name"]]
         else fin).append(r)
    fl = lambda r: 2 * val(r, NCU_METRICS[0]) + val(r, NCU_METRICS[1]) + val(r, NCU_METRICS[2])  # noqa: E731
    dfma = sum(val(r, NCU_METRICS[0]) for r in main)
    dmul = sum(val(r, NCU_METRICS[1]) for r in main)
    dadd = sum(val(r, NCU_METRICS[2]) for r in main)
    dur = sum(val(r, "gpu__time_duration.sum") for r in main)
    pipe = (sum(val(r, NCU_METRICS[6]) * val(r, "gpu__time_duration.sum") for r in main) / dur) if dur else None
    # KernelMetrics-shaped record (rooflab/metrics.py:110-217) of the whole
    # evaluation's production-kernel launches, in the reference's units.
    record = {
        "label": f"gpp_sacc_kernel {dims_of(args)} nw{args.nw} x{args.gpus} shards",
        "runtime": dur * 1e-9,
        "counters": {"dadd": int(dadd), "dmul": int(dmul), "dfma": int(dfma), "ddiv": 0, "dother": 0},
        "bytes": {k: sum(val(r, ROOFLAB_COLUMNS[k]) for r in main) for k in ("l1", "l2", "hbm")},
        "system": "B200",
    }
    if os.environ.get("GPP_ROOFLAB_CSV"):
        rooflab_csv(record, Path(os.environ["GPP_ROOFLAB_CSV"]))
    return {
        "rooflab_record": record,
        "source": f"live ncu capture of this build in this run ({len(main)} production-kernel + "
                  f"{len(fin)} finalize launches, --clock-control none, {time.perf_counter() - t0:.0f} s)",
        "lib_sha256": lib_sha256_cached(),
        "executed_flops_main": sum(fl(r) for r in main),
        "executed_flops_all": sum(fl(r) for r in data),
        "per_shard_main_flops": None,
        "dram_bytes_main": sum(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum") for r in main),
        "fma_ratio": dfma / (dfma + dmul + dadd) if dfma + dmul + dadd else None,
        "fp64_pipe_pct": pipe,
        "ncu_duration_ms_main": dur * 1e-6,
        "shards": args.gpus,
    }


def committed_capture(args) -> dict | None:
    """profiles/ncu_summary.json, only if it was taken of this exact build."""
    try:
        s = json.loads(NCU_SUMMARY.read_text())
    except (OSError, json.JSONDecodeError):
        return None
    if s.get("lib_sha256") != lib_sha256_cached():
        return None
    key = f"{args.workload}/nw{args.nw}/seed{args.seed}/{args.variant}/shards{args.gpus}"
    w = s.get("workloads", {}).get(key)
    if not w:
        return None
    return {**w, "source": f"profiles/ncu_summary.json ({s.get('source', '')}; lib sha256 matches this build)"}


# ----------------------------------------------------------------------------
def golden_parity(result, workload, seed, nw):
    g = ROOT / "tests" / "golden" / "gpp_big.json"
    if not g.exists():
        return None
    dims = list(WORKLOADS[workload])
    for c in json.loads(g.read_text())["cases"]:
        if c["dims"] == dims and c["seed"] == seed and c["nw"] == nw:
            from paper_2008_11326_b200.problem import GPPResult, max_rel_error

            src = c.get("reference_result") or c["evaluate_variant"]["rcp_sq"]
            want = GPPResult(np.array([complex(*z) for z in src["achtemp"]]),
                             np.array([complex(*z) for z in src["asxtemp"]]))
            return {"max_rel_err_vs_reference": max_rel_error(result, want),
                    "branch_stats_reference": c["branch_stats"]["rcp_sq"]}
    return None


def _config(args, dims):
    return {
        "workload": f"{args.workload} (nbands, ngpown, ncouls) = {dims}, nw={args.nw}",
        "nbands": dims[0], "ngpown": dims[1], "ncouls": dims[2], "nw": args.nw, "seed": args.seed,
        "variant": args.variant,
        "parallelism": f"band-shard x{args.gpus}" + (" + NCCL allreduce" if args.gpus > 1 else ""),
        "l2": "inputs (footprint > 126 MB L2) stream from HBM each step; no flush",
    }


def reference_numerator(args) -> tuple[float | None, str]:
    """The executed-FLOP numerator of this workload for the reference arm:
    the committed capture of this build (the GPU arm measures it live)."""
    try:
        s = json.loads(NCU_SUMMARY.read_text())
        w = s["workloads"][f"{args.workload}/nw{args.nw}/seed{args.seed}/{args.variant}/shards1"]
        return float(w["executed_flops_all"]), "profiles/ncu_summary.json (ncu-counted FLOPs of one evaluation by this build)"
    except (OSError, KeyError, ValueError, json.JSONDecodeError):
        return None, "no committed capture"


def run_reference(args, dist: Dist):
    """--impl reference: the reference's CPU path on this host (rank 0 only)."""
    if dist.rank != 0:
        return
    from paper_2008_11326_b200.counters import algorithmic_flops

    dims = WORKLOADS[args.workload]
    ref = CpuReference(dims, args.seed, args.nw)
    secs = ref.time(args.steps, args.warmup)
    t = statistics.mean(secs)
    from oracle import gpp_oracle as orc
    from paper_2008_11326_b200 import synth_problem

    _, near, far = orc.branch_stats(synth_problem(*dims, seed=args.seed, nw=args.nw, check=False), "rcp_sq")
    alg = algorithmic_flops(*dims, args.nw, near, far)
    num, num_src = reference_numerator(args)
    value = (num if num else alg) / t / 1e12
    sample = (f"each step = one whole evaluation of the {dims} nw={args.nw} workload through "
              f"{ref.what}; mean of {args.steps} after {args.warmup} warm-up")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": f"synthetic (synth_problem seed {args.seed})",
        "config": _config(args, dims),
        "numerator": {"flops_per_step": num or alg,
                      "what": ("ncu-counted FP64 FLOPs of the B200 kernels for one evaluation (" + num_src
                               + "), the same numerator as the GPU line: the ratio is a time ratio")
                      if num else "reference analytic FLOPs (no committed ncu capture)"},
        "effective_tflops": alg / t / 1e12,
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": blas_threads(), "kind": ref.kind,
                         "sample": sample, **host_info(),
                         **({"fallback_reason": ref.why} if hasattr(ref, "why") else {})},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
def run_ours(args, dist: Dist):
    from paper_2008_11326_b200 import fp64_peak, synth_problem
    from paper_2008_11326_b200._lib import load
    from paper_2008_11326_b200.counters import BranchStats, algorithmic_flops, counters_from_stats, fma_ratio
    from paper_2008_11326_b200.dist import MultiDeviceGPP, ShardedGPP, band_range

    dims = dims_of(args)
    nb, ng, nc = dims
    device = dist.local_rank
    load()
    # FP64 roofline denominator: measured live on this device (MEASURED_PEAKS.json has no FP64).
    fp64_peak(device, 20_000)
    peak_tf, _ = fp64_peak(device, 300_000)

    # ---- the problem, resident on the device(s) ---------------------------
    group = None
    if dist.single_process_group:
        group = MultiDeviceGPP(list(range(args.gpus)))
        group.synth(nb, ng, nc, seed=args.seed, nw=args.nw)
        result, (near, far), _ = group.run(args.variant, counts=True)
        ctx = group.ctxs[0]
        n_ranks = args.gpus
    else:
        shard = ShardedGPP.from_torch(device) if dist.world > 1 else ShardedGPP(device, 0, 1, None)
        ctx = shard.ctx
        ctx.synth(nb, ng, nc, seed=args.seed, nw=args.nw, band_range=shard.band_range(nb))
        result, (near, far), _ = ctx.run(args.variant)  # combined over ranks
        n_ranks = dist.world
    info = ctx.kernel_info(args.variant)
    alg_job = algorithmic_flops(nb, ng, nc, args.nw, near, far)

    def timed(iters):
        return group.time(args.variant, iters) if group else ctx.time(args.variant, iters)

    def launches():
        return sum(c.launch_count() for c in group.ctxs) if group else ctx.launch_count()

    # ---- device-resident timed region --------------------------------------
    timed(args.warmup)
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    for attempt in range(2):  # a run that saw a slowdown reason is re-measured once
        dist.barrier()
        clocks = Clocks(nvml_devices(args.gpus) if dist.rank == 0 else [])
        clocks.start()
        l0 = launches()
        total_ms, main_ms = timed(args.steps)
        gpu_launches = launches() - l0
        dist.barrier()
        clk = clocks.stop()
        retry = 1.0 if (clk and bad & set(clk.get("reasons", []))) else 0.0
        if attempt == 0 and dist.max(retry) > 0:
            continue
        if clk is not None:
            clk["remeasured"] = attempt > 0
        break
    gpu_launches = int(dist.sum(gpu_launches))
    t_step_ms = dist.max(total_ms) / args.steps
    t_main_ms = dist.max(main_ms) / args.steps

    # ---- end to end through the public API ---------------------------------
    e2e = e2e_pinned = None
    p = None
    if not args.no_e2e and args.workload != "weak":
        from paper_2008_11326_b200 import GPPProblem, evaluate_variant

        p = synth_problem(nb, ng, nc, seed=args.seed, nw=args.nw, check=False)
        # Writeable arrays: the public API re-uploads them on every call (a
        # fresh problem each step, as a user's own numpy arrays would be).
        q = GPPProblem(nb, ng, nc, p.wtilde.copy(order="F"), p.i_eps.copy(order="F"),
                       p.aqsntemp.copy(order="F"), p.aqsmtemp.copy(order="F"), p.wx.copy())
        if group:
            call = lambda: group.evaluate(q, args.variant)  # noqa: E731
            api = "MultiDeviceGPP.evaluate -> gpp_evaluate_host per device (one thread each)"
        elif dist.world > 1:
            call = lambda: shard.evaluate(q, args.variant)  # noqa: E731
            api = "ShardedGPP.evaluate -> gpp_evaluate_host (this rank's shard + NCCL)"
        else:
            call = lambda: evaluate_variant(q, args.variant, device=device)  # noqa: E731
            api = "evaluate_variant (the drop-in seam) -> gpp_evaluate_host"
        r_b0, r_b1 = (band_range(nb, n_ranks, dist.rank) if n_ranks > 1 else (0, nb))

        def h2d_rank(r):
            b0, b1 = band_range(nb, n_ranks, r)
            we = 2 * 16 * nc * ng // (n_ranks if n_ranks > 1 else 1)
            return we + 16 * nc * (b1 - b0) + 16 * ng * (b1 - b0) + 8 * args.nw * (b1 - b0)

        h2d = sum(h2d_rank(r) for r in range(n_ranks))
        d2h = (8 * 4 * args.nw) * n_ranks

        def time_e2e(reps=3):
            # The first passes over fresh host arrays are slower (first use of
            # the staging ring and of the pages): e2e gets its own warm-up,
            # then `reps` timed rounds of e2e_steps calls; the median round
            # is reported (host-side memory effects vary between rounds).
            for _ in range(max(args.warmup, 10)):
                call()
            rounds = []
            for _ in range(reps):
                dist.barrier()
                t0 = time.perf_counter()
                for _ in range(args.e2e_steps):
                    call()
                el = time.perf_counter() - t0
                dist.barrier()
                rounds.append(dist.max(el) / args.e2e_steps)
            return statistics.median(rounds), rounds

        el, rounds = time_e2e()
        e2e = {"value": None, "unit": "TFLOP/s", "ms_per_step": el * 1e3, "steps": args.e2e_steps,
               "rounds_ms": [round(x * 1e3, 4) for x in rounds],
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "inputs": "pageable numpy arrays (the library packs them into its pinned staging ring)",
               "path": api}
        if not group and dist.world == 1:
            from paper_2008_11326_b200._lib import check

            lib = load()
            arrays = [q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp]
            for a in arrays:
                check(lib.gpp_host_register(a.ctypes.data, a.nbytes), "gpp_host_register")
            try:
                elp, rounds_p = time_e2e()
            finally:
                for a in arrays:
                    lib.gpp_host_unregister(a.ctypes.data)
            e2e_pinned = {"ms_per_step": elp * 1e3, "rounds_ms": [round(x * 1e3, 4) for x in rounds_p],
                          "inputs": "the same arrays page-locked (gpp_host_register)"}

    # Time to solution of the reference's own factored algorithm on the device
    # (gpp_run_factored) -- a different algorithm, never the roofline.
    factored = None
    if n_ranks == 1:
        ctx.run_factored(args.variant, counts=False)
        fms = [ctx.run_factored(args.variant, counts=False)[2] for _ in range(5)]
        fres = ctx.run_factored(args.variant, counts=False)[0]
        factored = {"ms": statistics.median(fms),
                    "what": "gpp_run_factored: the reference's factored algorithm (kernel.py:98-114) -- "
                            "band weights W = aqsntemp conj(aqsmtemp)^T on the FP64 tensor cores (DMMA) fused "
                            "with the branch terms in one repo kernel; a different algorithm, not a roofline figure"}
        gp = golden_parity(fres, args.workload, args.seed, args.nw) if args.variant == "rcp_sq" else None
        if gp:
            factored["max_rel_err_vs_reference"] = gp["max_rel_err_vs_reference"]

    # ---- executed FLOPs: live ncu capture (rank 0), after every timing ------
    cap = None
    if dist.rank == 0:
        cap = None if args.no_ncu else ncu_capture(args)
        if not cap or "error" in cap:
            err = cap.get("error") if cap else "skipped (--no-ncu)"
            cap = committed_capture(args) or {"error": err}
    dist.barrier()

    if dist.rank != 0:
        (group.close() if group else ctx.close())
        return

    # ---- CPU baseline (rank 0, N=1 only) -----------------------------------
    cpu = None
    if n_ranks == 1 and not args.no_cpu_baseline and args.workload != "weak":
        ref = CpuReference(dims, args.seed, args.nw)
        secs = ref.time(steps=4, warmup=1)
        t_cpu = statistics.mean(secs)
        num = (cap or {}).get("executed_flops_all") or alg_job
        cpu = {"value": num / t_cpu / 1e12, "unit": "TFLOP/s", "cores": blas_threads(), "kind": ref.kind,
               "sample": f"4 whole evaluations (after 1 warm-up) of the {dims} nw={args.nw} workload through "
                         f"{ref.what}, {sum(secs):.1f} s; numerator = this line's executed-FLOP count",
               "ms_per_evaluation": t_cpu * 1e3, "effective_tflops": alg_job / t_cpu / 1e12,
               **host_info()}
        rr = ref.reference_result_seconds(WORKLOADS["tiny"], 42, 2)
        if rr is not None:
            cpu["reference_result_tiny_s"] = rr
        cpu["reference_result_paper_s"] = "see profiles/r02_cpu_reference_result.json (~90 s, run once)"

    # ---- assemble -----------------------------------------------------------
    exec_job = (cap or {}).get("executed_flops_all")
    exec_main = (cap or {}).get("executed_flops_main")
    value = exec_job / (t_step_ms * 1e-3) / 1e12 if exec_job else None
    tot_inst = args.nw * nb * ng * nc
    per_gpu_main = exec_main / n_ranks if exec_main else None
    achieved = per_gpu_main / (t_main_ms * 1e-3) / 1e12 if per_gpu_main else None
    cnt = counters_from_stats("rcp_sq", BranchStats(tot_inst, near, far), nb * ng * nc, True)
    r_exec = (cap or {}).get("fma_ratio")
    line = {
        "metric": METRIC,
        "value": value if value is not None else alg_job / (t_step_ms * 1e-3) / 1e12,
        "unit": "TFLOP/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_step_ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": f"synthetic (synth_problem seed {args.seed}, PCG64 as the reference draws it; drawn on "
                f"the device by gpp_synth for the timed region)",
        "config": _config(args, dims),
        "value_kind": ("ncu-counted: executed FP64 FLOPs per step (2*dfma + dmul + dadd, all GPUs) / step time"
                       if value is not None else
                       "EFFECTIVE (no ncu count available: " + str((cap or {}).get("error")) + ")"),
        "effective_tflops": alg_job / (t_step_ms * 1e-3) / 1e12,
        "effective_kind": "the reference's analytic FLOPs (kernel.py:191-212) / step time; the kernels execute "
                          f"{100.0 * exec_job / alg_job:.0f}% of them" if exec_job else "analytic / step time",
        "pct_fp64_peak": 100.0 * achieved / peak_tf if achieved else None,
        "roofline": {
            "bound": "fp64",
            "bound_note": ("the contract's enum is hbm|tensor; this path is bound by the FP64 vector pipe "
                           "(DFMA): no dense contraction for tensor cores (north star), DRAM at ~1.4 % of peak"),
            "achieved": achieved,
            "peak": peak_tf,
            "unit": "TFLOP/s",
            "frac": achieved / peak_tf if achieved else None,
            "traffic": ((cap or {}).get("dram_bytes_main") / n_ranks) if (cap or {}).get("dram_bytes_main") else None,
            "achieved_kind": "ncu-counted executed FP64 FLOPs of the production kernel per GPU / its CUDA-event time",
            "source": (cap or {}).get("source"),
            "lib_sha256": lib_sha256_cached(),
            "peak_source": "measured live: DFMA microbenchmark (gpp_fp64_peak) on this GPU in this run",
            "kernel": "gpp_sacc_kernel (rcp_sq production kernel)",
            "kernel_ms": t_main_ms,
            "executed_flops_per_launch": per_gpu_main,
            "algorithmic_flops_per_launch": alg_job / n_ranks,
            "fp64_pipe_active_pct_ncu": (cap or {}).get("fp64_pipe_pct"),
            "fma_ratio_executed": r_exec,
            "fma_ceiling_tflops": peak_tf * (1 + r_exec) / 2 if r_exec else None,
            "frac_of_fma_ceiling": (achieved / (peak_tf * (1 + r_exec) / 2)) if (achieved and r_exec) else None,
            "fma_ratio_analytic": fma_ratio(cnt),
        },
        "gpu_launches": gpu_launches,
        "clocks": clk,
        "e2e": e2e,
        "e2e_pinned": e2e_pinned,
        "cpu_baseline": cpu,
        "branch_stats": {"instances": tot_inst, "near": near, "far": far},
        "kernel_info": info,
        "factored_time_to_solution": factored,
        "ncu": cap,
    }
    num = exec_job or alg_job
    if e2e:
        e2e["value"] = num / (e2e["ms_per_step"] * 1e-3) / 1e12
        if e2e_pinned:
            e2e_pinned["value"] = num / (e2e_pinned["ms_per_step"] * 1e-3) / 1e12
    if factored:
        factored["effective_tflops_equiv"] = alg_job / (factored["ms"] * 1e-3) / 1e12
    if args.variant == "rcp_sq":
        line["parity"] = golden_parity(result, args.workload, args.seed, args.nw)
    print(json.dumps(line), flush=True)
    (group.close() if group else ctx.close())


def main():
    args = parse_args()
    if args.ncu_child:
        ncu_child(args)
        return
    dist = Dist(args.gpus)
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
