"""Version runner for the B200 path: mirror of rooflab/gpp/runner.py:55-333.

The reference's nine "versions" (runner.py:75-115) name an arithmetic variant
plus the traversal/launch shape the paper's V100 kernel used.  On B200 the
variant selects the CUDA kernel formulation (div / rcp = the reference's
per-instance formulas as written; rcp_sq = the optimised kernel); the
traversal is always the B200 one, so the launch shape reported in
``RunArtifacts`` is the real one of the kernel that ran (registers from
cudaFuncGetAttributes, resident CTAs from the occupancy API).

Counters stay integer-identical to the reference: they are assembled by the
reference's analytic model (counters.py) from the near/far counts the GPU
kernel produced as a by-product, instead of a second numpy pass
(runner.py:262-266, kernel.py:130-137).  Traces and the cache simulator
(runner.py:127-227, cachesim.py) model hardware the B200 path measures with
ncu instead; they are out of scope.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

from .counters import BranchStats, InstructionCounters, counters_from_stats
from .errors import DomainError
from .kernel import get_context
from .problem import GPPResult

WARP_SIZE = 32


@dataclass(frozen=True)
class VersionSpec:
    name: str
    variant: str
    order: str
    aqsm_band_fast: bool
    registers_per_thread: int
    threads_per_block: int
    description: str

    @property
    def t_per_instance(self) -> bool:
        return self.order == "iw_major"

    @property
    def far_takes_sqrt(self) -> bool:
        return self.variant == "rcp_sq"


# The reference's table (runner.py:75-115), values as it pins them
# (test_gpp.py:285-300).
VERSIONS: dict[str, VersionSpec] = {
    s.name: s
    for s in (
        VersionSpec("v0", "div", "band_major", False, 154, 128,
                    "baseline nest with library complex division and magnitude predicates"),
        VersionSpec("v1", "rcp", "band_major", False, 160, 128,
                    "complex division rewritten as reciprocal times multiply"),
        VersionSpec("v2", "rcp", "band_major", False, 160, 128,
                    "reciprocal form with the branch bodies folded together; modeled like v1"),
        VersionSpec("v3", "rcp_sq", "band_major", False, 154, 128,
                    "predicates compare squared magnitudes; sqrt survives only on the far branch"),
        VersionSpec("v4", "rcp_sq", "igp_major", False, 170, 128,
                    "nest reordered to igp, ig, band so the band reduction runs innermost"),
        VersionSpec("v5", "rcp_sq", "iw_major", False, 136, 128,
                    "iw hoisted outermost: one full pass of the nest per iw value"),
        VersionSpec("v6", "rcp_sq", "warp_blocked", False, 178, 128,
                    "band-blocked warp-lockstep traversal over ig chunks"),
        VersionSpec("v7", "rcp_sq", "warp_blocked", True, 184, 128,
                    "warp-lockstep traversal with aqsmtemp transposed to band-fastest"),
        VersionSpec("v8", "rcp_sq", "warp_blocked", True, 128, 512,
                    "v7 recompiled at 512 threads per block under a 128 register budget"),
    )
}
VERSION_NAMES = tuple(VERSIONS)

# The B200 ladder: which CUDA kernel re-derives each version's step
# (include/gpp_b200.h).  The reference's traversal-only versions (v2, v4, v6,
# v7) share the kernel of the arithmetic they keep; B200's traversal (thread
# <-> ig, band innermost, aqsmtemp/wx staged in shared memory, cp.async
# aqsntemp ring) is common to all kernels.
B200_KERNEL = {
    "v0": "div",            # library complex division, |.| predicates
    "v1": "rcp",            # reciprocal times multiply
    "v2": "rcp",            # branch bodies folded (predication: already so)
    "v3": "rcp_sq/split",   # squared predicates (integer compares), MUFU seeds
    "v4": "rcp_sq/split",   # band innermost (all B200 kernels)
    "v5": "rcp_sq/iw",      # per-tuple eps*t, P, Q reused across iw
    "v6": "rcp_sq/iw",      # cache blocking (smem staging, cp.async ring)
    "v7": "rcp_sq/seed",    # single rsqrt seed for 1/d and sqrt(d), far == !near
    "v8": "rcp_sq",         # per-(igp, iw) band sums, constants once per item
}


def version_spec(name: str) -> VersionSpec:
    try:
        return VERSIONS[name]
    except KeyError:
        raise DomainError(f"unknown version {name!r}, expected one of {', '.join(VERSIONS)}") from None


@dataclass(frozen=True)
class OccupancyResult:
    warps: int
    blocks: int
    max_warps: int = 64

    @property
    def occupancy(self) -> float:
        return self.warps / self.max_warps


@dataclass(frozen=True)
class RunArtifacts:
    """What one GPU evaluation produces (runner.py:230-246 shape)."""

    version: str
    dims: tuple[int, int, int]
    variant: str
    kernel: str
    result: GPPResult
    counters: InstructionCounters
    stats: BranchStats
    elapsed_s: float          # wall time of the evaluation call (perf_counter)
    kernel_s: float           # device time of the evaluation (CUDA events)
    registers_per_thread: int
    threads_per_block: int
    occupancy: OccupancyResult
    description: str
    trace: None = None
    sim: None = None


# Array ids of rooflab's element traces (runner.py:36-46), kept for name
# compatibility; the trace builders below are out of scope on B200.
ARRAY_NAMES = {0: "wtilde", 1: "i_eps", 2: "aqsntemp", 3: "aqsmtemp"}

_NO_TRACE = ("element traces model the V100 cache hierarchy for rooflab's cache simulator; "
             "out of scope on B200 -- profile the kernel with ncu (tools/ncu_summarize.py)")


def block_sizes(nbands: int, ncouls: int):
    """rooflab runner.py:127-136 (trace order helper): not provided."""
    raise DomainError(_NO_TRACE)


def tuple_order(name: str, nbands: int, ngpown: int, ncouls: int):
    """rooflab runner.py:190-197 (trace order helper): not provided."""
    raise DomainError(_NO_TRACE)


def build_trace(name: str, nbands: int, ngpown: int, ncouls: int):
    """rooflab runner.py:200-227 (element read trace): not provided."""
    raise DomainError(_NO_TRACE)


def _artifacts(ctx, problem, name, kernel, result, kernel_ms, elapsed, contraction) -> RunArtifacts:
    spec = version_spec(name)
    _, (near, far), _ = ctx.run(spec.variant, counts=True)
    nb, ng, nc = ctx.dims
    tuples = nb * ng * nc
    stats = BranchStats(instances=ctx.nw * tuples, near=near, far=far)
    t_products = tuples * (ctx.nw if spec.t_per_instance else 1)
    counters = counters_from_stats(spec.variant, stats, t_products, spec.far_takes_sqrt, contraction)
    info = ctx.kernel_info(kernel)
    warps = info["blocks_per_sm"] * info["threads_per_block"] // WARP_SIZE
    return RunArtifacts(
        version=name,
        dims=(nb, ng, nc),
        variant=spec.variant,
        kernel=kernel,
        result=result,
        counters=counters,
        stats=stats,
        elapsed_s=elapsed,
        kernel_s=kernel_ms * 1e-3,
        registers_per_thread=info["registers_per_thread"],
        threads_per_block=info["threads_per_block"],
        occupancy=OccupancyResult(warps=min(warps, 64), blocks=info["blocks_per_sm"]),
        description=spec.description,
    )


def run_version(problem, name: str, trace: bool = False, contraction: bool = True,
                device: int = 0) -> RunArtifacts:
    """Evaluate one version on the GPU and collect its artifacts (runner.py:249-286).

    As in the reference, the result comes from the version's *variant* alone
    (runner.py:258-260 calls evaluate_variant(problem, spec.variant)): every
    version sharing a variant returns bit-identical accumulators
    (test_gpp.py:88-94) -- v3..v8 all run the rcp_sq production kernel.  The
    paper's per-step kernels are ``run_ladder``.
    """
    spec = version_spec(name)
    if trace:
        raise DomainError("element traces belong to rooflab's cache model; profile with ncu instead")
    ctx = get_context(device)
    with ctx.lock:
        # Timed like the reference (runner.py:258-260): the evaluation alone;
        # the branch statistics come from a second, counting launch
        # (kernel.py:262 computes them in a separate pass too).
        start = time.perf_counter()
        if ctx.is_resident(problem):
            result, _, kernel_ms = ctx.run(spec.variant, counts=False)
        else:
            result, _, kernel_ms = ctx.evaluate_host(problem, spec.variant)
        elapsed = time.perf_counter() - start
        return _artifacts(ctx, problem, name, spec.variant, result, kernel_ms, elapsed, contraction)


def run_ladder(problem, name: str, contraction: bool = True, device: int = 0) -> RunArtifacts:
    """The B200 version ladder: version ``name``'s optimisation step
    re-derived as its own sm_100a kernel (B200_KERNEL) --
    the per-step evidence of the paper's trajectory.  Results agree with the
    reference to rounding (not bitwise across versions: the kernels' FP64
    arithmetic differs); counters are the reference's for the version."""
    version_spec(name)
    kernel = B200_KERNEL[name]
    ctx = get_context(device)
    with ctx.lock:
        ctx.upload(problem)
        start = time.perf_counter()
        result, _, kernel_ms = ctx.run(kernel, counts=False)
        elapsed = time.perf_counter() - start
        return _artifacts(ctx, problem, name, kernel, result, kernel_ms, elapsed, contraction)


def run_sweep(problem, names=None, device: int = 0) -> list[RunArtifacts]:
    """runner.py:289-308 without the cache simulation."""
    selected = tuple(VERSION_NAMES if names is None else names)
    return [run_version(problem, n, device=device) for n in selected]


def emit_metrics(artifacts: RunArtifacts, runtime: float | None = None, system: str | None = None) -> dict:
    """KernelMetrics-shaped record (runner.py:311-333, metrics.py:131-143)."""
    return {
        "label": artifacts.version,
        "runtime": artifacts.kernel_s if runtime is None else runtime,
        "counters": artifacts.counters.to_dict(),
        "bytes": None,
        **({"system": system} if system is not None else {}),
        "registers_per_thread": artifacts.registers_per_thread,
        "threads_per_block": artifacts.threads_per_block,
        "achieved_warps_per_sm": artifacts.occupancy.warps,
    }
