"""The reference's analytic FP64 instruction model, for the B200 path.

``run_version`` in the reference reports exact instruction counters built
from branch statistics (rooflab/gpp/kernel.py:117-212, rooflab/metrics.py:18-84).
The B200 path keeps that accounting so its counters are integer-identical to
the reference's -- the only difference is that the near/far statistics come
out of the CUDA kernel as a by-product instead of a second numpy pass.

These counts are also the ALGORITHMIC work used for the roofline:
``total_flops(counters)`` = 2*dfma + dadd + dmul + ddiv (metrics.py:63-76).
"""

from __future__ import annotations

from dataclasses import dataclass, fields

from .errors import DomainError, ValidationError

VARIANTS = ("div", "rcp", "rcp_sq")


@dataclass(frozen=True)
class InstructionCounters:
    """FP64 instruction counts by flop weight (metrics.py:18-60)."""

    dadd: int = 0
    dmul: int = 0
    dfma: int = 0
    ddiv: int = 0
    dother: int = 0

    def __post_init__(self) -> None:
        for f in fields(self):
            if getattr(self, f.name) < 0:
                raise ValidationError(f"counter {f.name} must be non-negative")

    def __add__(self, other: "InstructionCounters") -> "InstructionCounters":
        return InstructionCounters(
            *(getattr(self, f.name) + getattr(other, f.name) for f in fields(self))
        )

    def scaled(self, factor: int) -> "InstructionCounters":
        if factor < 0:
            raise DomainError(f"scale factor must be non-negative, got {factor!r}")
        return InstructionCounters(*(getattr(self, f.name) * factor for f in fields(self)))

    def to_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}


def total_flops(counters: InstructionCounters, div_weight: float = 1.0) -> float:
    """2*dfma + dadd + dmul + div_weight*ddiv (metrics.py:63-76)."""
    if div_weight < 0:
        raise DomainError(f"div_weight must be non-negative, got {div_weight!r}")
    return 2.0 * counters.dfma + counters.dadd + counters.dmul + div_weight * counters.ddiv


def fma_ratio(counters: InstructionCounters) -> float:
    """dfma / (dadd + dmul + dfma) (metrics.py:79-84)."""
    denom = counters.dadd + counters.dmul + counters.dfma
    if denom == 0:
        raise DomainError("fma_ratio undefined: no dadd/dmul/dfma instructions")
    return counters.dfma / denom


def fma_fraction(ratio: float) -> float:
    """Fraction of peak an FMA ratio can reach: (1 + r) / 2 (machine.py:44-53)."""
    if not 0.0 <= ratio <= 1.0:
        raise DomainError(f"fma_ratio must be in [0, 1], got {ratio!r}")
    return (1.0 + ratio) / 2.0


@dataclass(frozen=True)
class BranchStats:
    """How often each path of the nest runs (kernel.py:117-128)."""

    instances: int
    near: int
    far: int

    @property
    def degenerate(self) -> int:
        return self.instances - self.near - self.far


def _c(dadd=0, dmul=0, dfma=0, ddiv=0, dother=0) -> InstructionCounters:
    return InstructionCounters(dadd=dadd, dmul=dmul, dfma=dfma, ddiv=ddiv, dother=dother)


# Per-primitive decompositions, contraction on / off (kernel.py:144-178).
_PRIMITIVES = {
    #            contraction on                       contraction off
    "wdiff": (_c(dadd=1), _c(dadd=1)),
    "cdiv": (_c(dmul=3, dfma=3, ddiv=2), _c(dadd=3, dmul=6, ddiv=2)),
    "crcp": (_c(dmul=3, dfma=1, ddiv=1), _c(dadd=1, dmul=4, ddiv=1)),
    "cmul": (_c(dmul=2, dfma=2), _c(dadd=2, dmul=4)),
    "mag2": (_c(dmul=1, dfma=1), _c(dadd=1, dmul=2)),
    "abs": (_c(dmul=1, dfma=1, dother=1), _c(dadd=1, dmul=2, dother=1)),
    "cmp": (_c(dother=1), _c(dother=1)),
    "near_body": (_c(dmul=4, dfma=2), _c(dadd=2, dmul=6)),
    "far_body": (_c(dmul=2, ddiv=1), _c(dmul=2, ddiv=1)),
    "sqrt": (_c(dother=1), _c(dother=1)),
    "mac2": (_c(dfma=8), _c(dadd=8, dmul=8)),
    "tprod": (_c(dmul=2, dfma=2), _c(dadd=2, dmul=4)),
}


def primitive_table(contraction: bool = True) -> dict[str, InstructionCounters]:
    idx = 0 if contraction else 1
    return {name: pair[idx] for name, pair in _PRIMITIVES.items()}


def per_instance(variant: str, table: dict[str, InstructionCounters]) -> InstructionCounters:
    """Instructions every (band, igp, ig, iw) instance executes (kernel.py:181-188)."""
    if variant not in VARIANTS:
        raise DomainError(f"unknown variant {variant!r}, expected one of {VARIANTS}")
    common = table["wdiff"] + table["mac2"] + table["cmp"].scaled(2)
    if variant == "div":
        return common + table["cdiv"] + table["abs"].scaled(2)
    mags = table["abs"] if variant == "rcp" else table["mag2"]
    return common + table["crcp"] + table["cmul"] + mags.scaled(2)


def counters_from_stats(
    variant: str,
    stats: BranchStats,
    t_products: int,
    far_takes_sqrt: bool,
    contraction: bool = True,
) -> InstructionCounters:
    """Exact counts from branch statistics (kernel.py:191-212)."""
    table = primitive_table(contraction)
    out = per_instance(variant, table).scaled(stats.instances)
    out = out + table["near_body"].scaled(stats.near)
    out = out + table["cmp"].scaled(stats.instances - stats.near)
    far = table["far_body"] + (table["sqrt"] if far_takes_sqrt else _c())
    out = out + far.scaled(stats.far)
    return out + table["tprod"].scaled(t_products)


def algorithmic_flops(nbands: int, ngpown: int, ncouls: int, nw: int, near: int, far: int,
                      variant: str = "rcp_sq") -> int:
    """Analytic FLOPs of one full pass, as the reference's v8 counts them.

    For rcp_sq this is 35*I + 8*N + 3*F + 6*T.
    """
    tuples = nbands * ngpown * ncouls
    stats = BranchStats(instances=nw * tuples, near=near, far=far)
    counters = counters_from_stats(variant, stats, tuples, variant == "rcp_sq")
    return int(total_flops(counters))
