"""Randomised parity of the CUDA paths against the oracle (hypothesis):
ragged dims, seeds, frequency counts (incl. > 4, i.e. several groups),
band-indexed wx, band shards, every kernel family.  GPU only."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import gpp_oracle as orc
from paper_2008_11326_b200 import GPPContext, GPPProblem, synth_problem
from paper_2008_11326_b200.dist import shard_problem
from paper_2008_11326_b200.errors import SynthesisError

pytestmark = pytest.mark.gpu

TOL = 1e-10
_CTX = {}


def _err(got, want) -> float:
    """max_rel_error, except that components the reference has exactly zero
    (possible for tiny random problems, e.g. no near instance at some iw) are
    compared absolutely against the accumulators' scale."""
    worst = 0.0
    for g, w in ((got.achtemp, want.achtemp), (got.asxtemp, want.asxtemp)):
        g, w = np.asarray(g), np.asarray(w)
        scale = max(float(np.max(np.abs(w))), 1e-300)
        denom = np.where(np.abs(w) > 0, np.abs(w), scale)
        worst = max(worst, float(np.max(np.abs(g - w) / denom)))
    return worst


def _ctx():
    if "c" not in _CTX:
        _CTX["c"] = GPPContext(0)
    return _CTX["c"]


@st.composite
def problems(draw):
    nb = draw(st.integers(1, 70))
    ng = draw(st.integers(1, 13))
    nc = draw(st.integers(1, 700))
    seed = draw(st.integers(0, 2**31 - 1))
    nw = draw(st.integers(1, 6))
    banded = draw(st.booleans())
    try:
        p = synth_problem(nb, ng, nc, seed=seed, nw=nw)
    except SynthesisError:
        p = synth_problem(nb, ng, nc, seed=seed + 1, nw=nw)
    if banded:
        rng = np.random.default_rng(seed)
        wxb = np.asfortranarray(rng.uniform(1.0, 2.0, size=(nw, nb)))
        p = GPPProblem(nb, ng, nc, p.wtilde, p.i_eps, p.aqsntemp, p.aqsmtemp, wxb)
    b0 = draw(st.integers(0, nb - 1))
    b1 = draw(st.integers(b0 + 1, nb))
    kernel = draw(st.sampled_from(["rcp_sq", "rcp_sq/iw", "rcp_sq/split", "rcp", "div"]))
    return p, (b0, b1), kernel


@settings(max_examples=150, deadline=None, derandomize=True, suppress_health_check=list(HealthCheck))
@given(problems())
def test_random_problems(case):
    p, br, kernel = case
    whole = orc.reference_result(p)
    shard = shard_problem(p, *br)
    want_shard = orc.reference_result(shard)
    _, near, far = orc.branch_stats(shard, "rcp_sq" if kernel.startswith("rcp_sq") else kernel)
    ctx = _ctx()
    ctx.upload(p, force=True)
    got, nf, _ = ctx.run(kernel, counts=True)
    assert _err(got, whole) <= TOL
    fast, _, _ = ctx.run(kernel, counts=False)
    assert _err(fast, whole) <= TOL
    part, nfs, _ = ctx.evaluate_host(p, kernel, band_range=br, counts=True, slabs=3)
    assert _err(part, want_shard) <= TOL
    assert nfs == (near, far)


@st.composite
def schedule_problems(draw):
    """Larger band counts than problems(): several wx-table band windows,
    512-band items, balanced tails and ragged last chunks, at random."""
    nb = draw(st.integers(200, 1700))
    ng = draw(st.integers(1, 6))
    nc = draw(st.integers(500, 24000))
    nw = draw(st.integers(1, 5))
    seed = draw(st.integers(0, 2**31 - 1))
    banded = draw(st.booleans())
    p = synth_problem(nb, ng, nc, seed=seed, nw=nw, check=False)
    if banded:
        rng = np.random.default_rng(seed)
        wxb = np.asfortranarray(rng.uniform(1.0, 2.0, size=(nw, nb)))
        p = GPPProblem(nb, ng, nc, p.wtilde, p.i_eps, p.aqsntemp, p.aqsmtemp, wxb)
    return p


@settings(max_examples=12, deadline=None, derandomize=True, suppress_health_check=list(HealthCheck))
@given(schedule_problems())
def test_random_production_schedules(p):
    want = orc.evaluate_variant(p, "rcp_sq")
    _, near, far = orc.branch_stats(p, "rcp_sq")
    ctx = _ctx()
    ctx.upload(p, force=True)
    got, nf, _ = ctx.run("rcp_sq", counts=True)
    assert _err(got, want) <= TOL
    assert nf == (near, far)
    fast, _, _ = ctx.run("rcp_sq", counts=False)
    assert _err(fast, want) <= TOL
