"""Parity of the sm_100a kernels (through the C ABI) with the reference.

Gate (BASELINE.json north_star): max_rel_error <= 1e-10 against the
reference's achtemp/asxtemp on identical synthetic inputs, and near/far
counts EXACTLY equal to the reference's branch_stats (integer work).
Small cases compare against golden fixtures generated from the unmodified
reference (tests/golden/make_golden.py) and against the oracle run here;
paper / sweep / weak sizes against the committed reference outputs.
"""

import numpy as np
import pytest

from conftest import as_complex, load_cases
from oracle import gpp_oracle as orc
from paper_2008_11326_b200 import (
    GPPContext,
    GPPProblem,
    branch_stats,
    evaluate,
    evaluate_variant,
    reference_result,
    run_version,
    synth_problem,
)
from paper_2008_11326_b200.problem import max_rel_error

pytestmark = pytest.mark.gpu

TOL = 1e-10  # north_star: results within 1e-10 relative error
SMALL = load_cases("gpp_small.json")
BIG = load_cases("gpp_big.json")


class _R:
    def __init__(self, d):
        self.achtemp = as_complex(d["achtemp"])
        self.asxtemp = as_complex(d["asxtemp"])


def _ids(cases):
    return [f"{tuple(c['dims'])}-s{c['seed']}-nw{c['nw']}" for c in cases]


@pytest.mark.parametrize("case", SMALL, ids=_ids(SMALL))
@pytest.mark.parametrize("variant", ["div", "rcp", "rcp_sq"])
def test_small_cases_vs_reference(case, variant):
    """Both kernels: the counting one (general path) and the production one
    evaluate_variant runs (regular-item fast path)."""
    p = synth_problem(*case["dims"], seed=case["seed"], nw=case["nw"])
    got, stats, _ = evaluate(p, variant)
    fast = evaluate_variant(p, variant)
    for r in (got, fast):
        assert max_rel_error(r, _R(case["reference_result"])) <= TOL
        assert max_rel_error(r, _R(case["evaluate_variant"][variant])) <= TOL
    assert [stats.instances, stats.near, stats.far] == case["branch_stats"][variant]


@pytest.mark.parametrize("case", BIG, ids=_ids(BIG))
def test_big_cases_vs_reference(case):
    """Paper, weak and all 24 aspect-ratio sweep points (BASELINE configs[1],
    [3], [4]) against the unmodified reference's outputs.  The inputs are
    drawn on the device (gpp_synth, bit-exact with synth_problem:
    test_device_synthesis_is_bitexact); both kernels run -- the counting one
    for the exact near/far counts and the production one evaluate_variant
    uses."""
    nb, ng, nc = case["dims"]
    ctx = GPPContext(0)
    try:
        ctx.synth(nb, ng, nc, seed=case["seed"], nw=case["nw"])
        got, (near, far), _ = ctx.run("rcp_sq", counts=True)
        fast = ctx.run("rcp_sq", counts=False)[0]
    finally:
        ctx.close()
    want = _R(case.get("reference_result") or case["evaluate_variant"]["rcp_sq"])
    for r in (got, fast):
        err = max_rel_error(r, want)
        assert err <= TOL, err
    assert [case["nw"] * nb * ng * nc, near, far] == case["branch_stats"]["rcp_sq"]


def test_paper_size_public_path_vs_reference():
    """evaluate_variant on host arrays (first call: upload pipelined with the
    kernel; second: resident) at the paper size, nw 2 and 3."""
    for nw in (2, 3):
        case = next(c for c in BIG if c["dims"] == [512, 66, 32768] and c["seed"] == 1 and c["nw"] == nw)
        p = synth_problem(512, 66, 32768, seed=1, nw=nw, check=False)
        first = evaluate_variant(p, "rcp_sq")
        again = evaluate_variant(p, "rcp_sq")
        assert _bits_equal(first, again)
        want = _R(case.get("reference_result") or case["evaluate_variant"]["rcp_sq"])
        assert max_rel_error(first, want) <= TOL
        assert [branch_stats(p, "rcp_sq").near, branch_stats(p, "rcp_sq").far] == case["branch_stats"]["rcp_sq"][1:]


def _bits_equal(a, b) -> bool:
    return np.array_equal(a.achtemp, b.achtemp) and np.array_equal(a.asxtemp, b.asxtemp)


def test_plain_variants_paper_size():
    case = next(c for c in BIG if c["dims"] == [512, 66, 32768] and c["seed"] == 1 and c["nw"] == 2)
    p = synth_problem(512, 66, 32768, seed=1)
    want = _R(case["reference_result"])
    for variant in ("div", "rcp"):
        got, stats, _ = evaluate(p, variant)
        assert max_rel_error(got, want) <= TOL, variant
        assert stats.far == case["branch_stats"]["rcp_sq"][2]


def test_kat_golden_64x64x512():
    from paper_2008_11326_b200.problem import load_golden
    from conftest import GOLDEN

    dims, seed, golden = load_golden(GOLDEN / "gpp-golden-seed42-64x64x512.json")
    p = synth_problem(*dims, seed=seed)
    assert max_rel_error(reference_result(p), golden) <= 1e-12
    assert max_rel_error(evaluate_variant(p, "rcp_sq"), golden) <= 1e-12


@pytest.mark.parametrize("nw", [1, 4, 5, 9])
def test_other_frequency_counts_vs_oracle(nw):
    """nw is a parameter (groups of <= 4 per launch); oracle on the same input."""
    p = synth_problem(24, 7, 300, seed=11, nw=nw)
    want = orc.reference_result(p)
    inst, near, far = orc.branch_stats(p, "rcp_sq")
    for variant in ("rcp_sq", "div"):
        got, stats, _ = evaluate(p, variant)
        assert max_rel_error(got, want) <= TOL
        assert max_rel_error(evaluate_variant(p, variant), want) <= TOL
        assert (stats.instances, stats.near, stats.far) == (inst, near, far)


def test_band_indexed_wx_vs_oracle():
    """BerkeleyGW's wx_array(iw, n1): every band has its own frequencies."""
    base = synth_problem(40, 9, 700, seed=3)
    rng = np.random.default_rng(5)
    wxb = np.asfortranarray(rng.uniform(1.0, 2.0, size=(3, 40)))
    p = GPPProblem(40, 9, 700, base.wtilde, base.i_eps, base.aqsntemp, base.aqsmtemp, wxb)
    want = orc.reference_result(p)
    inst, near, far = orc.branch_stats(p, "rcp_sq")
    for variant in ("rcp_sq", "rcp", "div"):
        got, stats, _ = evaluate(p, variant)
        assert max_rel_error(got, want) <= TOL, variant
        assert max_rel_error(evaluate_variant(p, variant), want) <= TOL, variant
        assert (stats.instances, stats.near, stats.far) == (inst, near, far), variant


def test_band_shards_sum_to_whole():
    """Band sharding (the multi-GPU partition) on one device: shards add up."""
    p = synth_problem(64, 33, 1000, seed=1, nw=3)
    whole, (n0, f0), _ = _run(p, None)
    parts = [_run(p, r) for r in ((0, 17), (17, 40), (40, 64))]
    ach = sum(r[0].achtemp for r in parts)
    asx = sum(r[0].asxtemp for r in parts)
    assert max_rel_error(type(whole)(achtemp=ach, asxtemp=asx), whole) <= 1e-12
    assert sum(r[1][0] for r in parts) == n0 and sum(r[1][1] for r in parts) == f0


def _run(p, band_range):
    ctx = GPPContext(0)
    try:
        ctx.upload(p, band_range)
        return ctx.run("rcp_sq")
    finally:
        ctx.close()


@pytest.mark.parametrize("dims,nw", [((128, 66, 4096), 3), ((512, 66, 32768), 3),
                                     ((600, 33, 5000), 2), ((1100, 17, 9000), 3),
                                     ((300, 10, 3000), 1), ((64, 9, 700), 5)])
def test_bitwise_reproducible_on_every_path(dims, nw):
    """fixed inputs and variant give the same bits whatever
    the path: the first call (upload pipelined with the kernel over ig slabs),
    the resident re-run, any slab count, a fresh context.  Every schedule runs
    the same canonical items and the finalize sums them in slot order."""
    p = synth_problem(*dims, seed=1, nw=nw, check=False)
    for variant in ("rcp_sq", "div"):
        if variant == "div" and dims[0] * dims[1] * dims[2] > 10**8:
            continue
        first = evaluate_variant(p, variant)          # pipelined upload + evaluate
        again = evaluate_variant(p, variant)          # resident
        assert _bits_equal(first, again), variant
        ctx = GPPContext(0)
        try:
            for slabs in (1, 2, 3, 7, 0):
                r = ctx.evaluate_host(p, variant, slabs=slabs)[0]
                assert _bits_equal(r, first), (variant, slabs)
            ctx.upload(p, force=True)
            assert _bits_equal(ctx.run(variant, counts=False)[0], first), variant
        finally:
            ctx.close()


def test_versions_sharing_a_variant_agree_bitwise():
    """rooflab test_gpp.py:88-94 on this package: run_version's result comes
    from the version's variant alone (runner.py:258-260)."""
    for dims in ((64, 64, 512), (512, 66, 32768)):
        p = synth_problem(*dims, seed=1, nw=3, check=False)
        by_name = {name: run_version(p, name).result for name in
                   ("v0", "v1", "v2", "v3", "v4", "v5", "v6", "v7", "v8")}
        assert _bits_equal(by_name["v1"], by_name["v2"])
        for name in ("v4", "v5", "v6", "v7", "v8"):
            assert _bits_equal(by_name["v3"], by_name[name]), name
        assert _bits_equal(by_name["v8"], evaluate_variant(p, "rcp_sq"))


def test_writeable_inputs_are_reuploaded():
    p = synth_problem(8, 8, 64, seed=1)
    arrs = {k: np.array(getattr(p, k), order="F") for k in ("wtilde", "i_eps", "aqsntemp", "aqsmtemp", "wx")}
    q = GPPProblem(8, 8, 64, **arrs)
    first = evaluate_variant(q, "rcp_sq")
    arrs["aqsntemp"] *= 2.0
    second = evaluate_variant(q, "rcp_sq")
    np.testing.assert_allclose(second.achtemp, 2.0 * first.achtemp, rtol=1e-12)


def test_run_version_counters_match_reference():
    case = next(c for c in SMALL if c["dims"] == [64, 64, 512] and c["seed"] == 7 and c["nw"] == 2)
    p = synth_problem(64, 64, 512, seed=7)
    for name, want in case["counters"].items():
        art = run_version(p, name)
        assert art.counters.to_dict() == want, name
        assert max_rel_error(art.result, _R(case["reference_result"])) <= TOL
        assert art.registers_per_thread > 0 and art.kernel_s > 0


def test_branch_stats_api():
    p = synth_problem(4, 4, 64, seed=7)
    s = branch_stats(p, "div")
    assert s.near > 0 and s.far > 0 and s.instances == 2 * 4 * 4 * 64


def test_degenerate_inputs():
    """wtilde == 0 makes delw vanish: near iff |wdiff| > 0.5, never far."""
    p = synth_problem(5, 3, 40, seed=1)
    wt = np.array(p.wtilde, order="F")
    wt[:7, 1] = 0.0
    q = GPPProblem(5, 3, 40, wt, p.i_eps, p.aqsntemp, p.aqsmtemp, p.wx)
    want = orc.reference_result(q)
    inst, near, far = orc.branch_stats(q, "div")
    for variant in ("rcp_sq", "div", "rcp"):
        got, stats, _ = evaluate(q, variant)
        assert max_rel_error(got, want) <= TOL, variant
        assert max_rel_error(evaluate_variant(q, variant), want) <= TOL, variant
        assert (stats.near, stats.far) == (near, far), variant


def test_irregular_items_take_the_general_path():
    """Items with a degenerate-capable (ig, igp) -- wt.im == 0 makes d = 0
    possible, tiny |wt| makes |delw| <= 1e-12 possible -- must reproduce the
    reference's degenerate handling in the production kernel too."""
    p = synth_problem(12, 5, 300, seed=7)
    wt = np.array(p.wtilde, order="F")
    wt[3, 1] = complex(p.wx[0], 0.0)    # wdiff == 0 exactly for iw 0 (real wtilde)
    wt[10, 2] = 1e-14 + 0j              # |delw| ~ 1e-14: degenerate
    wt[200, 4] = complex(0.3, 0.0)      # real wtilde, not singular
    q = GPPProblem(12, 5, 300, wt, p.i_eps, p.aqsntemp, p.aqsmtemp, p.wx)
    want = orc.evaluate_variant(q, "rcp_sq")
    inst, near, far = orc.branch_stats(q, "rcp_sq")
    got, stats, _ = evaluate(q, "rcp_sq")
    assert (stats.near, stats.far) == (near, far)
    for r in (got, evaluate_variant(q, "rcp_sq")):
        assert np.all(np.isfinite(r.achtemp)) and np.all(np.isfinite(r.asxtemp))
        assert max_rel_error(r, want) <= TOL


@pytest.mark.parametrize("slabs", [0, 1, 3, 8, 1000])
def test_pipelined_host_evaluate(slabs):
    """gpp_evaluate_host: H2D by ig slabs overlapped with the kernel; same
    result as upload + run (bitwise: same items, same partial order per slab
    set), and ragged ncouls (not a multiple of 256)."""
    p = synth_problem(40, 9, 1000, seed=1, nw=3)
    want = orc.reference_result(p)
    ctx = GPPContext(0)
    try:
        got, nf, ms = ctx.evaluate_host(p, "rcp_sq", counts=True, slabs=slabs)
        assert max_rel_error(got, want) <= TOL
        inst, near, far = orc.branch_stats(p, "rcp_sq")
        assert nf == (near, far)
        again, _, _ = ctx.run("rcp_sq", counts=False)  # now resident
        assert max_rel_error(again, want) <= TOL
        part, _, _ = ctx.evaluate_host(p, "rcp_sq", band_range=(10, 30), slabs=slabs)
        ref = orc.reference_result(__import__("paper_2008_11326_b200.dist", fromlist=["x"]).shard_problem(p, 10, 30))
        assert max_rel_error(part, ref) <= TOL
    finally:
        ctx.close()


@pytest.mark.parametrize("nw", [3, 6])
def test_pipelined_taper_two_streams(nw):
    """The default (tapered) slab schedule over 40 ig blocks: slabs alternate
    between two compute streams, and with nw = 6 the second frequency group's
    slabs must wait for the first group's finalize.  Oracle parity, exact
    counts, and bitwise repeatability of the pipelined path."""
    p = synth_problem(24, 5, 40 * 256 - 17, seed=3, nw=nw)
    want = orc.reference_result(p)
    inst, near, far = orc.branch_stats(p, "rcp_sq")
    ctx = GPPContext(0)
    try:
        got, nf, _ = ctx.evaluate_host(p, "rcp_sq", counts=True)
        assert max_rel_error(got, want) <= TOL
        assert nf == (near, far)
        for _ in range(3):
            again, _, _ = ctx.evaluate_host(p, "rcp_sq", counts=True)
            assert np.array_equal(again.achtemp, got.achtemp)
            assert np.array_equal(again.asxtemp, got.asxtemp)
    finally:
        ctx.close()


@pytest.mark.parametrize("dims,nw", [((600, 3, 40000), 3), ((40, 5, 40000), 2)])
def test_pipelined_host_evaluate_production_schedules(dims, nw):
    """The pipelined host path with the production kernel's schedules inside
    each ig slab: two band windows (600 bands at nw 3) and balanced-tail
    launches on the other stream (40 bands, several items per CTA)."""
    p = synth_problem(*dims, seed=9, nw=nw, check=False)
    want = orc.evaluate_variant(p, "rcp_sq")
    inst, near, far = orc.branch_stats(p, "rcp_sq")
    ctx = GPPContext(0)
    try:
        for slabs in (0, 1, 5):
            got, nf, _ = ctx.evaluate_host(p, "rcp_sq", counts=True, slabs=slabs)
            assert max_rel_error(got, want) <= TOL
            assert nf == (near, far)
    finally:
        ctx.close()


@pytest.mark.parametrize("kernel", ["rcp_sq/split", "rcp_sq/iw"])
def test_ladder_kernels_vs_reference(kernel):
    """The intermediate kernels of the B200 version ladder give the reference's
    results and exact counts too."""
    ctx = GPPContext(0)
    try:
        for case in [c for c in SMALL if c["dims"] in ([47, 2, 33], [64, 64, 512], [32, 8, 512])]:
            p = synth_problem(*case["dims"], seed=case["seed"], nw=case["nw"])
            ctx.upload(p)
            got, nf, _ = ctx.run(kernel, counts=True)
            assert max_rel_error(got, _R(case["reference_result"])) <= TOL
            assert [case["nw"] * np.prod(case["dims"]), *nf] == case["branch_stats"]["rcp_sq"]
            fast, _, _ = ctx.run(kernel, counts=False)
            assert max_rel_error(fast, _R(case["reference_result"])) <= TOL
    finally:
        ctx.close()


def test_evaluate_variant_rejects_ladder_names():
    from paper_2008_11326_b200.errors import DomainError

    with pytest.raises(DomainError):
        evaluate_variant(synth_problem(2, 2, 16, seed=5), "rcp_sq/iw")


def test_single_process_group_api():
    """gpp_comm_init_all + gpp_run_group over the visible devices (one on the
    test boxes): the grouped path returns the whole problem's result."""
    import ctypes

    from paper_2008_11326_b200 import _lib
    from paper_2008_11326_b200.dist import MultiDeviceGPP

    n = ctypes.c_int()
    _lib.load().gpp_device_count(ctypes.byref(n))
    devices = list(range(min(n.value, 8)))
    p = synth_problem(37, 9, 600, seed=7, nw=3)
    want = orc.reference_result(p)
    inst, near, far = orc.branch_stats(p, "rcp_sq")
    g = MultiDeviceGPP(devices)
    try:
        g.upload(p)
        got, nf, ms = g.run("rcp_sq", counts=True)
        assert max_rel_error(got, want) <= TOL and nf == (near, far) and ms > 0
        fast, _, _ = g.run("rcp_sq", counts=False)
        assert max_rel_error(fast, want) <= TOL
    finally:
        g.close()
    with pytest.raises(ValueError):
        MultiDeviceGPP([0, 0])


@pytest.mark.parametrize("variant", ["div", "rcp", "rcp_sq"])
def test_factored_path_vs_reference(variant):
    """gpp_run_factored (band-weight GEMM fused with the terms in one repo kernel: the reference's own algorithm)."""
    ctx = GPPContext(0)
    try:
        for case in [c for c in SMALL if c["dims"] in ([5, 3, 40], [47, 2, 33], [64, 64, 512])]:
            p = synth_problem(*case["dims"], seed=case["seed"], nw=case["nw"])
            ctx.upload(p)
            got, nf, ms = ctx.run_factored(variant, counts=True)
            assert max_rel_error(got, _R(case["evaluate_variant"][variant])) <= 1e-12
            assert [case["nw"] * int(np.prod(case["dims"])), *nf] == case["branch_stats"][variant]
        case = next(c for c in BIG if c["dims"] == [512, 66, 32768] and c["seed"] == 1 and c["nw"] == 3)
        p = synth_problem(512, 66, 32768, seed=1, nw=3, check=False)
        ctx.upload(p)
        got, nf, ms = ctx.run_factored(variant, counts=True)
        assert max_rel_error(got, _R(case["evaluate_variant"]["rcp_sq"])) <= TOL
        if variant == "rcp_sq":
            assert [3 * 512 * 66 * 32768, *nf] == case["branch_stats"]["rcp_sq"]
        # band-indexed wx with distinct columns is not factorable
        wxb = np.asfortranarray(np.stack([p.wx] * 511 + [p.wx + 0.01], axis=1))
        q = GPPProblem(512, 66, 32768, p.wtilde, p.i_eps, p.aqsntemp, p.aqsmtemp, wxb)
        ctx.upload(q)
        from paper_2008_11326_b200.errors import DomainError
        with pytest.raises(DomainError):
            ctx.run_factored(variant)
    finally:
        ctx.close()


@pytest.mark.parametrize("dims,seed,nw,br", [
    ((5, 3, 40), 1, 2, None), ((47, 2, 33), 7, 3, None), ((64, 64, 512), 42, 2, (10, 50)),
    ((512, 66, 32768), 1, 3, None),
])
def test_device_synthesis_is_bitexact(dims, seed, nw, br):
    """gpp_synth draws synth_problem's arrays on the device (numpy PCG64 +
    uniform, bit-exact): the kernel sees identical inputs, so its result is
    bitwise the host-synthesized one."""
    p = synth_problem(*dims, seed=seed, nw=nw, check=False)
    a = GPPContext(0)
    b = GPPContext(0)
    try:
        a.synth(*dims, seed=seed, nw=nw, band_range=br)
        assert np.array_equal(a.synth_wx, p.wx)
        b.upload(p, br)
        ra, nfa, _ = a.run("rcp_sq", counts=True)
        rb, nfb, _ = b.run("rcp_sq", counts=True)
        assert nfa == nfb
        assert np.array_equal(ra.achtemp, rb.achtemp) and np.array_equal(ra.asxtemp, rb.asxtemp)
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("variant", ["div", "rcp", "rcp_sq"])
def test_variant_terms_vs_oracle(variant):
    """GPU variant_terms (kernel.py:63-95): masks exact, terms to rounding."""
    from paper_2008_11326_b200 import variant_terms

    for dims, seed, nw in (((4, 7, 300), 1, 2), ((3, 13, 129), 7, 3)):
        p = synth_problem(*dims, seed=seed, nw=nw)
        got = variant_terms(p, variant)
        sch, ssx, near, far = orc.variant_terms(p, variant)
        assert np.array_equal(got.near, near) and np.array_equal(got.far, far)
        scale = max(np.abs(sch).max(), np.abs(ssx).max())
        assert np.abs(got.sch - sch).max() <= 1e-14 * scale
        assert np.abs(got.ssx - ssx).max() <= 1e-14 * scale


# Schedules of the production kernel (csrc/gpp_lib.cu enqueue_eval): several
# band windows of the by-value wx table (512 bands at nw 3, 768 at nw 2, 1536
# at nw 1), the balanced-tail second launch, and items shorter than the
# aqsntemp ring (the ring re-primes).  Oracle on the same inputs.
@pytest.mark.parametrize("dims,nw", [
    ((600, 3, 300), 3),      # two band windows, few items
    ((1100, 2, 256), 2),     # two windows at nw 2
    ((1600, 2, 300), 1),     # two windows at nw 1
    ((258, 33, 8192), 3),    # 2-band last chunk (short items) + balanced tail
    ((5, 7, 70000), 3),      # 5-band items, balanced tail of 5-band rows
    ((2, 5, 40000), 1),      # every item shorter than the ring
    ((1, 1, 1), 3),
])
def test_production_schedules_vs_oracle(dims, nw):
    p = synth_problem(*dims, seed=5, nw=nw, check=False)
    want = orc.evaluate_variant(p, "rcp_sq")
    inst, near, far = orc.branch_stats(p, "rcp_sq")
    got, stats, _ = evaluate(p, "rcp_sq")
    assert max_rel_error(got, want) <= TOL
    assert max_rel_error(evaluate_variant(p, "rcp_sq"), want) <= TOL
    assert (stats.instances, stats.near, stats.far) == (inst, near, far)


def test_concurrent_contexts_from_threads():
    """Independent runs may proceed concurrently: two contexts
    on the same device, driven from two threads (ctypes releases the GIL),
    each with its own problem; the by-value wx tables and per-context
    buffers/streams keep them apart."""
    import threading

    probs = [synth_problem(300, 5, 9000, seed=s, nw=nw, check=False) for s, nw in ((3, 3), (4, 2))]
    wants = [orc.evaluate_variant(p, "rcp_sq") for p in probs]
    errs = [None, None]

    def work(k):
        ctx = GPPContext(0)
        try:
            ctx.upload(probs[k], force=True)
            worst = 0.0
            for _ in range(20):
                got, _, _ = ctx.run("rcp_sq", counts=False)
                worst = max(worst, max_rel_error(got, wants[k]))
            errs[k] = worst
        finally:
            ctx.close()

    ts = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert errs[0] is not None and errs[1] is not None
    assert max(errs) <= TOL


def test_public_seam_is_thread_safe():
    """The drop-in path itself (evaluate_variant / branch_stats, no explicit
    context) called from four threads at once with different problems and
    variants: every call returns exactly the bits of the same call made
    alone (per-thread contexts)."""
    import threading

    probs = [synth_problem(200, 7, 5000, seed=s, nw=nw, check=False)
             for s, nw in ((3, 3), (4, 2), (5, 3), (6, 1))]
    variants = ["rcp_sq", "rcp_sq", "rcp", "rcp_sq"]
    alone = [evaluate_variant(p, v) for p, v in zip(probs, variants)]
    counts = [branch_stats(p, "rcp_sq") for p in probs]
    bad = []
    barrier = threading.Barrier(4)

    def work(k):
        barrier.wait()
        for i in range(8):
            # alternate fresh (writeable copy: pipelined upload) and resident calls
            q = probs[k]
            if i % 2:
                q = GPPProblem(q.nbands, q.ngpown, q.ncouls, q.wtilde.copy(order="F"),
                               q.i_eps.copy(order="F"), q.aqsntemp.copy(order="F"),
                               q.aqsmtemp.copy(order="F"), q.wx.copy())
            got = evaluate_variant(q, variants[k])
            if not _bits_equal(got, alone[k]):
                bad.append((k, i))
            s = branch_stats(q, "rcp_sq")
            if (s.near, s.far) != (counts[k].near, counts[k].far):
                bad.append((k, i, "counts"))

    ts = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert bad == []


def test_shared_context_serialises_callers():
    """One explicit GPPContext driven from two threads: the library's
    per-context lock serialises the calls, so each thread's result is its own
    problem's, bit for bit."""
    import threading

    probs = [synth_problem(100, 5, 3000, seed=s, nw=3, check=False) for s in (8, 9)]
    alone = [evaluate_variant(p, "rcp_sq") for p in probs]
    ctx = GPPContext(0)
    bad = []

    def work(k):
        for _ in range(10):
            got = ctx.evaluate_host(probs[k], "rcp_sq")[0]
            if not _bits_equal(got, alone[k]):
                bad.append(k)

    try:
        ts = [threading.Thread(target=work, args=(k,)) for k in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    finally:
        ctx.close()
    assert bad == []


def test_empty_band_shard_contributes_zeros():
    """More ranks than bands: a rank's shard [b, b) is empty -- it uploads
    nothing, contributes zeros and still joins the collective (no rank can
    fail before the allreduce while its peers wait in it)."""
    p = synth_problem(6, 5, 700, seed=2, nw=3, check=False)
    whole = evaluate_variant(p, "rcp_sq")
    ctx = GPPContext(0)
    try:
        ctx.upload(p, (3, 3))
        r, (near, far), _ = ctx.run("rcp_sq", counts=True)
        assert not np.any(r.achtemp) and not np.any(r.asxtemp) and near == far == 0
        r2 = ctx.evaluate_host(p, "rcp_sq", band_range=(6, 6), counts=True)
        assert not np.any(r2[0].achtemp) and r2[1] == (0, 0)
        tot, main = ctx.time("rcp_sq", 3)
        assert tot >= 0.0
        parts = []
        for br in ((0, 3), (3, 3), (3, 6)):
            ctx.upload(p, br, force=True)
            parts.append(ctx.run("rcp_sq", counts=False)[0])
    finally:
        ctx.close()
    ach = sum(x.achtemp for x in parts)
    asx = sum(x.asxtemp for x in parts)
    assert max_rel_error(type(whole)(achtemp=ach, asxtemp=asx), whole) <= 1e-13


def test_group_path_bitmatches_single_context():
    """The single-process multi-device path (MultiDeviceGPP: gpp_comm_init_all,
    gpp_run_group, gpp_time_group, threaded evaluate) on one device gives the
    bits of the plain context; its timing entry point runs."""
    from paper_2008_11326_b200.dist import MultiDeviceGPP

    dims = (512, 66, 32768)
    ctx = GPPContext(0)
    try:
        ctx.synth(*dims, seed=1, nw=3)
        want = ctx.run("rcp_sq", counts=False)[0]
    finally:
        ctx.close()
    g = MultiDeviceGPP([0])
    try:
        g.synth(*dims, seed=1, nw=3)
        got, (near, far), _ = g.run("rcp_sq", counts=True)
        fast = g.run("rcp_sq", counts=False)[0]
        assert _bits_equal(fast, want)
        tot, main = g.time("rcp_sq", 3)
        assert tot > 0.0 and 0.0 < main <= tot
        p = synth_problem(*dims, seed=1, nw=3, check=False)
        e2e, _ = g.evaluate(p, "rcp_sq")
        assert _bits_equal(e2e, want)
    finally:
        g.close()


def test_pinned_pageable_and_column_split_uploads_bitwise():
    """Every upload route gives the same bits: pageable arrays (library
    staging ring), page-locked arrays (direct DMA), and the column-split
    wtilde / i_eps upload the band-sharded e2e path uses (forced on one rank
    with GPP_COLUMN_UPLOAD=1, in a subprocess)."""
    import subprocess
    import sys

    from paper_2008_11326_b200._lib import check, load

    p = synth_problem(300, 13, 9000, seed=4, nw=3, check=False)
    want = evaluate_variant(p, "rcp_sq")
    q = GPPProblem(p.nbands, p.ngpown, p.ncouls, p.wtilde.copy(order="F"), p.i_eps.copy(order="F"),
                   p.aqsntemp.copy(order="F"), p.aqsmtemp.copy(order="F"), p.wx.copy())
    assert _bits_equal(evaluate_variant(q, "rcp_sq"), want)  # pageable (writeable: re-uploaded)
    lib = load()
    arrs = [q.wtilde, q.i_eps, q.aqsntemp, q.aqsmtemp]
    for a in arrs:
        check(lib.gpp_host_register(a.ctypes.data, a.nbytes))
    try:
        assert _bits_equal(evaluate_variant(q, "rcp_sq"), want)  # pinned
    finally:
        for a in arrs:
            lib.gpp_host_unregister(a.ctypes.data)
    code = (
        "import json\n"
        "from paper_2008_11326_b200 import GPPContext, synth_problem\n"
        "p = synth_problem(300, 13, 9000, seed=4, nw=3, check=False)\n"
        "c = GPPContext(0)\n"
        "r = [c.evaluate_host(p, 'rcp_sq', band_range=br)[0] for br in (None, (0, 140), (140, 300))]\n"
        "f = lambda z: [[v.real, v.imag] for v in z]\n"
        "print(json.dumps([f(r[0].achtemp), f(r[0].asxtemp), f(r[1].achtemp + r[2].achtemp)]))\n"
    )
    import json
    import os

    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         env={**os.environ, "GPP_COLUMN_UPLOAD": "1"}, cwd=str(__import__("conftest").ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    ach, asx, shards = (as_complex(x) for x in json.loads(out.stdout.strip().splitlines()[-1]))
    assert np.array_equal(ach, want.achtemp) and np.array_equal(asx, want.asxtemp)
    assert max_rel_error(type(want)(achtemp=shards, asxtemp=want.asxtemp), want) <= 1e-12


@pytest.mark.parametrize("dims,nw", [((24, 7, 300), 5), ((130, 17, 2000), 1), ((700, 9, 1000), 4)])
def test_factored_kernel_odd_shapes_vs_oracle(dims, nw):
    """The fused factored kernel at ragged igp tiles (ngpown not a multiple
    of its 8-igp tile), band counts not a multiple of its 64-band staging,
    and frequency groups (nw 4, 5): against the oracle's factored path."""
    p = synth_problem(*dims, seed=3, nw=nw, check=False)
    want = orc.evaluate_variant(p, "rcp_sq")
    _, near, far = orc.branch_stats(p, "rcp_sq")
    ctx = GPPContext(0)
    try:
        ctx.upload(p)
        for variant in ("rcp_sq", "rcp", "div"):
            got, nf, _ = ctx.run_factored(variant, counts=True)
            assert max_rel_error(got, want) <= 1e-12, variant
            assert nf == (near, far), variant
    finally:
        ctx.close()


def test_error_after_comm_init_aborts_the_communicator():
    """An error on a rank that holds a communicator aborts it (ncclCommAbort),
    so its peers fail instead of waiting in a collective it will never join;
    the context then refuses further work with an NCCL error (a one-rank
    communicator on one GPU exercises the mechanism)."""
    from paper_2008_11326_b200.errors import DomainError, GPUError
    from paper_2008_11326_b200.kernel import comm_unique_id

    p = synth_problem(16, 5, 600, seed=3, nw=3, check=False)
    ctx = GPPContext(0)
    try:
        ctx.comm_init(1, 0, comm_unique_id())
        ctx.upload(p)
        ok = ctx.run("rcp_sq", counts=False)[0]
        assert _bits_equal(ok, evaluate_variant(p, "rcp_sq"))
        with pytest.raises(DomainError):
            ctx.upload(p, band_range=(5, 2), force=True)   # bad argument after comm init
        with pytest.raises(GPUError, match="aborted"):
            ctx.run("rcp_sq", counts=False)
    finally:
        ctx.close()


def test_release_context_frees_and_recreates():
    """release_context() drops the calling thread's context; the next call
    creates a fresh one and returns the same bits."""
    from paper_2008_11326_b200 import release_context
    from paper_2008_11326_b200.kernel import get_context

    p = synth_problem(40, 5, 900, seed=6, nw=3, check=False)
    a = evaluate_variant(p, "rcp_sq")
    c0 = get_context(0)
    release_context()
    c1 = get_context(0)
    assert c1 is not c0 and not c0._h
    assert _bits_equal(evaluate_variant(p, "rcp_sq"), a)
