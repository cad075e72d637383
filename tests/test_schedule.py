"""The production kernel's launch schedule (csrc/gpp_lib.cu: window_launches,
split_tail, choose_bchunk) through gpp_plan -- host logic, no GPU needed.

Every (row, band) pair of the problem -- a row being one (256-ig block, igp
tile) -- must be covered by exactly one item of exactly one launch: the whole
waves of each band window plus its balanced tail.  The band windows must fit
the kernel's by-value wx table (kWxParam = 1536 doubles)."""
import numpy as np
import pytest

from paper_2008_11326_b200.kernel import plan_schedule

K_WX_PARAM = 1536


def _coverage(nbands, ngpown, ncouls, nw, sms):
    plan = plan_schedule(nbands, ngpown, ncouls, nw, sms)
    igp_tile = plan[0]["igp_tile"]
    assert all(L["igp_tile"] == igp_tile for L in plan)
    assert igp_tile == 3 if nw == 1 else igp_tile in (2, 3, 4)
    n_rows = -(-ncouls // 256) * -(-ngpown // igp_tile)
    cov = np.zeros((n_rows, nbands), dtype=np.int32)
    for L in plan:
        assert 0 <= L["band0"] and L["band0"] + L["nbands"] <= nbands
        assert L["nbands"] * min(nw, 3) <= K_WX_PARAM
        assert 1 <= L["bchunk"] <= (256 if nw == 1 else 512)
        k = np.arange(L["n_items"])
        chunk, row = k // L["n_rows"], L["row0"] + k % L["n_rows"]
        assert row.max(initial=0) < n_rows
        b0 = L["band0"] + chunk * L["bchunk"]
        b1 = np.minimum(b0 + L["bchunk"], L["band0"] + L["nbands"])
        assert np.all(b1 > b0)
        for r, lo, hi in zip(row, b0, b1):
            cov[r, lo:hi] += 1
    return plan, cov


def test_paper_size_schedule():
    """(512, 66, 32768) at nw 3 on 148 SMs: 3-igp tiles (no padding, one CTA
    per SM: 148 resident CTAs), 19 whole waves of 512-band items (one per
    (igb, igp tile) row), then the last wave's 4 rows in 14-band chunks."""
    plan = plan_schedule(512, 66, 32768, 3, 148)
    assert plan == [
        {"row0": 0, "n_rows": 2816, "band0": 0, "nbands": 512, "bchunk": 512, "n_items": 19 * 148,
         "igp_tile": 3},
        {"row0": 2816 - 4, "n_rows": 4, "band0": 0, "nbands": 512, "bchunk": 14, "n_items": 4 * 37,
         "igp_tile": 3},
    ]


@pytest.mark.parametrize("ngpown,nw,tile", [
    (16, 3, 4), (33, 3, 3), (66, 3, 3), (132, 3, 4), (264, 3, 4), (528, 3, 4),
    (16, 2, 4), (33, 2, 3), (66, 2, 4), (528, 2, 4), (5, 2, 3), (7, 3, 4), (1, 3, 2), (66, 1, 3),
])
def test_igp_tile_choice(ngpown, nw, tile):
    """The production kernel's igp tile: least padded cost, weighted by the
    measured per-column time of each instantiation (tools/probe_variants_sweep.py
    picks the same tile at every sweep point)."""
    assert plan_schedule(512, ngpown, 8192, nw, 148)[0]["igp_tile"] == tile


@pytest.mark.parametrize("dims,nw,sms", [
    ((512, 66, 32768), 3, 148),
    ((64, 66, 32768), 3, 148),     # 8-way band shard of the paper size
    ((600, 7, 5000), 3, 148),      # two band windows
    ((1100, 5, 3000), 2, 148),
    ((1600, 4, 2000), 1, 148),
    ((258, 33, 8192), 3, 148),     # 2-band last chunk
    ((5, 7, 70000), 3, 148),
    ((1, 1, 1), 3, 148),
    ((300, 9, 20000), 2, 50),      # other SM counts
])
def test_every_instance_is_scheduled_exactly_once(dims, nw, sms):
    _, cov = _coverage(*dims, nw, sms)
    assert cov.min() == 1 and cov.max() == 1


def test_random_schedules_cover_exactly_once():
    rng = np.random.default_rng(0)
    for _ in range(25):
        nbands = int(rng.integers(1, 700))
        ngpown = int(rng.integers(1, 40))
        ncouls = int(rng.integers(1, 20000))
        nw = int(rng.integers(1, 5))
        sms = int(rng.integers(1, 200))
        _, cov = _coverage(nbands, ngpown, ncouls, nw, sms)
        assert cov.min() == 1 and cov.max() == 1, (nbands, ngpown, ncouls, nw, sms)


def test_tail_only_when_it_shortens_the_modelled_makespan():
    # A problem whose items are an exact multiple of the resident CTAs has
    # no partial wave, hence no tail launch.
    plan = plan_schedule(256, 2, 296 * 256, 3, 148)
    assert plan[0]["igp_tile"] == 2 and len(plan) == 1 and plan[0]["n_items"] % 296 == 0


def _items(L, slot_of):
    """(slot -> (row, band0, band1)) of one launch's items."""
    k = np.arange(L["n_items"])
    chunk, row = k // L["n_rows"], L["row0"] + k % L["n_rows"]
    b0 = L["band0"] + chunk * L["bchunk"]
    b1 = np.minimum(b0 + L["bchunk"], L["band0"] + L["nbands"])
    return dict(zip(slot_of(chunk, row, k).tolist(), zip(row.tolist(), b0.tolist(), b1.tolist())))


def _canonical_items(dims, nw, sms):
    out, slot0 = {}, 0
    for L in plan_schedule(*dims, nw, sms):
        out.update(_items(L, lambda c, r, k, s0=slot0: s0 + k))
        slot0 += L["n_items"]
    return out


@pytest.mark.parametrize("dims,nw", [((512, 66, 32768), 3), ((64, 66, 32768), 3), ((600, 7, 5000), 3),
                                     ((1100, 5, 3000), 2), ((300, 10, 3000), 1), ((512, 16, 8192), 3)])
def test_slab_pieces_run_the_canonical_items(dims, nw):
    """The basis of bitwise reproducibility: however the ig
    blocks are cut into slabs for the pipelined evaluate, the slabs' launches
    run exactly the canonical items -- the same (row, band range) -- each
    writing its canonical slot, so the slot-order finalize sums the same
    values in the same order as the resident run."""
    from paper_2008_11326_b200.kernel import plan_piece

    canon = _canonical_items(dims, nw, 148)
    n_blk = -(-dims[2] // 256)
    rng = np.random.default_rng(sum(dims) + nw)
    for trial in range(4):
        cuts = sorted(set(rng.integers(1, max(n_blk, 2), size=min(6, n_blk)).tolist()) - {0, n_blk})
        bounds = [0, *cuts, n_blk] if trial else [0, n_blk]
        got = {}
        for b0, b1 in zip(bounds[:-1], bounds[1:]):
            for L in plan_piece(*dims, nw, b0, b1, 148):
                items = _items(L, lambda c, r, k, L=L: L["slot_base"] + c * L["slot_stride"] + r)
                assert not set(items) & set(got), "a slot written twice"
                got.update(items)
        assert got == canon, (bounds, len(got), len(canon))
