"""Band sharding across ranks on CPU: world_size 2 with the gloo backend.

Each rank evaluates its band shard with the oracle (the GPU path runs the
same partition through gpp_upload's band range), the partial achtemp /
asxtemp and near/far counts are summed with an all_reduce -- the host-side
mirror of the library's single ncclAllReduce -- and must equal the whole
problem's result.  No GPU needed.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from paper_2008_11326_b200.dist import band_range, shard_problem
from paper_2008_11326_b200.problem import GPPProblem, synth_problem


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, seed, nw, band_wx, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import gpp_oracle as orc

        p = _problem(dims, seed, nw, band_wx)
        b0, b1 = band_range(p.nbands, world, rank)
        part = shard_problem(p, b0, b1)
        r = orc.evaluate_variant(part, "rcp_sq")
        _, near, far = orc.branch_stats(part, "rcp_sq")
        vec = torch.tensor(np.concatenate([r.achtemp.view(np.float64), r.asxtemp.view(np.float64)]),
                           dtype=torch.float64)
        cnt = torch.tensor([near, far], dtype=torch.int64)
        tdist.all_reduce(vec)
        tdist.all_reduce(cnt)
        if rank == 0:
            out.put((vec.numpy().copy(), cnt.numpy().copy()))
    finally:
        tdist.destroy_process_group()


def _problem(dims, seed, nw, band_wx):
    p = synth_problem(*dims, seed=seed, nw=nw)
    if not band_wx:
        return p
    rng = np.random.default_rng(9)
    wxb = np.asfortranarray(rng.uniform(1.0, 2.0, size=(nw, dims[0])))
    return GPPProblem(*dims, p.wtilde, p.i_eps, p.aqsntemp, p.aqsmtemp, wxb)


@pytest.mark.parametrize("dims,seed,nw,band_wx", [
    ((17, 5, 96), 1, 3, False),
    ((8, 8, 64), 7, 2, True),
])
def test_two_rank_band_shards_reduce_to_whole(dims, seed, nw, band_wx):
    from oracle import gpp_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, seed, nw, band_wx, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    vec, cnt = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    whole = orc.evaluate_variant(_problem(dims, seed, nw, band_wx), "rcp_sq")
    _, near, far = orc.branch_stats(_problem(dims, seed, nw, band_wx), "rcp_sq")
    got = vec.view(np.complex128)
    np.testing.assert_allclose(got[:nw], whole.achtemp, rtol=1e-12)
    np.testing.assert_allclose(got[nw:], whole.asxtemp, rtol=1e-12)
    assert list(cnt) == [near, far]


@pytest.mark.parametrize("nbands,world", [(512, 1), (512, 2), (512, 8), (7, 3), (3, 8)])
def test_band_range_partitions(nbands, world):
    ranges = [band_range(nbands, world, r) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == nbands
    for (a0, a1), (c0, _) in zip(ranges, ranges[1:]):
        assert a1 == c0
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        band_range(nbands, world, world)


def test_shard_views_are_contiguous_columns():
    p = synth_problem(10, 3, 32, seed=2)
    s = shard_problem(p, 4, 7)
    assert s.nbands == 3 and s.aqsntemp.flags.f_contiguous and s.aqsmtemp.flags.f_contiguous
    assert np.shares_memory(s.aqsntemp, p.aqsntemp)
