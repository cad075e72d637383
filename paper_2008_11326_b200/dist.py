"""Band (n1) sharding across GPUs: one process per GPU.

SURVEY.md section 8e: the band sum is an independent reduction, so rank r
evaluates the contiguous band range [b0, b1) (its columns of aqsntemp and
aqsmtemp are one contiguous slice each in F-order), wtilde / i_eps / wx are
replicated, and the per-rank partial achtemp / asxtemp and branch counts
(4*nw doubles + 2 integers) are combined by ONE ncclAllReduce issued by the
library on its own stream right after the finalize kernel (gpp_run /
gpp_time, csrc/gpp_lib.cu).  torch.distributed is only the bootstrap that
broadcasts the 128-byte NCCL unique id.
"""

from __future__ import annotations

import numpy as np

from .kernel import GPPContext, comm_unique_id
from .problem import GPPProblem


def band_range(nbands: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced band shard [b0, b1) of ``rank`` (first ranks take
    the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    base, extra = divmod(int(nbands), world)
    b0 = rank * base + min(rank, extra)
    return b0, b0 + base + (1 if rank < extra else 0)


def shard_problem(problem, b0: int, b1: int) -> GPPProblem:
    """The band shard [b0, b1) of a problem as its own GPPProblem (views).

    Used by the CPU tests to check the partition against the oracle; the GPU
    path passes the whole arrays plus the range to gpp_upload instead.
    """
    wx = np.asarray(problem.wx)
    if wx.ndim == 2:
        wx = wx[:, b0:b1]
    return GPPProblem(
        nbands=b1 - b0,
        ngpown=problem.ngpown,
        ncouls=problem.ncouls,
        wtilde=problem.wtilde,
        i_eps=problem.i_eps,
        aqsntemp=problem.aqsntemp[:, b0:b1],
        aqsmtemp=problem.aqsmtemp[:, b0:b1],
        wx=wx,
        seed=getattr(problem, "seed", None),
    )


class ShardedGPP:
    """One rank of a band-sharded evaluation (its GPU context + NCCL comm)."""

    def __init__(self, device: int, rank: int, world: int, unique_id: bytes | None):
        self.rank, self.world = int(rank), int(world)
        self.ctx = GPPContext(device)
        if self.world > 1:
            if unique_id is None:
                raise ValueError("a NCCL unique id is required for world > 1")
            self.ctx.comm_init(self.world, self.rank, unique_id)

    @classmethod
    def from_torch(cls, device: int) -> "ShardedGPP":
        """Bootstrap from an initialised torch.distributed process group."""
        import torch.distributed as tdist

        world, rank = tdist.get_world_size(), tdist.get_rank()
        obj = [comm_unique_id() if rank == 0 else None]
        if world > 1:
            tdist.broadcast_object_list(obj, src=0)
        return cls(device, rank, world, obj[0])

    def band_range(self, nbands: int) -> tuple[int, int]:
        return band_range(nbands, self.world, self.rank)

    def upload(self, problem, force: bool = False) -> None:
        self.ctx.upload(problem, self.band_range(int(problem.nbands)), force=force)

    def run(self, variant: str = "rcp_sq", counts: bool = True):
        """Evaluate this rank's shard; the result is the all-rank total."""
        return self.ctx.run(variant, counts=counts)

    def evaluate(self, problem, variant: str = "rcp_sq", counts: bool = False):
        """End to end from host arrays: this rank uploads its band shard of
        aqsntemp / aqsmtemp and 1/N of the igp columns of wtilde / i_eps, the
        columns are broadcast over NVLink, the shard is evaluated pipelined
        with its upload, and the partials are all-reduced (gpp_evaluate_host
        with the communicator attached): (total GPPResult, (near, far) | None,
        device ms)."""
        return self.ctx.evaluate_host(problem, variant, band_range=self.band_range(int(problem.nbands)),
                                      counts=counts)

    def close(self) -> None:
        self.ctx.close()


class MultiDeviceGPP:
    """Single-process band sharding over several local GPUs (SURVEY.md
    section 2, native component 3): one context per device in one NCCL clique
    (ncclCommInitAll), every shard launched from this thread, one grouped
    ncclAllReduce of the partials (gpp_run_group)."""

    def __init__(self, devices):
        import ctypes

        from . import _lib

        self.devices = [int(d) for d in devices]
        if not self.devices or len(set(self.devices)) != len(self.devices):
            raise ValueError("devices must be a non-empty list of distinct device ids")
        self._lib = _lib.load()
        self.ctxs = [GPPContext(d) for d in self.devices]
        self._arr = (ctypes.c_void_p * len(self.ctxs))(*[c._h.value for c in self.ctxs])
        _lib.check(self._lib.gpp_comm_init_all(self._arr, len(self.ctxs)), "gpp_comm_init_all")

    def upload(self, problem, force: bool = False) -> None:
        n = len(self.ctxs)
        for rank, ctx in enumerate(self.ctxs):
            ctx.upload(problem, band_range(int(problem.nbands), n, rank), force=force)

    def synth(self, nbands: int, ngpown: int, ncouls: int, seed: int = 42, nw: int = 2) -> None:
        """Draw every device's band shard of synth_problem on that device."""
        n = len(self.ctxs)
        for rank, ctx in enumerate(self.ctxs):
            ctx.synth(nbands, ngpown, ncouls, seed=seed, nw=nw,
                      band_range=band_range(nbands, n, rank))

    def time(self, variant: str = "rcp_sq", iters: int = 10) -> tuple[float, float]:
        """Device-resident timing of ``iters`` group evaluations (each with its
        grouped allreduce, no host sync in between; gpp_time_group):
        (slowest device total ms, slowest device summed main-kernel ms)."""
        import ctypes

        from . import _lib
        from .kernel import _variant_code

        tot, main = ctypes.c_float(), ctypes.c_float()
        _lib.check(self._lib.gpp_time_group(self._arr, len(self.ctxs), _variant_code(variant), int(iters),
                                            ctypes.byref(tot), ctypes.byref(main)), "gpp_time_group")
        return float(tot.value), float(main.value)

    def evaluate(self, problem, variant: str = "rcp_sq"):
        """End to end from host arrays on every device at once: one thread per
        device runs gpp_evaluate_host on its band shard (column-split
        wtilde / i_eps upload + NCCL broadcast, allreduce of the partials).
        Returns (total GPPResult, slowest device ms)."""
        import threading

        n = len(self.ctxs)
        out: list = [None] * n
        errs: list = []

        def work(rank):
            try:
                out[rank] = self.ctxs[rank].evaluate_host(
                    problem, variant, band_range=band_range(int(problem.nbands), n, rank))
            except Exception as e:  # noqa: BLE001 -- re-raised below
                errs.append(e)

        ts = [threading.Thread(target=work, args=(r,)) for r in range(n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]
        return out[0][0], max(o[2] for o in out)

    def run(self, variant: str = "rcp_sq", counts: bool = True):
        """(GPPResult, (near, far) | None, slowest-device kernel ms) of the whole problem."""
        import ctypes

        from . import _lib
        from .kernel import _variant_code
        from .problem import GPPResult

        nw = self.ctxs[0].nw
        ach = np.empty(2 * nw)
        asx = np.empty(2 * nw)
        nf = np.zeros(2, dtype=np.int64)
        ms = ctypes.c_float()
        nf_ptr = nf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) if counts else None
        _lib.check(self._lib.gpp_run_group(self._arr, len(self.ctxs), _variant_code(variant),
                                           _lib.dptr(ach), _lib.dptr(asx), nf_ptr, ctypes.byref(ms)),
                   "gpp_run_group")
        result = GPPResult(achtemp=ach.view(np.complex128).copy(), asxtemp=asx.view(np.complex128).copy())
        return result, ((int(nf[0]), int(nf[1])) if counts else None), float(ms.value)

    def close(self) -> None:
        for c in self.ctxs:
            c.close()
