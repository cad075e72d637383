"""The B200 GPP evaluation: drop-in for ``rooflab.gpp.kernel``'s seam.

``evaluate_variant(problem, variant)`` has the reference signature and
result type (rooflab/gpp/kernel.py:98-114) but runs the (band, igp, ig, iw)
nest as the sm_100a kernel in libgpp_b200.so.  ``branch_stats`` returns the
kernel's exact near/far counts (kernel.py:130-137) and ``reference_result``
evaluates the literal nest formulation (problem.py:179-208, the ``div``
arithmetic) on the GPU.

``GPPContext`` is the device-buffer manager: one library context per CUDA
device and calling thread; inputs are uploaded once and re-used while the
caller keeps passing the same read-only arrays (the reference marks
synthesized arrays read-only, problem.py:154-155).  Writeable arrays are
re-uploaded on every call.

Reproducibility and concurrency: every evaluation of the same
inputs and variant returns the same bits -- the first call (upload pipelined
with the kernel) and later calls on the resident problem run the same
canonical items and sum them in the same order -- and
independent runs may proceed concurrently: each thread gets its own context
(``get_context``), and a context shared explicitly between threads serialises
its callers (a lock here and one in the library).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib
from .counters import VARIANTS, BranchStats
from .errors import DomainError
from .problem import GPPResult, problem_nw

_ARRAYS = ("wtilde", "i_eps", "aqsntemp", "aqsmtemp", "wx")


def prepare_arrays(problem) -> dict[str, np.ndarray]:
    """Validate a duck-typed GPPProblem and return F-contiguous arrays."""
    nb, ng, nc = int(problem.nbands), int(problem.ngpown), int(problem.ncouls)
    if min(nb, ng, nc) < 1:
        raise DomainError(f"dims must all be at least 1, got {(nb, ng, nc)}")
    want = {
        "wtilde": (nc, ng),
        "i_eps": (nc, ng),
        "aqsntemp": (nc, nb),
        "aqsmtemp": (ng, nb),
    }
    out = {}
    for name, shape in want.items():
        arr = np.asarray(getattr(problem, name))
        if arr.shape != shape:
            raise DomainError(f"{name} has shape {arr.shape}, expected {shape}")
        if arr.dtype != np.complex128 or not arr.flags.f_contiguous:
            arr = np.asfortranarray(arr, dtype=np.complex128)
        out[name] = arr
    nw = problem_nw(problem)
    wx = np.asarray(problem.wx)
    if wx.ndim == 2 and wx.shape != (nw, nb):
        raise DomainError(f"band-indexed wx must have shape ({nw}, {nb}), got {wx.shape}")
    if wx.dtype != np.float64 or not wx.flags.f_contiguous:
        wx = np.asfortranarray(wx, dtype=np.float64)
    out["wx"] = wx
    return out


def _variant_code(variant: str) -> int:
    """Code of a reference variant (div / rcp / rcp_sq) or of one of the
    intermediate ladder kernels ("rcp_sq/split", "rcp_sq/iw")."""
    code = _lib.KERNEL_CODES.get(variant)
    if code is None:
        raise DomainError(f"unknown variant {variant!r}, expected one of {VARIANTS}")
    return code


def _reference_variant(variant: str) -> None:
    if variant not in VARIANTS:
        raise DomainError(f"unknown variant {variant!r}, expected one of {VARIANTS}")


class GPPContext:
    """One libgpp_b200 context (device buffers + stream) on one CUDA device."""

    def __init__(self, device: int = 0):
        self._lib = _lib.load()
        self.device = int(device)
        # Guards the Python-side cache state; the library serialises callers of
        # one context too (gpp_lib.cu CtxLock).
        self.lock = threading.RLock()
        handle = ctypes.c_void_p()
        _lib.check(self._lib.gpp_create(ctypes.byref(handle), self.device), "gpp_create")
        self._h = handle
        self._key = None
        self._keep = None
        self.nw = 0
        self.band_range = (0, 0)
        self.dims = (0, 0, 0)

    # -- lifecycle ---------------------------------------------------------
    def close(self) -> None:
        if self._h:
            self._lib.gpp_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- data --------------------------------------------------------------
    def _make_key(self, problem, arrays, band_range):
        nb = int(problem.nbands)
        b0, b1 = (0, nb) if band_range is None else (int(band_range[0]), int(band_range[1]))
        key = (
            tuple((id(a), a.__array_interface__["data"][0], a.shape) for a in arrays.values()),
            (nb, int(problem.ngpown), int(problem.ncouls)),
            (b0, b1),
        )
        cacheable = all(not a.flags.writeable for a in arrays.values())
        return key, cacheable, (b0, b1)

    def _remember(self, problem, arrays, key, cacheable, br):
        self.nw = int(arrays["wx"].shape[0])
        self.band_range = br
        self.dims = (int(problem.nbands), int(problem.ngpown), int(problem.ncouls))
        self._key = key if cacheable else None
        self._keep = arrays if cacheable else None  # pin ids while cached

    def is_resident(self, problem, band_range: tuple[int, int] | None = None) -> bool:
        """Whether ``problem`` (read-only arrays) is already on the device."""
        arrays = prepare_arrays(problem)
        key, cacheable, _ = self._make_key(problem, arrays, band_range)
        return cacheable and key == self._key

    def upload(self, problem, band_range: tuple[int, int] | None = None, force: bool = False):
        """Copy ``problem`` (or its band shard) to the device unless cached."""
        arrays = prepare_arrays(problem)
        key, cacheable, (b0, b1) = self._make_key(problem, arrays, band_range)
        if not force and cacheable and key == self._key:
            return
        self._key = None
        wx = arrays["wx"]
        _lib.check(
            self._lib.gpp_upload(
                self._h, int(problem.nbands), int(problem.ngpown), int(problem.ncouls), int(wx.shape[0]),
                _lib.dptr(arrays["wtilde"]), _lib.dptr(arrays["i_eps"]),
                _lib.dptr(arrays["aqsntemp"]), _lib.dptr(arrays["aqsmtemp"]),
                _lib.dptr(wx), 1 if wx.ndim == 2 else 0, b0, b1,
            ),
            "gpp_upload",
        )
        self._remember(problem, arrays, key, cacheable, (b0, b1))

    def evaluate_host(self, problem, variant: str = "rcp_sq",
                      band_range: tuple[int, int] | None = None, counts: bool = False,
                      slabs: int = 0):
        """Upload + evaluate with the H2D copy pipelined against the kernel
        (gpp_evaluate_host): (GPPResult, (near, far) | None, device_ms)."""
        code = _variant_code(variant)
        arrays = prepare_arrays(problem)
        key, cacheable, (b0, b1) = self._make_key(problem, arrays, band_range)
        self._key = None
        wx = arrays["wx"]
        nw = int(wx.shape[0])
        ach = np.empty(2 * nw, dtype=np.float64)
        asx = np.empty(2 * nw, dtype=np.float64)
        nf = np.zeros(2, dtype=np.int64)
        ms = ctypes.c_float()
        nf_ptr = nf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) if counts else None
        _lib.check(
            self._lib.gpp_evaluate_host(
                self._h, code, int(problem.nbands), int(problem.ngpown), int(problem.ncouls), nw,
                _lib.dptr(arrays["wtilde"]), _lib.dptr(arrays["i_eps"]),
                _lib.dptr(arrays["aqsntemp"]), _lib.dptr(arrays["aqsmtemp"]),
                _lib.dptr(wx), 1 if wx.ndim == 2 else 0, b0, b1, int(slabs),
                _lib.dptr(ach), _lib.dptr(asx), nf_ptr, ctypes.byref(ms),
            ),
            "gpp_evaluate_host",
        )
        self._remember(problem, arrays, key, cacheable, (b0, b1))
        result = GPPResult(achtemp=ach.view(np.complex128).copy(),
                           asxtemp=asx.view(np.complex128).copy())
        return result, ((int(nf[0]), int(nf[1])) if counts else None), float(ms.value)

    def synth(self, nbands: int, ngpown: int, ncouls: int, seed: int = 42, nw: int = 2,
              band_range: tuple[int, int] | None = None) -> None:
        """Draw synth_problem(nbands, ngpown, ncouls, seed, nw) directly on
        the device (gpp_synth, bit-exact with the host draw; no H2D of the
        arrays).  The device then holds the problem (or its band shard)."""
        from .problem import MAX_NW

        for name, value in (("nbands", nbands), ("ngpown", ngpown), ("ncouls", ncouls)):
            if value < 1:
                raise DomainError(f"{name} must be at least 1, got {value!r}")
        if not 1 <= nw <= MAX_NW:
            raise DomainError(f"nw must be in [1, {MAX_NW}], got {nw!r}")
        b0, b1 = (0, nbands) if band_range is None else (int(band_range[0]), int(band_range[1]))
        rng = np.random.default_rng(seed)
        st = rng.bit_generator.state["state"]
        mask = (1 << 64) - 1
        words = np.array([st["state"] & mask, st["state"] >> 64, st["inc"] & mask, st["inc"] >> 64],
                         dtype=np.uint64)
        # wx is drawn last (problem.py:141): skip the 4 nc ng + 2 nc nb + 2 ng nb array draws.
        rng.bit_generator.advance(4 * ncouls * ngpown + 2 * ncouls * nbands + 2 * ngpown * nbands)
        wx = rng.uniform(1.0, 2.0, size=nw)
        self._key = None
        _lib.check(self._lib.gpp_synth(self._h, int(nbands), int(ngpown), int(ncouls), int(nw),
                                       words.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                       _lib.dptr(wx), b0, b1), "gpp_synth")
        self.nw = int(nw)
        self.band_range = (b0, b1)
        self.dims = (int(nbands), int(ngpown), int(ncouls))
        self.synth_wx = wx

    def run(self, variant: str = "rcp_sq", counts: bool = True):
        """Evaluate the uploaded problem: (GPPResult, (near, far) | None, kernel_ms).

        ``counts=True`` runs the counting kernel (branch statistics as a
        by-product, two predicated integer adds per instance); ``False`` runs
        the production kernel that evaluate_variant uses.
        """
        code = _variant_code(variant)
        if self.nw < 1:
            raise DomainError("no problem uploaded")
        ach = np.empty(2 * self.nw, dtype=np.float64)
        asx = np.empty(2 * self.nw, dtype=np.float64)
        nf = np.zeros(2, dtype=np.int64)
        ms = ctypes.c_float()
        nf_ptr = nf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) if counts else None
        _lib.check(
            self._lib.gpp_run(self._h, code, _lib.dptr(ach), _lib.dptr(asx), nf_ptr, ctypes.byref(ms)),
            "gpp_run",
        )
        result = GPPResult(achtemp=ach.view(np.complex128).copy(),
                           asxtemp=asx.view(np.complex128).copy())
        return result, ((int(nf[0]), int(nf[1])) if counts else None), float(ms.value)

    def run_factored(self, variant: str = "rcp_sq", counts: bool = True):
        """The reference's factored algorithm on the device (one fused repo kernel)
        (gpp_run_factored): (GPPResult, (near, far) | None, device_ms).
        Band-invariant wx only; a different algorithm from run()."""
        _reference_variant(variant)
        if self.nw < 1:
            raise DomainError("no problem uploaded")
        ach = np.empty(2 * self.nw, dtype=np.float64)
        asx = np.empty(2 * self.nw, dtype=np.float64)
        nf = np.zeros(2, dtype=np.int64)
        ms = ctypes.c_float()
        nf_ptr = nf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) if counts else None
        _lib.check(self._lib.gpp_run_factored(self._h, _variant_code(variant), _lib.dptr(ach),
                                              _lib.dptr(asx), nf_ptr, ctypes.byref(ms)),
                   "gpp_run_factored")
        result = GPPResult(achtemp=ach.view(np.complex128).copy(),
                           asxtemp=asx.view(np.complex128).copy())
        return result, ((int(nf[0]), int(nf[1])) if counts else None), float(ms.value)

    def time(self, variant: str = "rcp_sq", iters: int = 10) -> tuple[float, float]:
        """Device-resident timing of ``iters`` evaluations: (total_ms, main_kernel_ms)."""
        tot, main = ctypes.c_float(), ctypes.c_float()
        _lib.check(self._lib.gpp_time(self._h, _variant_code(variant), int(iters),
                                      ctypes.byref(tot), ctypes.byref(main)), "gpp_time")
        return float(tot.value), float(main.value)

    def launch_count(self) -> int:
        """Kernels this context has launched so far (gpp_launch_count)."""
        n = ctypes.c_int64(0)
        _lib.check(self._lib.gpp_launch_count(self._h, ctypes.byref(n)), "gpp_launch_count")
        return int(n.value)

    def kernel_info(self, variant: str = "rcp_sq") -> dict:
        vals = [ctypes.c_int32() for _ in range(6)]
        _lib.check(self._lib.gpp_kernel_info(self._h, _variant_code(variant),
                                             *[ctypes.byref(v) for v in vals]), "gpp_kernel_info")
        keys = ("registers_per_thread", "threads_per_block", "blocks_per_sm", "grid",
                "igp_tile", "band_chunk")
        return {k: int(v.value) for k, v in zip(keys, vals)}

    def comm_init(self, nranks: int, rank: int, unique_id: bytes) -> None:
        if len(unique_id) != 128:
            raise DomainError("NCCL unique id must be 128 bytes")
        _lib.check(self._lib.gpp_comm_init(self._h, int(nranks), int(rank), unique_id),
                   "gpp_comm_init")


def comm_unique_id() -> bytes:
    lib = _lib.load()
    buf = ctypes.create_string_buffer(128)
    _lib.check(lib.gpp_comm_unique_id(buf), "gpp_comm_unique_id")
    return buf.raw


_TLS = threading.local()


def get_context(device: int = 0) -> GPPContext:
    """The calling thread's context on ``device`` (created on first use).
    Per-thread contexts let independent runs proceed concurrently
     without sharing device buffers."""
    ctxs = getattr(_TLS, "contexts", None)
    if ctxs is None:
        ctxs = _TLS.contexts = {}
    ctx = ctxs.get(device)
    if ctx is None:
        ctx = ctxs[device] = GPPContext(device)
    return ctx


def release_context(device: int | None = None) -> None:
    """Free the calling thread's context(s) (device buffers, streams) now
    instead of at thread exit -- e.g. in long-lived pool threads that are
    done with a large problem.  ``device=None``: every device."""
    ctxs = getattr(_TLS, "contexts", None) or {}
    for d in ([device] if device is not None else list(ctxs)):
        ctx = ctxs.pop(d, None)
        if ctx is not None:
            with ctx.lock:
                ctx.close()


def evaluate(problem, variant: str = "rcp_sq", device: int = 0, counts: bool = True):
    """Upload (cached) + run: (GPPResult, BranchStats | None, kernel_ms).
    The first sight of a problem pipelines its upload with the evaluation
    (gpp_evaluate_host); both paths return the same bits."""
    ctx = get_context(device)
    with ctx.lock:
        if ctx.is_resident(problem):
            result, nf, ms = ctx.run(variant, counts=counts)
        else:
            result, nf, ms = ctx.evaluate_host(problem, variant, counts=counts)
    stats = None
    if nf is not None:
        nb, ng, nc = ctx.dims
        stats = BranchStats(instances=ctx.nw * nb * ng * nc, near=nf[0], far=nf[1])
    return result, stats, ms


def evaluate_variant(problem, variant: str, device: int = 0) -> GPPResult:
    """Drop-in for rooflab.gpp.kernel.evaluate_variant (kernel.py:98-114)."""
    _reference_variant(variant)
    return evaluate(problem, variant, device, counts=False)[0]


def branch_stats(problem, variant: str, device: int = 0) -> BranchStats:
    """Drop-in for rooflab.gpp.kernel.branch_stats (kernel.py:130-137)."""
    _reference_variant(variant)
    return evaluate(problem, variant, device)[1]


def reference_result(problem, device: int = 0) -> GPPResult:
    """The literal-nest formulation (problem.py:179-208: library complex
    division and magnitude predicates) evaluated per instance on the GPU."""
    return evaluate(problem, "div", device, counts=False)[0]


class VariantTerms:
    """Per-(iw, ig, igp) branch terms (rooflab/gpp/kernel.py:48-60)."""

    def __init__(self, sch, ssx, near, far):
        self.sch, self.ssx, self.near, self.far = sch, ssx, near, far


def variant_terms(problem, variant: str, device: int = 0) -> VariantTerms:
    """Drop-in for rooflab.gpp.kernel.variant_terms (kernel.py:63-95),
    computed on the GPU; arrays of shape (nw, ncouls, ngpown)."""
    _reference_variant(variant)
    ctx = get_context(device)
    with ctx.lock:
        return _variant_terms(ctx, problem, variant)


def _variant_terms(ctx, problem, variant):
    ctx.upload(problem)
    nw, nc, ng = ctx.nw, int(problem.ncouls), int(problem.ngpown)
    sch = np.empty((nw, nc, ng), dtype=np.complex128)
    ssx = np.empty((nw, nc, ng), dtype=np.complex128)
    near = np.empty((nw, nc, ng), dtype=np.uint8)
    far = np.empty((nw, nc, ng), dtype=np.uint8)
    u8 = ctypes.POINTER(ctypes.c_uint8)
    _lib.check(ctx._lib.gpp_variant_terms(ctx._h, _variant_code(variant),
                                          sch.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                          ssx.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                          near.ctypes.data_as(u8), far.ctypes.data_as(u8)),
               "gpp_variant_terms")
    return VariantTerms(sch, ssx, near.astype(bool), far.astype(bool))


def complex_reciprocal(z):
    """1/z as conj(z) / |z|^2 (rooflab/gpp/kernel.py:33-45); host-side helper."""
    from .problem import TOL_ZERO

    arr = np.asarray(z)
    denom = arr.real * arr.real + arr.imag * arr.imag
    if np.any(denom <= TOL_ZERO * TOL_ZERO):
        raise DomainError("complex_reciprocal: input magnitude at or below tol_zero")
    out = np.conj(arr) * (1.0 / denom)
    return out if isinstance(z, np.ndarray) else complex(out)


def evaluate_factored(problem, variant: str = "rcp_sq", device: int = 0) -> GPPResult:
    """The reference's production algorithm (kernel.py:98-114: the GEMM of the
    band weights, then the branch terms) on the GPU.  Time-to-solution path
    for band-invariant wx; evaluate_variant runs the per-instance nest."""
    _reference_variant(variant)
    ctx = get_context(device)
    with ctx.lock:
        ctx.upload(problem)
        return ctx.run_factored(variant, counts=False)[0]


def plan_schedule(nbands: int, ngpown: int, ncouls: int, nw: int, sms: int = 148) -> list[dict]:
    """The production kernel's canonical launches for a whole evaluation
    (first frequency group) on a GPU with ``sms`` SMs (gpp_plan; host logic
    only, no GPU needed): band windows, whole-wave launches and balanced
    tails, and the igp tile chosen for ngpown."""
    lib = _lib.load()
    n = ctypes.c_int32(0)
    _lib.check(lib.gpp_plan(nbands, ngpown, ncouls, nw, sms, 0, ctypes.byref(n), None), "gpp_plan")
    out = np.zeros((max(n.value, 1), 7), dtype=np.int64)
    _lib.check(lib.gpp_plan(nbands, ngpown, ncouls, nw, sms, n.value, ctypes.byref(n),
                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))), "gpp_plan")
    keys = ("row0", "n_rows", "band0", "nbands", "bchunk", "n_items", "igp_tile")
    return [dict(zip(keys, (int(v) for v in row))) for row in out[: n.value]]


def plan_piece(nbands: int, ngpown: int, ncouls: int, nw: int, blk0: int, blk1: int,
               sms: int = 148) -> list[dict]:
    """The production kernel's sub-launches for the ig slab [blk0, blk1) of
    the pipelined evaluate (gpp_plan_piece; host logic only), with the
    canonical slot mapping of their items."""
    lib = _lib.load()
    n = ctypes.c_int32(0)
    _lib.check(lib.gpp_plan_piece(nbands, ngpown, ncouls, nw, sms, blk0, blk1, 0, ctypes.byref(n), None),
               "gpp_plan_piece")
    out = np.zeros((max(n.value, 1), 9), dtype=np.int64)
    _lib.check(lib.gpp_plan_piece(nbands, ngpown, ncouls, nw, sms, blk0, blk1, n.value, ctypes.byref(n),
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))), "gpp_plan_piece")
    keys = ("row0", "n_rows", "band0", "nbands", "bchunk", "n_items", "igp_tile", "slot_base", "slot_stride")
    return [dict(zip(keys, (int(v) for v in row))) for row in out[: n.value]]


def fp64_peak(device: int = 0, iters: int = 200_000) -> tuple[float, float]:
    """Measured FP64 DFMA throughput of the device: (TFLOP/s, ms)."""
    lib = _lib.load()
    tf, ms = ctypes.c_double(), ctypes.c_float()
    _lib.check(lib.gpp_fp64_peak(int(device), int(iters), ctypes.byref(tf), ctypes.byref(ms)),
               "gpp_fp64_peak")
    return float(tf.value), float(ms.value)
