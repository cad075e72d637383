"""The C ABI without a GPU: the library loads, exports every symbol the header
declares, and validates arguments before touching CUDA.  Also the host-side
mirror of the reference interface (validation, errors, golden I/O)."""

import ctypes
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2008_11326_b200 import _lib
from paper_2008_11326_b200.errors import DomainError, GPUError, RooflabError, SynthesisError
from paper_2008_11326_b200.kernel import prepare_arrays
from paper_2008_11326_b200.problem import (
    GPPProblem,
    check_branch_safety,
    load_golden,
    max_rel_error,
    save_golden,
    synth_problem,
)

HEADER = ROOT / "include" / "gpp_b200.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gpp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_what_the_shim_binds():
    assert header_functions() == sorted(_lib.SIGNATURES)


def test_library_exports_every_symbol():
    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (gpp_\w+)", out))
    for name in header_functions():
        assert name in exported, name
        assert getattr(lib, name) is not None
    assert lib.gpp_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def _ctx():
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.gpp_create(ctypes.byref(h), 0) == 0
    return lib, h


def test_argument_validation_without_gpu():
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.gpp_create(ctypes.byref(h), -1) == _lib.GPP_ERR_ARG
    assert b"device" in lib.gpp_last_error()
    lib, h = _ctx()
    try:
        z = np.zeros(8)
        p = _lib.dptr(z)
        # dims
        assert lib.gpp_upload(h, 0, 1, 1, 2, p, p, p, p, p, 0, 0, 1) == _lib.GPP_ERR_ARG
        # nw
        assert lib.gpp_upload(h, 1, 1, 1, 0, p, p, p, p, p, 0, 0, 1) == _lib.GPP_ERR_ARG
        # null pointer
        assert lib.gpp_upload(h, 1, 1, 1, 2, None, p, p, p, p, 0, 0, 1) == _lib.GPP_ERR_ARG
        # band range (an empty shard [3, 3) is valid: more ranks than bands)
        assert lib.gpp_upload(h, 4, 1, 1, 2, p, p, p, p, p, 0, 3, 2) == _lib.GPP_ERR_ARG
        assert lib.gpp_upload(h, 4, 1, 1, 2, p, p, p, p, p, 0, 0, 5) == _lib.GPP_ERR_ARG
        assert lib.gpp_upload(h, 4, 1, 1, 2, p, p, p, p, p, 0, -1, 2) == _lib.GPP_ERR_ARG
        # run before upload / bad variant
        out = np.zeros(4)
        assert lib.gpp_run(h, 2, _lib.dptr(out), _lib.dptr(out), None, None) == _lib.GPP_ERR_ARG
        assert lib.gpp_run(h, 7, _lib.dptr(out), _lib.dptr(out), None, None) == _lib.GPP_ERR_ARG
        assert b"variant" in lib.gpp_last_error()
        assert lib.gpp_time(h, 2, 0, None, None) == _lib.GPP_ERR_ARG
        assert lib.gpp_comm_init(h, 2, 2, b"\0" * 128) == _lib.GPP_ERR_ARG
    finally:
        lib.gpp_destroy(h)
    lib.gpp_destroy(None)  # no-op


@pytest.mark.skipif(
    __import__("os").path.exists("/dev/nvidiactl"), reason="checks the no-device failure path"
)
def test_no_device_fails_loudly():
    """Without a GPU there is no fallback: valid calls fail with GPP_ERR_CUDA."""
    lib, h = _ctx()
    try:
        z = np.zeros(8)
        p = _lib.dptr(z)
        assert lib.gpp_upload(h, 1, 1, 1, 2, p, p, p, p, p, 0, 0, 1) == _lib.GPP_ERR_CUDA
        assert len(lib.gpp_last_error()) > 0
    finally:
        lib.gpp_destroy(h)
    from paper_2008_11326_b200 import evaluate_variant

    with pytest.raises(GPUError):
        evaluate_variant(synth_problem(2, 2, 16, seed=5), "rcp_sq")


def test_status_mapping():
    with pytest.raises(DomainError):
        _lib.check(_lib.GPP_ERR_ARG)
    for code in (_lib.GPP_ERR_CUDA, _lib.GPP_ERR_NCCL, _lib.GPP_ERR_OOM):
        with pytest.raises(GPUError) as ei:
            _lib.check(code)
        assert ei.value.status == code
        assert isinstance(ei.value, RooflabError)


def test_prepare_arrays_validation_and_layout():
    p = synth_problem(3, 2, 16, seed=5)
    arrs = prepare_arrays(p)
    for name in ("wtilde", "i_eps", "aqsntemp", "aqsmtemp"):
        assert arrs[name].flags.f_contiguous and arrs[name].dtype == np.complex128
        assert arrs[name] is getattr(p, name)  # no copy for conforming input
    # C-order input is converted, values preserved
    q = GPPProblem(3, 2, 16, np.ascontiguousarray(p.wtilde), p.i_eps, p.aqsntemp, p.aqsmtemp, p.wx)
    a2 = prepare_arrays(q)
    assert a2["wtilde"].flags.f_contiguous and np.array_equal(a2["wtilde"], p.wtilde)
    bad = GPPProblem(3, 2, 16, p.wtilde[:8], p.i_eps, p.aqsntemp, p.aqsmtemp, p.wx)
    with pytest.raises(DomainError):
        prepare_arrays(bad)
    badwx = GPPProblem(3, 2, 16, p.wtilde, p.i_eps, p.aqsntemp, p.aqsmtemp, np.ones((2, 4)))
    with pytest.raises(DomainError):
        prepare_arrays(badwx)
    okwx = GPPProblem(3, 2, 16, p.wtilde, p.i_eps, p.aqsntemp, p.aqsmtemp, np.ones((3, 3)))
    assert prepare_arrays(okwx)["wx"].shape == (3, 3)


def test_problem_api_mirror():
    p = synth_problem(2, 3, 16, seed=5)
    assert p.dims == (2, 3, 16) and p.tuples == 96 and p.nw == 2
    assert p.footprint_bytes() == 16 * (2 * 16 * 3 + 16 * 2 + 3 * 2)
    with pytest.raises(ValueError):
        p.wtilde[0, 0] = 0.0
    with pytest.raises(DomainError):
        synth_problem(0, 4, 32)
    a, b = synth_problem(4, 4, 32, seed=9), synth_problem(4, 4, 32, seed=9)
    assert np.array_equal(a.wtilde, b.wtilde)
    three = synth_problem(4, 4, 32, seed=9, nw=3)
    assert np.array_equal(three.wx[:2], a.wx)


def test_margin_rejection():
    """test_gpp.py:339-357 restated."""
    base = synth_problem(2, 2, 4, seed=5)
    wt = np.array(base.wtilde, order="F")
    wt[0, 0] = base.wx[0] - 0.5
    rigged = GPPProblem(2, 2, 4, wt, base.i_eps, base.aqsntemp, base.aqsmtemp, base.wx)
    with pytest.raises(SynthesisError, match="cutoff"):
        check_branch_safety(rigged)


def test_golden_roundtrip_and_max_rel_error(tmp_path):
    dims, seed, g = load_golden(ROOT / "tests" / "golden" / "gpp-golden-seed42-64x64x512.json")
    save_golden(dims, seed, g, tmp_path / "g.json")
    d2, s2, g2 = load_golden(tmp_path / "g.json")
    assert (d2, s2) == (dims, seed) and max_rel_error(g2, g) == 0.0
    zero = type(g)(achtemp=np.zeros(2, complex), asxtemp=np.zeros(2, complex))
    with pytest.raises(DomainError):
        max_rel_error(g, zero)


def test_complex_reciprocal_mirror():
    """kernel.py:33-45 mirror: test_gpp.py:164-184 restated."""
    from paper_2008_11326_b200 import complex_reciprocal

    rng = np.random.default_rng(5)
    z = rng.uniform(0.1, 10.0, 100_000) * np.exp(1j * rng.uniform(0.0, 2 * np.pi, 100_000))
    rel = np.abs(complex_reciprocal(z) - 1.0 / z) / np.abs(1.0 / z)
    assert float(rel.max()) <= 4 * np.finfo(np.float64).eps
    with pytest.raises(DomainError):
        complex_reciprocal(0j)
    assert complex_reciprocal(2 + 0j) == 0.5 + 0j
