"""ctypes binding of libgpp_b200.so (C ABI: include/gpp_b200.h).

The library is built in-tree (paper_2008_11326_b200/lib/libgpp_b200.so) by
``__graft_entry__.build()`` / ``make -C paper_2008_11326_b200/csrc``.  There is
no fallback: if the shared object is missing, ``load()`` raises GPUError.
ctypes releases the GIL for the duration of every call.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import DomainError, GPUError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libgpp_b200.so"

GPP_OK, GPP_ERR_ARG, GPP_ERR_CUDA, GPP_ERR_NCCL, GPP_ERR_OOM = 0, 1, 2, 3, 4
VARIANT_CODES = {"div": 0, "rcp": 1, "rcp_sq": 2}
# Intermediate rcp_sq kernels of the version ladder (include/gpp_b200.h).
KERNEL_CODES = {**VARIANT_CODES, "rcp_sq/split": 3, "rcp_sq/iw": 4, "rcp_sq/seed": 5}

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_i64_p = ctypes.POINTER(ctypes.c_int64)
_c_i32_p = ctypes.POINTER(ctypes.c_int32)
_c_float_p = ctypes.POINTER(ctypes.c_float)

# name -> (restype, argtypes); every symbol include/gpp_b200.h declares.
SIGNATURES = {
    "gpp_abi_version": (ctypes.c_int, []),
    "gpp_last_error": (ctypes.c_char_p, []),
    "gpp_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "gpp_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int]),
    "gpp_destroy": (None, [ctypes.c_void_p]),
    "gpp_upload": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
         _c_double_p, _c_double_p, _c_double_p, _c_double_p, _c_double_p, ctypes.c_int32,
         ctypes.c_int64, ctypes.c_int64],
    ),
    "gpp_synth": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
         ctypes.POINTER(ctypes.c_uint64), _c_double_p, ctypes.c_int64, ctypes.c_int64],
    ),
    "gpp_run": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int32, _c_double_p, _c_double_p, _c_i64_p, _c_float_p],
    ),
    "gpp_evaluate_host": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
         _c_double_p, _c_double_p, _c_double_p, _c_double_p, _c_double_p, ctypes.c_int32,
         ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, _c_double_p, _c_double_p, _c_i64_p, _c_float_p],
    ),
    "gpp_run_factored": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int32, _c_double_p, _c_double_p, _c_i64_p, _c_float_p],
    ),
    "gpp_variant_terms": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int32, _c_double_p, _c_double_p, ctypes.POINTER(ctypes.c_uint8),
         ctypes.POINTER(ctypes.c_uint8)],
    ),
    "gpp_time": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, _c_float_p, _c_float_p]),
    "gpp_launch_count": (ctypes.c_int, [ctypes.c_void_p, _c_i64_p]),
    "gpp_plan": (
        ctypes.c_int,
        [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
         ctypes.c_int32, _c_i32_p, _c_i64_p],
    ),
    "gpp_plan_piece": (
        ctypes.c_int,
        [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
         ctypes.c_int32, ctypes.c_int32, _c_i32_p, _c_i64_p],
    ),
    "gpp_kernel_info": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int32, _c_i32_p, _c_i32_p, _c_i32_p, _c_i32_p, _c_i32_p, _c_i32_p],
    ),
    "gpp_comm_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "gpp_comm_init": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]),
    "gpp_comm_init_all": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int]),
    "gpp_run_group": (
        ctypes.c_int,
        [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int32, _c_double_p, _c_double_p,
         _c_i64_p, _c_float_p],
    ),
    "gpp_time_group": (
        ctypes.c_int,
        [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int32, ctypes.c_int32, _c_float_p,
         _c_float_p],
    ),
    "gpp_host_register": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t]),
    "gpp_host_unregister": (ctypes.c_int, [ctypes.c_void_p]),
    "gpp_fp64_peak": (ctypes.c_int, [ctypes.c_int, ctypes.c_int32, ctypes.POINTER(ctypes.c_double), _c_float_p]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the library; raise GPUError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("GPP_B200_LIB", LIB_PATH))
    if not path.exists():
        raise GPUError(
            f"CUDA library {path} is missing: build it with __graft_entry__.build() "
            "or `make -C paper_2008_11326_b200/csrc` (there is no CPU fallback)",
            GPP_ERR_CUDA,
        )
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.gpp_abi_version() != 1:
        raise GPUError(f"{path}: unexpected ABI version {lib.gpp_abi_version()}")
    _lib = lib
    return lib


def check(status: int, what: str = "") -> None:
    """Map a C-ABI status to the reference's exception hierarchy."""
    if status == GPP_OK:
        return
    msg = (load().gpp_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == GPP_ERR_ARG:
        raise DomainError(text)
    raise GPUError(text, status)


def dptr(arr) -> ctypes.POINTER(ctypes.c_double):
    return arr.ctypes.data_as(_c_double_p)
