"""ctypes binding of the C ABI in include/cals_b200.h (libcals_b200.so).

The product path has no CPU fallback: if the library cannot be loaded, or
no CUDA device is present, every call raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcals_b200.so")

_lib = None
_lock = threading.Lock()

c_int_p = C.POINTER(C.c_int)
c_i64_p = C.POINTER(C.c_int64)
c_dbl_p = C.POINTER(C.c_double)
c_void_pp = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); mirrors include/cals_b200.h exactly
SIGNATURES = {
    "cals_abi_version": (C.c_int, []),
    "cals_last_error": (C.c_char_p, []),
    "cals_tensor_create": (C.c_int, [C.c_int, c_i64_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     c_void_pp]),
    "cals_tensor_destroy": (C.c_int, [C.c_void_p]),
    "cals_tensor_sqnorm": (C.c_int, [C.c_void_p, C.c_void_p, c_dbl_p]),
    "cals_tensor_data": (C.c_int, [C.c_void_p, c_void_pp, c_i64_p]),
    "cals_mttkrp_workspace_bytes": (C.c_int, [C.c_void_p, C.c_int, C.c_int64,
                                              C.POINTER(C.c_size_t)]),
    "cals_mttkrp": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_void_pp, C.c_int64, C.c_void_p,
                              C.c_int64, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "cals_mttkrp_variants": (C.c_int, [c_int_p]),
    "cals_mttkrp_kernel_info": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, c_int_p, c_dbl_p]),
    "cals_update_factor": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
                                     C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                     C.c_void_p]),
    "cals_update_scratch_bytes": (C.c_size_t, [C.c_int]),
    "cals_engine_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_int,
                                     c_void_pp]),
    "cals_engine_destroy": (C.c_int, [C.c_void_p]),
    "cals_engine_prepare": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cals_engine_set_tensor": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cals_engine_pool": (C.c_int, [C.c_void_p, c_void_pp, c_i64_p]),
    "cals_engine_load_pool": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "cals_engine_run": (C.c_int, [C.c_void_p, C.c_double, C.c_int, C.c_double, C.c_int,
                                  C.c_void_p, c_int_p]),
    "cals_engine_results": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]),
    "cals_engine_pool_download": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "cals_engine_last_launches": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cals_engine_trace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                    c_int_p]),
    "cals_engine_variant": (C.c_int, [C.c_void_p, C.c_int, c_int_p, c_int_p, c_int_p, c_int_p]),
    "cals_fp64_peak_probe": (C.c_int, [C.c_void_p, c_dbl_p]),
    "cals_int8_peak_probe": (C.c_int, [C.c_void_p, c_dbl_p]),
    "cals_engine_set_line_search": (C.c_int, [C.c_void_p, C.c_int, C.c_double]),
    "cals_engine_set_nonneg": (C.c_int, [C.c_void_p, C.c_int]),
    "cals_nnls_rows": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int,
                                 C.c_void_p]),
    "cals_engine_nnls_warnings": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cals_engine_update_failures": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cals_engine_begin":(C.c_int, [C.c_void_p, C.c_double, C.c_int, C.c_double, C.c_void_p]),
    "cals_engine_enqueue_mttkrp": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "cals_engine_enqueue_update": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "cals_engine_enqueue_plan": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cals_engine_done": (C.c_int, [C.c_void_p, c_int_p]),
    "cals_engine_buffers": (C.c_int, [C.c_void_p, c_void_pp, c_void_pp, c_i64_p, c_i64_p,
                                      c_void_pp]),
}


class NativeUnavailable(RuntimeError):
    """libcals_b200.so is missing or unusable (no CPU fallback exists)."""


class NativeError(RuntimeError):
    """A C-ABI call returned a negative code."""

    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code


def load(require_cuda: bool = True):
    """Load the library once; with ``require_cuda`` also insist on a GPU."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_cuda:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the CALS hot path only runs on the GPU")
    return _lib


def call(name: str, *args) -> int:
    lib = load()
    rc = getattr(lib, name)(*args)
    if isinstance(rc, int) and rc < 0:
        msg = lib.cals_last_error()
        raise NativeError(name, rc, msg.decode() if msg else "")
    return rc


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
