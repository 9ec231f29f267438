"""ctypes binding of libgdwd_b200.so (C ABI: include/gdwd_b200.h).

There is no CPU fallback: if the library is missing or cannot load, every
product entry point raises ``GdwdLibraryError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libgdwd_b200.so"

OK = 0
ERR_CUDA, ERR_VALUE, ERR_INDEFINITE, ERR_SCHUR, ERR_LANCZOS, ERR_ASSERT, ERR_UNSUPPORTED, ERR_ABORTED = range(1, 9)
BACKEND_CODE = {"auto": 0, "direct": 1, "smw2": 2, "iterative": 3}
BACKEND_NAME = {v: k for k, v in BACKEND_CODE.items()}

# exported symbols (checked by the CPU test-suite against include/gdwd_b200.h)
SYMBOLS = [
    "gdwd_ctx_create", "gdwd_ctx_destroy", "gdwd_last_error", "gdwd_version", "gdwd_upload_dense",
    "gdwd_upload_csc", "gdwd_set_problem", "gdwd_matvec", "gdwd_matvec_t", "gdwd_abi_sizes", "gdwd_score", "gdwd_between_class_median", "gdwd_kkt_residuals", "gdwd_libsvm_parse", "gdwd_libsvm_sizes",
    "gdwd_libsvm_copy", "gdwd_libsvm_free", "gdwd_preprocess_csc", "gdwd_solve", "gdwd_get_state",
    "gdwd_get_history", "gdwd_newton_sweep", "gdwd_chol_inverse", "gdwd_gram", "gdwd_psqmr_dense",
    "gdwd_solve_begin", "gdwd_solve_iterate", "gdwd_solve_end", "gdwd_time_iterations", "gdwd_set_profile",
    "gdwd_get_profile", "gdwd_reset_counters", "gdwd_frobenius_sq", "gdwd_comm_unique_id",
    "gdwd_comm_init_nccl", "gdwd_comm_init_host", "gdwd_generate_dense", "gdwd_scale_dense",
    "gdwd_download_dense", "gdwd_set_lanczos_start", "gdwd_allreduce_host", "gdwd_time_gram",
    "gdwd_upload_hint", "gdwd_chol_inverse_bordered", "gdwd_get_upload_factor",
]


class GdwdLibraryError(RuntimeError):
    """The CUDA library is unavailable (no CPU fallback exists)."""


class GdwdConfig(C.Structure):
    _fields_ = [
        ("max_iter", C.c_int32), ("backend", C.c_int32), ("use_sgs", C.c_int32),
        ("psqmr_switch_steps", C.c_int32), ("ell", C.c_int32), ("seed", C.c_int32),
        ("use_graph", C.c_int32), ("poll_every", C.c_int32), ("smw_gram_space", C.c_int32),
        ("persistent", C.c_int32), ("iter_gram", C.c_int32),
        ("steplength", C.c_double), ("tol_feas", C.c_double), ("tol_cgap", C.c_double),
        ("tol_cap", C.c_double), ("sigma0", C.c_double), ("epsilon_c", C.c_double), ("mu", C.c_double),
    ]


class GdwdResult(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("converged", C.c_int32), ("backend", C.c_int32),
        ("psqmr_total", C.c_int32), ("double_count", C.c_int32), ("status", C.c_int32),
        ("beta", C.c_double), ("sigma", C.c_double), ("eps_c", C.c_double),
        ("setup_ms", C.c_double), ("loop_ms", C.c_double), ("resid", C.c_double * 11),
    ]


ITER_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.c_double, C.c_double)
ALLREDUCE_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)

_lib = None
_lock = threading.Lock()

_P = C.POINTER(C.c_double)
_I64 = C.c_int64


def _declare(lib):
    vp = C.c_void_p
    sig = {
        "gdwd_ctx_create": (C.c_int, [C.c_int32, C.POINTER(vp)]),
        "gdwd_ctx_destroy": (None, [vp]),
        "gdwd_last_error": (C.c_char_p, [vp]),
        "gdwd_version": (C.c_int, []),
        "gdwd_abi_sizes": (None, [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "gdwd_upload_dense": (C.c_int, [vp, _P, _I64, _I64]),
        "gdwd_upload_csc": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P, _I64, _I64]),
        "gdwd_set_problem": (C.c_int, [vp, _P, _P, _P, C.c_double, C.c_double, C.c_double]),
        "gdwd_matvec": (C.c_int, [vp, _P, _P]),
        "gdwd_matvec_t": (C.c_int, [vp, _P, _P]),
        "gdwd_score": (C.c_int, [vp, _P, C.c_double, _P, _P, C.POINTER(C.c_int64)]),
        "gdwd_kkt_residuals": (C.c_int, [vp, _P, _P, _P, _P, _P, C.c_double, C.c_double, _P]),
        "gdwd_libsvm_parse": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int64, C.c_int32, C.c_int32, C.POINTER(vp),
                                        C.POINTER(C.c_int64), C.c_char_p, C.c_int64]),
        "gdwd_libsvm_sizes": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int32)]),
        "gdwd_libsvm_copy": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P, _P,
                                       C.POINTER(C.c_int64)]),
        "gdwd_libsvm_free": (None, [vp]),
        "gdwd_preprocess_csc": (C.c_int, [C.c_int64, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P,
                                          C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P,
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P, C.POINTER(C.c_int64)]),
        "gdwd_between_class_median": (C.c_int, [vp, C.POINTER(C.c_int64), C.c_int64, C.POINTER(C.c_int64),
                                                C.c_int64, _P, C.POINTER(C.c_int64)]),
        "gdwd_solve": (C.c_int, [vp, C.POINTER(GdwdConfig), _P, _I64, ITER_CB, vp, C.POINTER(GdwdResult)]),
        "gdwd_solve_begin": (C.c_int, [vp, C.POINTER(GdwdConfig), _P, _I64]),
        "gdwd_solve_iterate": (C.c_int, [vp, C.c_int32, ITER_CB, vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "gdwd_solve_end": (C.c_int, [vp, C.POINTER(GdwdResult)]),
        "gdwd_time_iterations": (C.c_int, [vp, C.c_int32, _P, C.POINTER(C.c_int32)]),
        "gdwd_set_profile": (C.c_int, [vp, C.c_int32]),
        "gdwd_get_profile": (C.c_int, [vp, C.c_char_p, _I64, C.POINTER(C.c_int64)]),
        "gdwd_reset_counters": (C.c_int, [vp]),
        "gdwd_frobenius_sq": (C.c_int, [vp, _P]),
        "gdwd_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
        "gdwd_generate_dense": (C.c_int, [vp, C.c_int32, C.c_uint64, _I64, _I64, _I64, _I64, C.c_double]),
        "gdwd_scale_dense": (C.c_int, [vp, _P, C.c_double]),
        "gdwd_download_dense": (C.c_int, [vp, _P]),
        "gdwd_set_lanczos_start": (C.c_int, [vp, _P, _I64]),
        "gdwd_comm_init_nccl": (C.c_int, [vp, C.c_int32, C.c_int32, C.POINTER(C.c_uint8), C.c_int64]),
        "gdwd_comm_init_host": (C.c_int, [vp, C.c_int32, C.c_int32, ALLREDUCE_CB, vp, C.c_int64]),
        "gdwd_allreduce_host": (C.c_int, [vp, _P, _I64]),
        "gdwd_time_gram": (C.c_int, [vp, C.c_int32, _P]),
        "gdwd_get_state": (C.c_int, [vp, _P, _P, _P, _P, _P, _P, _P, _P]),
        "gdwd_get_history": (C.c_int, [vp, _P, _I64, C.POINTER(C.c_int64)]),
        "gdwd_newton_sweep": (C.c_int, [C.c_int32, _I64, _P, C.c_double, C.c_double, _P, _P, C.c_double, C.c_int32,
                                        C.c_int32, _P, C.POINTER(C.c_int32)]),
        "gdwd_chol_inverse": (C.c_int, [C.c_int32, _P, _I64, _P]),
        "gdwd_chol_inverse_bordered": (C.c_int, [C.c_int32, _P, _I64, C.c_int32, _P]),
        "gdwd_upload_hint": (C.c_int, [vp, C.c_int32, C.c_double]),
        "gdwd_get_upload_factor": (C.c_int, [vp, _P, _P, C.POINTER(C.c_int32)]),
        "gdwd_gram": (C.c_int, [C.c_int32, _P, _I64, _I64, C.c_int32, C.c_double, C.c_double, _P]),
        "gdwd_psqmr_dense": (C.c_int, [C.c_int32, _P, _I64, _P, _P, C.c_double, C.c_int32, _P, _P,
                                       C.POINTER(C.c_int32), _P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


def load(path: os.PathLike | str | None = None):
    """Load (once) and return the library; raise GdwdLibraryError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise GdwdLibraryError(
                f"{p} not found: build it with `python -m paper_2305_12019_b200.build` "
                "(the solver has no CPU fallback)")
        try:
            _lib = _declare(C.CDLL(str(p)))
        except OSError as exc:
            raise GdwdLibraryError(f"cannot load {p}: {exc}") from exc
        return _lib


def ptr(a: np.ndarray | None):
    """double* of a C-contiguous float64 array (None -> NULL)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_P)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


__all__ = ["ALLREDUCE_CB", "BACKEND_CODE", "BACKEND_NAME", "GdwdConfig", "GdwdLibraryError", "GdwdResult", "ITER_CB",
           "LIB_PATH", "SYMBOLS", "f64", "load", "ptr"]
