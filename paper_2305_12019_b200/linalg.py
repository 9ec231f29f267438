"""Device linear-algebra seams (reference ``pkg/src/gdwd/linalg``).

``psqmr`` here takes a dense symmetric operator (the solver's own PSQMR runs
the matrix-free normal operator inside the device loop); ``cholesky_inverse``
and ``gram`` expose the one-time factorisation and the FP64 tensor-core
Gram used by the DIRECT / SMW2 regimes.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .solver import IndefiniteMatrixError, _check


@dataclass(frozen=True)
class PsqmrResult:
    """linalg/psqmr.py:18-24."""

    x: np.ndarray
    iterations: int
    converged: bool
    breakdown: bool
    residual_norm: float


def psqmr_dense(A: np.ndarray, b: np.ndarray, precond_diag: Optional[np.ndarray] = None, tol: float = 1e-8,
                max_iter: Optional[int] = None, x0: Optional[np.ndarray] = None, device: int = 0) -> PsqmrResult:
    """psqmr (linalg/psqmr.py:27-95) for ``A x = b`` with A dense symmetric
    and an optional Jacobi-style diagonal preconditioner M (applies v / M)."""
    A = _lib.f64(A)
    b = _lib.f64(b)
    m = b.size
    if A.shape != (m, m):
        raise ValueError("A must be m x m")
    if max_iter is None:
        max_iter = max(2 * m, 20)
    M = None if precond_diag is None else _lib.f64(precond_diag)
    x0a = None if x0 is None else _lib.f64(x0)
    out = np.empty(m)
    info = (C.c_int32 * 4)()
    rn = C.c_double()
    lib = _lib.load()
    _check(lib.gdwd_psqmr_dense(device, _lib.ptr(A), m, _lib.ptr(b), _lib.ptr(M), float(tol), int(max_iter),
                                _lib.ptr(x0a), _lib.ptr(out), info, C.byref(rn)), None, "psqmr")
    return PsqmrResult(out, int(info[0]), bool(info[1]), bool(info[2]), float(rn.value))


def cholesky_inverse(S: np.ndarray, device: int = 0, block: Optional[int] = None) -> np.ndarray:
    """S^{-1} of an SPD matrix via the device recursive Cholesky + triangular
    inverse (linalg/cholesky.py:25-66).  Raises IndefiniteMatrixError.
    ``block``: the row-block (bordered) chain the pipelined upload uses,
    ``block`` rows per step, instead of the recursion."""
    S = _lib.f64(S)
    m = S.shape[0]
    if S.shape != (m, m):
        raise ValueError("expected a square matrix")
    out = np.empty_like(S)
    lib = _lib.load()
    if block is None:
        rc = lib.gdwd_chol_inverse(device, _lib.ptr(S), m, _lib.ptr(out))
    else:
        rc = lib.gdwd_chol_inverse_bordered(device, _lib.ptr(S), m, int(block), _lib.ptr(out))
    if rc == _lib.ERR_INDEFINITE:
        raise IndefiniteMatrixError("non-positive pivot")
    _check(rc, None, "chol_inverse")
    return out


def gram(X: np.ndarray, sum_over_rows: bool, div: float = 1.0, shift: float = 0.0, device: int = 0) -> np.ndarray:
    """Gram of a row-major [rows, cols] matrix on the FP64 tensor cores:
    X^T X (sum_over_rows) or X X^T, then / div + shift I."""
    X = _lib.f64(X)
    r, c = X.shape
    M = c if sum_over_rows else r
    out = np.empty((M, M))
    lib = _lib.load()
    _check(lib.gdwd_gram(device, _lib.ptr(X), r, c, int(bool(sum_over_rows)), float(div), float(shift),
                         _lib.ptr(out)), None, "gram")
    return out


__all__ = ["PsqmrResult", "cholesky_inverse", "gram", "psqmr_dense"]
