"""Empirical slack penalty C (reference ``solver.py:190-232``).

``compute_penalty_C(x, y, q, seed)`` keeps the reference signature, return
value ``(C, dist)`` and errors.  The class split and the seeded subsampling
(``np.random.default_rng(seed).choice`` per class beyond 2000 samples,
``solver.py:208-213``) are the reference's own host calls, so the same
samples are chosen; the O(n_+ n_- d) part -- squared norms, the between-class
Gram and the median of the positive distances -- runs on the device
(``gdwd_between_class_median``: FP64 tensor-core Gram + radix selection).
"""

from __future__ import annotations

import ctypes as C
import math
from typing import Optional

import numpy as np

from . import _lib
from .scoring import device_matrix
from .solver import SingleClassError, _check
from .sparse import SparseMatrixCSC

_SUBSAMPLE_LIMIT = 2000  # solver.py:190


def between_class_median(x: SparseMatrixCSC, pos: np.ndarray, neg: np.ndarray,
                         device: Optional[int] = None) -> tuple[float, int]:
    """(median of the positive between-class distances, their count) for the
    samples (columns of x) listed in pos and neg."""
    dm = device_matrix(x, device)
    ia = np.ascontiguousarray(pos, dtype=np.int64)
    ib = np.ascontiguousarray(neg, dtype=np.int64)
    med = C.c_double(0.0)
    cnt = C.c_int64(0)
    p64 = C.POINTER(C.c_int64)
    _check(dm.lib.gdwd_between_class_median(dm.ctx, ia.ctypes.data_as(p64), ia.size, ib.ctypes.data_as(p64),
                                            ib.size, C.byref(med), C.byref(cnt)), dm.ctx, "between_class_median")
    return float(med.value), int(cnt.value)


def compute_penalty_C(x: SparseMatrixCSC, y: np.ndarray, q: float, seed: int = 0,
                      device: Optional[int] = None) -> tuple[float, float]:
    """``C = 10^(q+1) * max(1, 10^(q-1) * ln(n) * max(1000, d)^(1/3) / dist^(q+1))``
    with ``dist`` the median between-class Euclidean distance (classes
    subsampled to 2000 points each beyond that size; exact zero distances
    excluded) -- solver.py:193-232."""
    from .sparse import as_csc

    x = as_csc(x)
    y = np.asarray(y, dtype=np.float64)
    n = y.size
    pos = np.flatnonzero(y > 0)
    neg = np.flatnonzero(y < 0)
    if pos.size == 0 or neg.size == 0:
        raise SingleClassError("both classes are required to set the penalty")
    rng = np.random.default_rng(seed)
    if pos.size > _SUBSAMPLE_LIMIT:
        pos = np.sort(rng.choice(pos, _SUBSAMPLE_LIMIT, replace=False))
    if neg.size > _SUBSAMPLE_LIMIT:
        neg = np.sort(rng.choice(neg, _SUBSAMPLE_LIMIT, replace=False))
    dist, count = between_class_median(x, pos, neg, device)
    if count == 0:
        raise ValueError("all between-class distances are zero")
    c = 10.0 ** (q + 1.0) * max(
        1.0,
        10.0 ** (q - 1.0) * math.log(n) * max(1000.0, float(x.nrows)) ** (1.0 / 3.0)
        / dist ** (q + 1.0),
    )
    return c, dist


__all__ = ["between_class_median", "compute_penalty_C"]
