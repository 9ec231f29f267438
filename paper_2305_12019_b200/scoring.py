"""Applying a trained model on the device (reference ``solver.py:610-642``).

``decision_values`` / ``predict`` / ``train_error`` keep the reference
signatures and conventions:

* scores are ``beta + x_raw^T w_composite`` over the raw samples (columns of
  ``x``); features beyond the training dimension are ignored and missing
  trailing features count as zero (``solver.py:617-629``);
* ``predict`` is ``where(score > 0, +1, -1)`` (``:632-636``; a zero score
  gives -1 -- the reference's docstring says +1, its code does not);
* ``train_error`` counts ``y * sign(score) <= 0`` -- a zero score is wrong for
  both classes (``:639-642``).

The raw matrix is uploaded once per ``SparseMatrixCSC`` (dense sample-major
or CSC/CSR, as for the solver) and scored by one fused pass
(``gdwd_score``: the Z^T w kernel with a score / error-count epilogue).
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .model import ModelFile
from .solver import DeviceProblem, _check
from .sparse import SparseMatrixCSC, as_csc


class DeviceMatrix(DeviceProblem):
    """A raw (unscaled) sample matrix resident in HBM, for scoring."""

    def __init__(self, x: SparseMatrixCSC, device: int = 0):
        super().__init__(None, device)
        self.n, self.d = x.ncols, x.nrows
        lib = self.lib
        if x.is_dense:
            _check(lib.gdwd_upload_dense(self.ctx, _lib.ptr(x.values), self.d, self.n), self.ctx, "upload")
        else:
            cp = np.ascontiguousarray(x.colptr, dtype=np.int64)
            ri = np.ascontiguousarray(x.rowidx, dtype=np.int64)
            _check(lib.gdwd_upload_csc(self.ctx, cp.ctypes.data_as(C.POINTER(C.c_int64)),
                                       ri.ctypes.data_as(C.POINTER(C.c_int64)), _lib.ptr(_lib.f64(x.values)),
                                       self.d, self.n), self.ctx, "upload")

    def score(self, w: np.ndarray, beta: float, y: Optional[np.ndarray] = None, want_scores: bool = True):
        """(scores or None, wrong count or None) for weights of length d."""
        w = _lib.f64(w)
        if w.shape != (self.d,):
            raise ValueError(f"dimension mismatch: weights have length {w.shape}, expected ({self.d},)")
        out = np.empty(self.n) if want_scores else None
        yv = None
        if y is not None:
            yv = _lib.f64(y)
            if yv.shape != (self.n,):
                raise ValueError("labels must have one entry per sample")
        cnt = C.c_int64(0)
        _check(self.lib.gdwd_score(self.ctx, _lib.ptr(w), float(beta), _lib.ptr(yv) if yv is not None else None,
                                   _lib.ptr(out) if out is not None else None, C.byref(cnt)), self.ctx, "score")
        return out, (int(cnt.value) if yv is not None else None)


def device_matrix(x: SparseMatrixCSC, device: Optional[int] = None) -> DeviceMatrix:
    """The (cached) device copy of a raw sample matrix."""
    x = as_csc(x)
    want = 0 if device is None else int(device)
    dev = getattr(x, "_device", None)
    if dev is None or dev.ctx is None or dev.device != want:
        dev = DeviceMatrix(x, want)
        x._device = dev
    return dev


def _effective_weights(model: ModelFile, d_in: int) -> np.ndarray:
    """solver.py:617-629: the composite weights padded with zeros or cut to
    the input dimension."""
    composite = model.composite_weights()
    d_tr = composite.size
    if d_in == d_tr:
        return composite
    if d_in > d_tr:
        return np.concatenate([composite, np.zeros(d_in - d_tr)])
    return composite[:d_in]


def decision_values(model: ModelFile, x: SparseMatrixCSC, device: Optional[int] = None) -> np.ndarray:
    """Scores ``beta + x_raw @ w_composite`` for raw samples (columns)
    (solver.py:610-629)."""
    dm = device_matrix(x, device)
    scores, _ = dm.score(_effective_weights(model, x.nrows), model.beta)
    return scores


def predict(model: ModelFile, x: SparseMatrixCSC, device: Optional[int] = None) -> np.ndarray:
    """Hard labels ``where(score > 0, +1, -1)`` (solver.py:632-636)."""
    scores = decision_values(model, x, device)
    return np.where(scores > 0.0, 1.0, -1.0)


def train_error(model: ModelFile, x: SparseMatrixCSC, y: np.ndarray, device: Optional[int] = None) -> float:
    """Percentage of samples with ``y * sign(score) <= 0`` (solver.py:639-642),
    counted on the device in the scoring pass."""
    y = np.asarray(y, dtype=np.float64)
    dm = device_matrix(x, device)
    _, wrong = dm.score(_effective_weights(model, x.nrows), model.beta, y, want_scores=False)
    return 100.0 * (float(wrong) / y.size)


__all__ = ["DeviceMatrix", "decision_values", "device_matrix", "predict", "train_error"]
