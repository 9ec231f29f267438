"""Host-side container for the scaled data matrix Z~ (d x n, samples as columns).

Mirrors the reference type ``SparseMatrixCSC`` (reference
``pkg/src/gdwd/linalg/sparse.py:20-79``): same field names, same invariants,
same ``scipy`` view, ``frobenius_norm`` and ``row_sq_sums``.

Difference that matters on B200: a fully dense matrix (every one of the d*n
entries stored, the common case for the BASELINE dense configs) is kept as
the sample-major ``values`` array only; its CSC index arrays are synthesised
lazily, because the device never needs them (a dense sample row is uploaded
as-is).  ``values`` of a dense CSC matrix *is*
the row-major [n, d] sample matrix, so no copy or transpose is involved.
"""

from __future__ import annotations

from typing import Optional

import numpy as np


class SparseFormatError(ValueError):
    """Invalid CSC structure (reference ``sparse.py:16-17``)."""


class SparseMatrixCSC:
    """Immutable CSC matrix; ``values[colptr[j]:colptr[j+1]]`` is column j."""

    __slots__ = ("nrows", "ncols", "_colptr", "_rowidx", "values", "_dense", "_scipy", "_device")

    def __init__(self, nrows: int, ncols: int, colptr, rowidx, values):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self._colptr = np.asarray(colptr, dtype=np.int64)
        self._rowidx = np.asarray(rowidx, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self._dense = False
        self._scipy = None
        self._device = None  # scoring.DeviceMatrix cache
        cp = self._colptr
        if cp.shape != (self.ncols + 1,):
            raise SparseFormatError("colptr must have length ncols+1")
        if cp[0] != 0 or cp[-1] != self.values.size:
            raise SparseFormatError("colptr endpoints do not match stored entries")
        if np.any(np.diff(cp) < 0):
            raise SparseFormatError("colptr must be nondecreasing")
        if self._rowidx.size != self.values.size:
            raise SparseFormatError("rowidx and values length mismatch")
        if self._rowidx.size and (self._rowidx.min() < 0 or self._rowidx.max() >= self.nrows):
            raise SparseFormatError("row index out of bounds")
        self._dense = self.values.size == self.nrows * self.ncols and self.nrows > 0

    @classmethod
    def from_dense_samples(cls, samples: np.ndarray) -> "SparseMatrixCSC":
        """Wrap a row-major [n, d] sample matrix (column i of Z~ = row i) as a
        fully stored d x n CSC matrix without materialising index arrays."""
        samples = np.ascontiguousarray(samples, dtype=np.float64)
        if samples.ndim != 2:
            raise ValueError("expected a 2-D [n, d] sample matrix")
        self = cls.__new__(cls)
        self.ncols, self.nrows = (int(s) for s in samples.shape)
        self.values = samples.reshape(-1)
        self._colptr = None
        self._rowidx = None
        self._dense = self.nrows > 0
        self._scipy = None
        self._device = None
        return self

    # -- reference fields --------------------------------------------------
    @property
    def colptr(self) -> np.ndarray:
        if self._colptr is None:
            self._colptr = np.arange(self.ncols + 1, dtype=np.int64) * self.nrows
        return self._colptr

    @property
    def rowidx(self) -> np.ndarray:
        if self._rowidx is None:
            self._rowidx = np.tile(np.arange(self.nrows, dtype=np.int64), self.ncols)
        return self._rowidx

    @property
    def is_dense(self) -> bool:
        """True when every entry is stored (column-major dense layout)."""
        return self._dense

    def dense_samples(self) -> np.ndarray:
        """Row-major [n, d] view of a fully stored matrix (zero-copy)."""
        if not self._dense:
            raise ValueError("matrix is not fully stored")
        return self.values.reshape(self.ncols, self.nrows)

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    @property
    def scipy(self):
        """scipy ``csc_matrix`` view (reference ``sparse.py:52-57``)."""
        if self._scipy is None:
            import scipy.sparse as sp

            self._scipy = sp.csc_matrix(
                (self.values, self.rowidx, self.colptr), shape=(self.nrows, self.ncols)
            )
        return self._scipy

    def frobenius_norm(self) -> float:
        """reference ``sparse.py:63-64``."""
        return float(np.sqrt(np.sum(self.values * self.values)))

    def row_sq_sums(self) -> np.ndarray:
        """diag(Z Z^T) (reference ``sparse.py:66-70``)."""
        if self._dense:
            sq = self.dense_samples()
            return np.einsum("ij,ij->j", sq, sq)
        return np.bincount(self.rowidx, weights=self.values * self.values, minlength=self.nrows)

    def column(self, j: int) -> np.ndarray:
        lo, hi = self.colptr[j], self.colptr[j + 1]
        out = np.zeros(self.nrows)
        out[self.rowidx[lo:hi]] = self.values[lo:hi]
        return out

    def toarray(self) -> np.ndarray:
        if self._dense:
            return self.dense_samples().T.copy()
        return self.scipy.toarray()

    def with_values(self, values: np.ndarray) -> "SparseMatrixCSC":
        """Same structure, new values (used by scale_problem)."""
        if self._dense:
            return SparseMatrixCSC.from_dense_samples(values.reshape(self.ncols, self.nrows))
        return SparseMatrixCSC(self.nrows, self.ncols, self.colptr.copy(), self.rowidx.copy(), values)


def as_csc(x) -> SparseMatrixCSC:
    """``x`` itself, or -- drop-in use -- a reference ``SparseMatrixCSC``
    (reference linalg/sparse.py:20-50: nrows, ncols, colptr, rowidx, values)
    converted once and cached on that object."""
    if isinstance(x, SparseMatrixCSC):
        return x
    conv = getattr(x, "_gdwd_csc", None)
    if conv is None:
        conv = SparseMatrixCSC(x.nrows, x.ncols, x.colptr, x.rowidx, x.values)
        try:
            object.__setattr__(x, "_gdwd_csc", conv)
        except (AttributeError, TypeError):
            pass
    return conv


def csc_from_scipy(m) -> SparseMatrixCSC:
    """reference ``sparse.py:82-94``: duplicates summed, zeros pruned, sorted."""
    import scipy.sparse as sp

    c = sp.csc_matrix(m, copy=True)
    c.sum_duplicates()
    c.eliminate_zeros()
    c.sort_indices()
    return SparseMatrixCSC(c.shape[0], c.shape[1], c.indptr.astype(np.int64),
                           c.indices.astype(np.int64), c.data.astype(np.float64))


def csc_from_dense(a: np.ndarray) -> SparseMatrixCSC:
    """reference ``sparse.py:97-98``."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 2 and a.size and np.all(a != 0.0):
        return SparseMatrixCSC.from_dense_samples(np.ascontiguousarray(a.T))
    import scipy.sparse as sp

    return csc_from_scipy(sp.csc_matrix(a))


def csc_from_triplets(triplets, nrows: int, ncols: int) -> SparseMatrixCSC:
    """reference ``sparse.py:101-126``."""
    trip = list(triplets)
    if not trip:
        return SparseMatrixCSC(nrows, ncols, np.zeros(ncols + 1, np.int64),
                               np.zeros(0, np.int64), np.zeros(0))
    rows = np.asarray([t[0] for t in trip], dtype=np.int64)
    cols = np.asarray([t[1] for t in trip], dtype=np.int64)
    vals = np.asarray([t[2] for t in trip], dtype=np.float64)
    if rows.min() < 0 or rows.max() >= nrows:
        raise SparseFormatError(f"row index out of bounds for {nrows} rows")
    if cols.min() < 0 or cols.max() >= ncols:
        raise SparseFormatError(f"column index out of bounds for {ncols} columns")
    if not np.all(np.isfinite(vals)):
        raise SparseFormatError("non-finite value in triplets")
    import scipy.sparse as sp

    return csc_from_scipy(sp.coo_matrix((vals, (rows, cols)), shape=(nrows, ncols)))


def csr_of(z: SparseMatrixCSC):
    """Feature-major CSR arrays of Z~ (int32 indices), built on the host for
    the device's Z.t gather kernel.  Returns (rowptr[d+1], colidx[nnz], val[nnz])."""
    m = z.scipy.tocsr()
    m.sort_indices()
    return (m.indptr.astype(np.int32 if m.nnz < 2**31 else np.int64),
            m.indices.astype(np.int32), m.data.astype(np.float64))


__all__ = ["SparseFormatError", "SparseMatrixCSC", "as_csc", "csc_from_dense", "csc_from_scipy",
           "csc_from_triplets", "csr_of"]
