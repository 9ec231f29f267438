"""LIBSVM ingest, preprocessing and model files (reference ``ingest.py``).

Same names, signatures, records and errors as the reference:

* ``parse_libsvm(source, require_labels=True) -> RawDataset`` -- parsing is
  native and multi-threaded (``gdwd_libsvm_parse`` in ``csrc/ingest.cpp``)
  with the reference grammar and error messages (``ingest.py:102-182``); the
  {-1,+1} label mapping is the reference's ``_map_labels`` (``:90-99``).
* ``preprocess(raw) -> (x_clean, labels, FeatureMeta)`` -- native,
  multi-threaded max-abs scaling and zero-feature removal, bit-identical to
  the numpy version (``ingest.py:185-211``).
* ``write_model`` / ``read_model`` -- the versioned JSON model file
  (``ingest.py:214-296``), plain host I/O.
"""

from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass
from pathlib import Path
from typing import IO, Optional, Union

import numpy as np

from . import _lib
from .model import MODEL_FORMAT_VERSION, FeatureMeta, ModelFile, identity_meta
from .sparse import SparseMatrixCSC


class ParseError(ValueError):
    """Malformed input; the message carries the 1-based line number."""

    def __init__(self, line_no: int, message: str):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


class ModelFormatError(ValueError):
    """Model file is missing fields, malformed, or has the wrong version."""


@dataclass(frozen=True)
class RawDataset:
    """Parsed samples as columns of X; ``labels`` is None for unlabeled data."""

    X: SparseMatrixCSC
    labels: Optional[np.ndarray]
    source_path: str


def _threads() -> int:
    v = os.environ.get("GDWD_INGEST_THREADS")
    return int(v) if v else 0


def _map_labels(raw: np.ndarray, line_nos: np.ndarray) -> np.ndarray:
    """ingest.py:90-99: keep {-1,+1}; otherwise the smaller of exactly two
    values maps to -1."""
    distinct = np.unique(raw)
    if distinct.size > 2:
        raise ParseError(int(line_nos[0]), f"more than two distinct labels: {distinct.tolist()[:5]}")
    if set(distinct.tolist()) <= {-1.0, 1.0}:
        return raw.copy()
    if distinct.size == 1:
        raise ParseError(int(line_nos[0]), f"single non-binary label value {distinct[0]}")
    lo = distinct[0]
    return np.where(raw == lo, -1.0, 1.0)


def parse_libsvm(source: Union[str, Path, IO[str]], require_labels: bool = True) -> RawDataset:
    """Parse LIBSVM text ``<label> <idx>:<val> ...`` (1-based, strictly
    increasing indices per line; ``#`` starts a comment) -- ingest.py:102-182."""
    lib = _lib.load()
    if isinstance(source, (str, Path)):
        path = str(source)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        args = (path.encode(), None, 0)
    else:
        path = getattr(source, "name", "<stream>")
        text = source.read()
        if isinstance(text, str):
            text = text.encode("utf-8")
        args = (None, text, len(text))
    handle = C.c_void_p()
    err_line = C.c_int64(0)
    msg = C.create_string_buffer(512)
    rc = lib.gdwd_libsvm_parse(args[0], args[1], args[2], int(bool(require_labels)), _threads(), C.byref(handle),
                               C.byref(err_line), msg, len(msg))
    if rc == _lib.ERR_VALUE:
        raise ParseError(int(err_line.value), msg.value.decode("utf-8", "replace"))
    if rc != 0:
        raise OSError(msg.value.decode("utf-8", "replace") or f"parse failed (code {rc})")
    try:
        n, d, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        unl = C.c_int32()
        lib.gdwd_libsvm_sizes(handle, C.byref(n), C.byref(d), C.byref(nnz), C.byref(unl))
        colptr = np.empty(n.value + 1, dtype=np.int64)
        rowidx = np.empty(nnz.value, dtype=np.int64)
        values = np.empty(nnz.value, dtype=np.float64)
        labels = np.empty(n.value, dtype=np.float64)
        lines = np.empty(n.value, dtype=np.int64)
        p64 = C.POINTER(C.c_int64)
        lib.gdwd_libsvm_copy(handle, colptr.ctypes.data_as(p64), rowidx.ctypes.data_as(p64), _lib.ptr(values),
                             _lib.ptr(labels), lines.ctypes.data_as(p64))
    finally:
        lib.gdwd_libsvm_free(handle)
    x = SparseMatrixCSC(d.value, n.value, colptr, rowidx, values)
    if unl.value:
        return RawDataset(X=x, labels=None, source_path=path)
    return RawDataset(X=x, labels=_map_labels(labels, lines), source_path=path)


def preprocess(raw: RawDataset) -> tuple[SparseMatrixCSC, Optional[np.ndarray], FeatureMeta]:
    """Drop all-zero features and divide each kept feature by its max-abs
    (ingest.py:185-211).  Returns the cleaned matrix, the labels and the
    transform record needed for prediction."""
    x = raw.X
    lib = _lib.load()
    d, n = x.nrows, x.ncols
    colptr = np.ascontiguousarray(x.colptr, dtype=np.int64)
    rowidx = np.ascontiguousarray(x.rowidx, dtype=np.int64)
    values = np.ascontiguousarray(x.values, dtype=np.float64)
    kept_count = C.c_int64(0)
    kept_ids = np.empty(max(d, 1), dtype=np.int64)
    scales = np.empty(max(d, 1), dtype=np.float64)
    new_colptr = np.empty(n + 1, dtype=np.int64)
    new_rowidx = np.empty(values.size, dtype=np.int64)
    new_values = np.empty(values.size, dtype=np.float64)
    new_nnz = C.c_int64(0)
    p64 = C.POINTER(C.c_int64)
    rc = lib.gdwd_preprocess_csc(d, n, colptr.ctypes.data_as(p64), rowidx.ctypes.data_as(p64), _lib.ptr(values),
                                 _threads(), C.byref(kept_count), kept_ids.ctypes.data_as(p64), _lib.ptr(scales),
                                 new_colptr.ctypes.data_as(p64), new_rowidx.ctypes.data_as(p64),
                                 _lib.ptr(new_values), C.byref(new_nnz))
    if rc != 0:
        if kept_count.value == 0 and np.all(np.isfinite(values)):
            raise ValueError("all features are zero")
        raise ValueError("matrix has non-finite or out-of-range entries")
    k = kept_count.value
    m = new_nnz.value
    x_clean = SparseMatrixCSC(k, n, new_colptr, new_rowidx[:m], new_values[:m])
    meta = FeatureMeta(kept_ids=kept_ids[:k].copy(), scales=scales[:k].copy(), d_original=d)
    return x_clean, raw.labels, meta


_REQUIRED_FIELDS = ("format_version", "q", "C", "z_scale", "mu", "feature_meta", "w", "beta", "solver_info")


def write_model(model: ModelFile, path: Union[str, Path]) -> None:
    """Versioned, human-readable JSON; shortest round-trip floats, so
    write/read is exact (ingest.py:228-251)."""
    doc = {
        "format_version": model.format_version,
        "q": float(model.q),
        "C": float(model.C),
        "z_scale": float(model.z_scale),
        "mu": float(model.mu),
        "feature_meta": {
            "kept_ids": model.feature_meta.kept_ids.tolist(),
            "scales": model.feature_meta.scales.tolist(),
            "d_original": int(model.feature_meta.d_original),
        },
        "w": model.w.tolist(),
        "beta": float(model.beta),
        "solver_info": model.solver_info,
    }
    text = json.dumps(doc, indent=1, allow_nan=False)
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(text)
        fh.write("\n")


def read_model(path: Union[str, Path]) -> ModelFile:
    """ingest.py:254-296: validates the version and every field."""
    try:
        with open(path, "r", encoding="utf-8") as fh:
            doc = json.load(fh)
    except json.JSONDecodeError as exc:
        raise ModelFormatError(f"malformed model file: {exc}") from exc
    if not isinstance(doc, dict):
        raise ModelFormatError("malformed model file: expected a JSON object")
    if "format_version" not in doc:
        raise ModelFormatError("missing field 'format_version'")
    if doc["format_version"] != MODEL_FORMAT_VERSION:
        raise ModelFormatError(
            f"unsupported model format_version {doc['format_version']!r}; "
            f"this reader handles version {MODEL_FORMAT_VERSION}"
        )
    for name in _REQUIRED_FIELDS:
        if name not in doc:
            raise ModelFormatError(f"missing field {name!r}")
    fm = doc["feature_meta"]
    for name in ("kept_ids", "scales", "d_original"):
        if name not in fm:
            raise ModelFormatError(f"missing field 'feature_meta.{name}'")
    meta = FeatureMeta(
        kept_ids=np.asarray(fm["kept_ids"], dtype=np.int64),
        scales=np.asarray(fm["scales"], dtype=np.float64),
        d_original=int(fm["d_original"]),
    )
    return ModelFile(
        q=float(doc["q"]),
        C=float(doc["C"]),
        z_scale=float(doc["z_scale"]),
        mu=float(doc["mu"]),
        feature_meta=meta,
        w=np.asarray(doc["w"], dtype=np.float64),
        beta=float(doc["beta"]),
        solver_info=doc["solver_info"],
        format_version=int(doc["format_version"]),
    )


__all__ = ["FeatureMeta", "ModelFile", "ModelFormatError", "ParseError", "RawDataset", "identity_meta",
           "parse_libsvm", "preprocess", "read_model", "write_model"]
