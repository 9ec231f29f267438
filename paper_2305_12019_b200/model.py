"""Model records returned by the solver (reference ``ingest.py:39-87``).

The records the solver's ``SolveResult`` carries; LIBSVM parsing,
preprocessing and the JSON model file are in ``ingest.py``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MODEL_FORMAT_VERSION = 1


@dataclass(frozen=True)
class FeatureMeta:
    """Preprocessing record: kept original features and their divisors."""

    kept_ids: np.ndarray
    scales: np.ndarray
    d_original: int

    def __post_init__(self):
        object.__setattr__(self, "kept_ids", np.asarray(self.kept_ids, dtype=np.int64))
        object.__setattr__(self, "scales", np.asarray(self.scales, dtype=np.float64))
        if np.any(self.scales <= 0):
            raise ValueError("scales must be positive")
        if np.any(np.diff(self.kept_ids) <= 0):
            raise ValueError("kept_ids must be strictly increasing")


def identity_meta(d: int) -> FeatureMeta:
    return FeatureMeta(kept_ids=np.arange(d), scales=np.ones(d), d_original=d)


@dataclass
class ModelFile:
    """Trained classifier (w in the preprocessed feature space, already
    divided by the global data scale) plus solver metadata."""

    q: float
    C: float
    z_scale: float
    mu: float
    feature_meta: FeatureMeta
    w: np.ndarray
    beta: float
    solver_info: dict = field(default_factory=dict)
    format_version: int = MODEL_FORMAT_VERSION

    def composite_weights(self) -> np.ndarray:
        out = np.zeros(self.feature_meta.d_original)
        out[self.feature_meta.kept_ids] = self.w / self.feature_meta.scales
        return out


__all__ = ["FeatureMeta", "MODEL_FORMAT_VERSION", "ModelFile", "identity_meta"]
