"""Penalty parameter C (compute_penalty_C, solver.py:193-232): the oracle
pinned to the reference's values (tests/golden/penalty.json), then the
device path (FP64 tensor-core between-class Gram + radix-select median)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import gdwd_oracle as O

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))


def _cases():
    import importlib

    mg = importlib.import_module("make_golden_inputs")
    return mg.penalty_inputs()


def _ref():
    return json.loads((GOLDEN / "penalty.json").read_text())


@pytest.mark.parametrize("name", ["dense", "dense_q2", "sparse_sub", "duplicates"])
def test_oracle_penalty_matches_reference(name):
    x, y, q, seed = _cases()[name]
    ref = _ref()[name]
    c, dist = O.penalty_C(x.scipy, y, q, seed)
    assert dist == ref["dist"] and c == ref["C"]


def test_penalty_formula_kat():
    """SPEC: q=1, n=100, d=50, dist=2 -> C = 100 max(1, ln(100) 10 / 4)."""
    import math

    c = 10.0 ** 2 * max(1.0, 1.0 * math.log(100) * 1000.0 ** (1.0 / 3.0) / 2.0 ** 2)
    assert abs(c - 1151.29) < 0.01


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dense", "dense_q2", "sparse_sub", "duplicates"])
def test_device_penalty_matches_reference(name):
    import paper_2305_12019_b200 as G

    x, y, q, seed = _cases()[name]
    ref = _ref()[name]
    c, dist = G.compute_penalty_C(x, y, q, seed)
    assert abs(dist - ref["dist"]) <= 1e-12 * ref["dist"]
    assert abs(c - ref["C"]) <= 1e-12 * ref["C"]


@pytest.mark.gpu
def test_device_penalty_errors():
    import paper_2305_12019_b200 as G
    from paper_2305_12019_b200.sparse import SparseMatrixCSC

    x = SparseMatrixCSC.from_dense_samples(np.ones((4, 3)))
    with pytest.raises(G.SingleClassError):
        G.compute_penalty_C(x, np.ones(4), 1.0)
    with pytest.raises(ValueError):  # every cross-class pair coincides
        G.compute_penalty_C(x, np.array([1.0, -1.0, 1.0, -1.0]), 1.0)
