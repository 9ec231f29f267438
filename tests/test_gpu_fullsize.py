"""Parity at BASELINE.json's full sizes (pytest -m gpu): the first 20
iterates of the device solver against the CPU oracle on the same seeded
inputs, to 1e-9 relative (configs 2, 3, 4; config 1 is pinned against the
reference itself in test_gpu_parity.py).  The oracle uses dense BLAS products
for the dense configs (same math, different summation order)."""

import numpy as np
import pytest

import paper_2305_12019_b200 as G
from oracle import gdwd_oracle as O
from paper_2305_12019_b200 import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-9
K = 20


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _oracle_iterates(prob, operator, k=K):
    its = []
    O.solve(prob, O.OracleConfig(max_iter=k), operator=operator, record=False,
            callback=lambda st, res: its.append({key: np.array(st[key], copy=True) if key != "beta" else st[key]
                                                 for key in ("w", "alpha", "r", "xi", "beta")}))
    return its


def _device_iterates(prob, k=K, **kw):
    its = []
    G.sgs_admm_solve(prob, G.SolverConfig(q=prob.q, max_iter=k),
                     callback=lambda st, res: its.append(dict(w=st.w.copy(), alpha=st.alpha.copy(), r=st.r.copy(),
                                                              xi=st.xi.copy(), beta=st.beta)), **kw)
    return its


def _compare(dev, ref):
    assert len(dev) == len(ref)
    for i, (a, b) in enumerate(zip(dev, ref)):
        for key in ("w", "alpha", "r", "xi"):
            assert relerr(a[key], b[key]) < TOL, (i, key, relerr(a[key], b[key]))
        assert abs(a["beta"] - b["beta"]) <= TOL * max(1.0, abs(b["beta"])), i


@pytest.fixture(scope="module")
def c2():
    return synth.make_problem(synth.CONFIGS["c2"], 0)


def test_c2_first20_gram_space(c2):
    _compare(_device_iterates(c2), _oracle_iterates(c2, "dense"))


def test_c2_persistent_iterate20(c2):
    ref = _oracle_iterates(c2, "dense")[-1]
    out = G.sgs_admm_solve(c2, G.SolverConfig(q=c2.q, max_iter=K), persistent=True)
    st = out.final_state
    for key in ("w", "alpha", "r", "xi"):
        assert relerr(getattr(st, key), ref[key]) < TOL, key


def test_c3_first20():
    prob = synth.make_problem(synth.CONFIGS["c3"], 0)
    _compare(_device_iterates(prob), _oracle_iterates(prob, "dense"))


def test_c4_first20():
    prob = synth.make_problem(synth.CONFIGS["c4"], 0)
    _compare(_device_iterates(prob, k=10), _oracle_iterates(prob, "csc", k=10))
