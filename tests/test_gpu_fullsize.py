"""Parity at BASELINE.json's full sizes (pytest -m gpu).

* first 20 iterates of the device solver against the CPU oracle run here on
  the same seeded inputs, 1e-9 relative (configs 2, 3, 4; the oracle uses
  dense BLAS products for the dense configs: same math, different summation
  order);
* final state against fixtures recorded by running the REFERENCE itself to
  its stopping rule or max_iter (tests/golden/full_*.npz, made by
  make_golden_full.py): configs 2, 3, 4 and a config-5 proxy (d = 6000,
  n = 30000, q = 4: ITERATIVE with the Gram operator, the c5 production
  path), under sigma replay; config 1 is pinned the same way in
  test_gpu_parity.py."""

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
    _compare(_device_iterates(prob), _oracle_iterates(prob, "csc"))


# ---------------------------------------------------------------------------
# final state against the REFERENCE run to its stopping rule / max_iter
# (tests/golden/make_golden_full.py; reference solver.py:548-602)
# ---------------------------------------------------------------------------
FULL = ["c2", "c3", "c4", "c5p"]
from conftest import GOLDEN  # noqa: E402

FULL = [f for f in FULL if (GOLDEN / f"full_{f}.npz").exists()]  # TEMP while fixtures are generated
FINAL_TOL = 1e-6  # north_star: final w, beta, objective within 1e-6 relative


def _full_problem(name, fx):
    cfg = synth.CONFIGS[str(fx["cfg"])]
    if name == "c5p":
        cfg = cfg.scaled(d=int(fx["d"]), n=int(fx["n"]))
    prob = synth.make_problem(cfg, 0)
    import hashlib

    sha = hashlib.sha256(np.ascontiguousarray(prob.z_tilde.values).tobytes()).hexdigest()[:16]
    assert sha == str(fx["z_sha"]), "generator changed since the fixture was made"
    return prob


@pytest.fixture(scope="module", params=FULL)
def full_case(request):
    from conftest import GOLDEN

    fx = dict(np.load(GOLDEN / f"full_{request.param}.npz", allow_pickle=False))
    return request.param, fx, _full_problem(request.param, fx)


def test_full_final_state_sigma_replay(full_case):
    """The whole solve (2000 iterations or the stopping rule) under the
    reference's sigma sequence: same iteration count and
    converged flag, the same number of Step-1c re-solves, final w, beta and
    primal objective within 1e-6, the same train error."""
    name, fx, prob = full_case
    hist = fx["hist"]
    out = G.sgs_admm_solve(prob, G.SolverConfig(q=prob.q, max_iter=int(fx["max_iter"])), sigma_schedule=hist[:, 11])
    assert out.backend_used.value == str(fx["backend"])
    assert out.iterations == int(fx["iterations"]) and out.converged == bool(fx["converged"])
    assert out.double_count == int(fx["double_count"]), (out.double_count, int(fx["double_count"]))
    if str(fx["backend"]) == "iterative":
        assert out.psqmr_total == int(fx["psqmr_total"]), (out.psqmr_total, int(fx["psqmr_total"]))
    assert relerr(out.final_state.w, fx["final_w"]) < FINAL_TOL, relerr(out.final_state.w, fx["final_w"])
    b = float(fx["final_beta"])
    assert abs(out.final_state.beta - b) <= FINAL_TOL * max(abs(b), 1e-12), (out.final_state.beta, b)
    op = float(fx["obj_primal"])
    assert abs(out.final_residuals.obj_primal - op) <= FINAL_TOL * abs(op)
    assert out.train_error_pct == float(fx["train_error"])
    # the device KKT history follows the reference's per-iteration scalars
    dev_sigma = out.history[:, 11]
    assert np.array_equal(dev_sigma, hist[: out.iterations, 11])


def test_full_first_iterates(full_case):
    """Iterates 1 and 20 (full w; 4096 sampled coordinates of alpha, r, xi)
    against the reference run, 1e-9 relative, through the callback path and
    (when it applies) the persistent kernel without callback."""
    name, fx, prob = full_case
    got = {}

    def cb(st, res):
        if st.iter in (1, 20):
            got[st.iter] = (st.w.copy(), st.alpha.copy(), st.r.copy(), st.xi.copy())

    G.sgs_admm_solve(prob, G.SolverConfig(q=prob.q, max_iter=K), callback=cb)
    idx = fx["idx_n"]
    assert relerr(got[1][0], fx["w1"]) < TOL
    assert relerr(got[20][0], fx["w20"]) < TOL
    for j, key in ((1, "alpha"), (2, "r"), (3, "xi")):
        assert relerr(got[20][j][idx], fx["s20_" + key]) < TOL, key
    out = G.sgs_admm_solve(prob, G.SolverConfig(q=prob.q, max_iter=K))  # no callback: graph / persistent path
    assert relerr(out.final_state.w, fx["w20"]) < TOL
    assert relerr(out.final_state.alpha[idx], fx["s20_alpha"]) < TOL
