"""The CPU oracle (oracle/gdwd_oracle.py) pinned against fixtures produced by
running the reference package itself (tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest

from conftest import TRAJ_CASES, VAR_CASES, load_kat, solver_options, load_traj, problem_for, relerr
from oracle import gdwd_oracle as O


def test_kat_newton():
    for a, s, q, w, r0, root, its in load_kat()["newton_r"]:
        got, git = O.newton_scalar(a, s, q, w, r0)
        assert got == root and git == its
    # SPEC.md:215-217
    assert O.newton_scalar(0.0, 1.0, 1.0, 1.0, 1.0)[0] == 1.0
    assert abs(O.newton_scalar(0.0, 2.0, 1.0, 1.0, 1.0)[0] - 0.7937005) < 1e-7
    assert abs(O.newton_scalar(10.0, 1.0, 1.0, 1.0, 1.0)[0] - 10.0099) < 1e-4


def test_kat_select_sigma_weights():
    k = load_kat()
    for n, d, kind in k["select_solver"]:
        assert O.select_backend(n, d) == kind
    for s, p, d, out in k["update_sigma"]:
        assert O.sigma_rule(s, p, d) == out
    y = np.array([1.0] * 90 + [-1.0] * 10)
    for q, key in ((1.0, "q1"), (2.0, "q2")):
        w = O.class_weights(y, q)
        assert [w[0], w[-1]] == k["compute_weights"][key]


def test_kat_linalg():
    k = load_kat()
    R = O.chol_upper(np.array([[4.0, 2.0], [2.0, 3.0]]))
    assert np.array_equal(R, np.array(k["cholesky"]["R"]))
    assert np.array_equal(O.chol_apply(R, np.array([6.0, 5.0])), np.array(k["cholesky"]["solve"]))
    with pytest.raises(O.Indefinite):
        O.chol_upper(np.array([[1.0, 2.0], [2.0, 1.0]]))
    p = O.psqmr(lambda v: np.array([1.0, 2.0, 3.0]) * v, np.array([1.0, 2.0, 3.0]), tol=1e-12)
    assert np.array_equal(p.x, np.array(k["psqmr_diag"]["x"])) and p.iterations == k["psqmr_diag"]["iterations"]
    rng = np.random.default_rng(7)
    B = rng.standard_normal((50, 50))
    S = B @ B.T + 50 * np.eye(50)
    b = rng.standard_normal(50)
    M = np.diag(S).copy()
    p2 = O.psqmr(lambda v: S @ v, b, precond=lambda v: v / M, tol=1e-10, max_iter=200)
    ref = k["psqmr_spd50"]
    assert p2.iterations == ref["iterations"] and p2.converged == ref["converged"]
    assert np.array_equal(p2.x, np.array(ref["x"]))
    lam, _ = O.lanczos_topk(lambda v: np.array([5.0, 4.0, 3.0, 2.0, 1.0]) * v, 5, 2)
    assert np.allclose(lam, k["lanczos_diag"]["eigenvalues"], rtol=0, atol=1e-12)


def _hist_row(res, st):
    return [res[f] for f in O.KKT_FIELDS] + [st["sigma"], st["beta"]]


@pytest.mark.parametrize("case", TRAJ_CASES + VAR_CASES)
def test_oracle_matches_reference_trajectory(case):
    tr = load_traj(case)
    prob = problem_for(tr)
    assert hashlib.sha256(prob.z_tilde.values.tobytes()).hexdigest()[:16] == str(tr["z_sha"])
    full = bool(tr["full"])
    rows, vecs = [], {k: [] for k in ("w", "u", "rho", "r", "xi", "alpha")}

    def cb(st, res):
        rows.append(_hist_row(res, st))
        for k in vecs:
            v = np.array(st[k], copy=True)
            if not full:
                v = v[tr["idx_d"]] if k in ("w", "u", "rho") else v[tr["idx_n"]]
            vecs[k].append(v)

    backend = "auto"
    cfg = O.OracleConfig(max_iter=int(tr["max_iter"]), backend=backend,
                         psqmr_switch_steps=int(tr["switch"]) if "switch" in tr else 50, **solver_options(tr))
    if case.startswith("var_"):
        cfg.backend = str(tr["backend"])
    if case.startswith(("tiny_", "prox_")):
        cfg.backend = {"tiny_direct": "direct", "tiny_smw2": "smw2", "tiny_iter": "iterative",
                       "tiny_iter_c4gen": "iterative", "tiny_direct_q2": "direct",
                       "tiny_sparse": "iterative", "prox_tiny": "iterative", "prox_tiny_q2": "iterative"}[case]
    out = O.solve(prob, cfg, operator="csc", callback=cb)
    assert out.backend == str(tr["backend"])
    assert out.converged == bool(tr["converged"])
    assert out.iterations == int(tr["iterations"])
    assert out.double_count == int(tr["double_count"])
    assert out.psqmr_total == int(tr["psqmr_total"])
    h = np.array(rows)
    # the oracle restates the reference's arithmetic with the same scipy
    # products: agreement is at rounding level along the whole trajectory
    assert np.allclose(h[:, :13], tr["hist"][:, :13], rtol=1e-9, atol=1e-14)
    for k, v in vecs.items():
        assert relerr(np.array(v), tr["it_" + k]) < 1e-10, k


def test_oracle_lanczos_failure_matches_reference():
    """The reference raises LanczosConvergenceError when the proximal switch
    needs eigenpairs Lanczos cannot deliver in 100 steps; so does the oracle."""
    tr = load_traj("prox_lanczos_fail")
    assert str(tr["error"]) == "LanczosConvergenceError"
    prob = problem_for(tr)
    with pytest.raises(O.LanczosFailed):
        O.solve(prob, O.OracleConfig(max_iter=int(tr["max_iter"]), psqmr_switch_steps=int(tr["switch"])))
