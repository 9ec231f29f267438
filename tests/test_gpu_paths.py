"""Every alternative device path against the reference's trajectories
(pytest -m gpu).  The default plan picks one path per problem shape, so the
small fixtures alone would leave some paths unexercised:

* the fused tail pass (zft.cuh) is planned only for tiles >= 32 KB: forced on
  here (GDWD_FT_FORCE) for every dense X-space fixture, in its one-CTA form
  and in its cluster form (GDWD_FT_CS=2: DSMEM exchange);
* the CSR gather Z~ t (the fallback when the sample-blocked layout does not
  fit): GDWD_SP_SB=0 on the sparse fixtures;
* the host-driven PSQMR loop (used for sharded solves): GDWD_PSQMR_GRAPH=0.

Same bars as tests/test_gpu_parity.py: first 20 iterates to 1e-9; whole runs
under sigma replay with the reference's iteration count, re-solve count and
PSQMR total exactly and final w within 1e-6."""

import numpy as np
import pytest

import paper_2305_12019_b200 as G
from conftest import TRAJ_CASES, VAR_CASES, load_traj, problem_for, relerr
from test_gpu_parity import config_for, run_traj

pytestmark = pytest.mark.gpu
TOL20 = 1e-9


def _x_space_dense(tr, case):
    prob = problem_for(tr)
    if not prob.z_tilde.is_dense:
        return None
    return prob


def _check(case, tr, prob, **kw):
    cfg = config_for(case, tr, prob)
    out, h, vecs = run_traj(prob, cfg, bool(tr["full"]), tr["idx_d"], tr["idx_n"], **kw)
    k = min(20, len(tr["hist"]))
    for key in ("w", "u", "rho", "r", "xi", "alpha"):
        for i in range(k):
            assert relerr(vecs[key][i], tr["it_" + key][i]) < TOL20, (key, i)
    out2 = G.sgs_admm_solve(prob, cfg, sigma_schedule=tr["hist"][:, 11], **kw)
    assert out2.iterations == int(tr["iterations"]) and out2.converged == bool(tr["converged"])
    assert out2.double_count == int(tr["double_count"])
    assert out2.psqmr_total == int(tr["psqmr_total"])
    assert relerr(out2.final_state.w, tr["final_w"]) < 1e-6


@pytest.mark.parametrize("cs", ["1", "2"])
@pytest.mark.parametrize("case", TRAJ_CASES + VAR_CASES)
def test_fused_tail_forced(case, cs, monkeypatch):
    tr = load_traj(case)
    prob = _x_space_dense(tr, case)
    if prob is None:
        pytest.skip("sparse fixture: no dense X pass to fuse")
    monkeypatch.setenv("GDWD_FT_FORCE", "1")
    monkeypatch.setenv("GDWD_FT_CS", cs)
    # Gram-space SMW2 / DIRECT-in-sample-space never read X: iterate over X
    _check(case, tr, prob, smw_gram_space=False)


@pytest.mark.parametrize("case", [c for c in TRAJ_CASES + VAR_CASES if "sparse" in c])
def test_sparse_csr_gather_fallback(case, monkeypatch):
    monkeypatch.setenv("GDWD_SP_SB", "0")
    tr = load_traj(case)
    prob = problem_for(tr)  # uploaded fresh in this context: the setting is read at context creation
    _check(case, tr, prob)


@pytest.mark.parametrize("case", ["tiny_iter", "tiny_iter_c4gen", "iter_natural", "tiny_sparse", "sparse_natural",
                                  "prox_tiny", "prox_tiny_q2", "var_converge_iter", "var_min_iter"])
def test_host_driven_psqmr(case, monkeypatch):
    monkeypatch.setenv("GDWD_PSQMR_GRAPH", "0")
    tr = load_traj(case)
    _check(case, tr, problem_for(tr))
