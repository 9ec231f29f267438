"""Public-API behaviour on the device path that the reference defines
outside the numerics: callback contract and abort (solver.py:546), repeated
solves on a resident problem, max_iter edge, operand validation, backend
switches on one uploaded matrix."""

import numpy as np
import pytest

import paper_2305_12019_b200 as G
from conftest import load_traj, problem_for, relerr

pytestmark = pytest.mark.gpu


class Stop(Exception):
    pass


def test_callback_exception_propagates_and_context_recovers():
    prob = problem_for(load_traj("tiny_direct"))
    cfg = G.SolverConfig(q=prob.q, max_iter=50, backend=G.Backend.DIRECT)
    seen = []

    def cb(st, res):
        seen.append(st.iter)
        if st.iter == 7:
            raise Stop("user stop")

    with pytest.raises(Stop):
        G.sgs_admm_solve(prob, cfg, callback=cb)
    assert seen == list(range(1, 8))
    # the resident problem is still usable, and a fresh solve is unaffected
    a = G.sgs_admm_solve(prob, cfg)
    b = G.sgs_admm_solve(prob, cfg)
    assert a.iterations == 50 and np.array_equal(a.final_state.w, b.final_state.w)


def test_callback_sees_every_iteration_with_reference_fields():
    tr = load_traj("tiny_smw2")
    prob = problem_for(tr)
    cfg = G.SolverConfig(q=prob.q, max_iter=12, backend=G.Backend.SMW2)
    rows = []
    out = G.sgs_admm_solve(prob, cfg, callback=lambda st, res: rows.append((st.iter, st.sigma, res.eta_p)))
    assert [r[0] for r in rows] == list(range(1, 13))
    assert out.history.shape[0] == 12
    assert np.array_equal(np.array([r[1] for r in rows]), tr["hist"][:12, 11])


def test_max_iter_one_and_result_fields():
    tr = load_traj("tiny_iter")
    prob = problem_for(tr)
    out = G.sgs_admm_solve(prob, G.SolverConfig(q=prob.q, max_iter=1, backend=G.Backend.ITERATIVE))
    assert out.iterations == 1 and not out.converged
    assert out.backend_used.value == "iterative"
    assert out.final_state.w.shape == (prob.d,) and out.final_state.alpha.shape == (prob.n,)
    assert np.isfinite(out.final_state.beta)
    for key in ("w", "alpha", "r", "xi"):
        ref = tr["it_" + key][0]
        got = getattr(out.final_state, key)
        assert np.linalg.norm(got - ref) <= 1e-9 * max(np.linalg.norm(ref), 1e-300), key


def test_backend_switch_on_one_resident_matrix():
    """DIRECT, SMW2 and ITERATIVE on the same uploaded Z~ each reproduce the
    reference's backend-specific first iterate (factor caches keyed by backend)."""
    prob = problem_for(load_traj("tiny_direct"))
    outs = {}
    for be in (G.Backend.DIRECT, G.Backend.SMW2, G.Backend.ITERATIVE, G.Backend.DIRECT):
        outs.setdefault(be, []).append(G.sgs_admm_solve(prob, G.SolverConfig(q=prob.q, max_iter=15, backend=be)))
    d0, d1 = outs[G.Backend.DIRECT]
    assert np.array_equal(d0.final_state.w, d1.final_state.w)
    # exact solves agree with each other to rounding
    s = outs[G.Backend.SMW2][0]
    assert np.linalg.norm(s.final_state.w - d0.final_state.w) <= 1e-8 * np.linalg.norm(d0.final_state.w)


def test_matvec_operand_validation():
    prob = problem_for(load_traj("tiny_direct"))
    dp = G.solver.device_problem(prob)
    with pytest.raises(ValueError):
        dp.matvec(np.ones(prob.n + 1))
    with pytest.raises(ValueError):
        dp.rmatvec(np.ones(prob.d + 1))
    v = np.random.default_rng(0).standard_normal(prob.n)
    ref = prob.z_tilde.scipy @ v
    assert np.allclose(dp.matvec(v), ref, rtol=1e-13, atol=1e-13)


def test_csc_upload_validation_reports_first_error_in_sample_order():
    """gdwd_upload_csc validates on all host cores; the error reported is the
    one a sequential pass meets first (a sample's colptr before its row
    indices), with the reference's exception type (ValueError code)."""
    import ctypes as C

    from paper_2305_12019_b200 import _lib

    lib = _lib.load()
    ctx = C.c_void_p()
    assert lib.gdwd_ctx_create(0, C.byref(ctx)) == 0
    try:
        n, d, per = 20000, 300, 3
        rng = np.random.default_rng(5)
        colptr = np.arange(0, per * (n + 1), per, dtype=np.int64)
        rowidx = np.sort(rng.integers(0, d, size=(n, per)), axis=1).ravel().astype(np.int64)
        vals = rng.standard_normal(per * n)

        def up(cp, ri):
            return lib.gdwd_upload_csc(ctx, cp.ctypes.data_as(C.POINTER(C.c_int64)),
                                       ri.ctypes.data_as(C.POINTER(C.c_int64)), _lib.ptr(vals), d, n)

        assert up(colptr, rowidx) == 0
        bad_i = rowidx.copy()
        bad_i[per * 12345 + 1] = d  # index out of range at sample 12345
        bad_p = colptr.copy()
        bad_p[15000] = bad_p[15001] + 1  # colptr decreases at sample 15000
        assert up(colptr, bad_i) == 2
        assert b"row index out of bounds" in lib.gdwd_last_error(ctx)
        assert up(bad_p, rowidx) == 2
        assert b"nondecreasing" in lib.gdwd_last_error(ctx)
        both = bad_p.copy()
        assert up(both, bad_i) == 2  # the index error comes first in sample order
        assert b"row index out of bounds" in lib.gdwd_last_error(ctx)
        late_i = rowidx.copy()
        late_i[per * 17000] = -1
        assert up(bad_p, late_i) == 2  # the colptr error comes first
        assert b"nondecreasing" in lib.gdwd_last_error(ctx)
    finally:
        lib.gdwd_ctx_destroy(ctx)


def test_frobenius_after_pinned_upload_then_scale():
    """A pinned dense upload defers its ||X||_F^2 read-back; a later
    scale_dense must not be overwritten by that stale value."""
    import ctypes as C
    import math

    import torch

    from paper_2305_12019_b200 import _lib
    from paper_2305_12019_b200.solver import DeviceProblem, _check

    rng = np.random.default_rng(5)
    n, d = 300, 1600  # pinned + n <= d: the chunked overlapped upload path
    X = rng.standard_normal((n, d))
    pin = torch.empty(n * d, dtype=torch.float64, pin_memory=True).numpy()
    pin[:] = X.reshape(-1)
    dp = DeviceProblem(None, 0)
    lib = dp.lib
    _check(lib.gdwd_upload_dense(dp.ctx, _lib.ptr(pin), d, n), dp.ctx, "upload")
    y = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    zs = 7.5
    _check(lib.gdwd_scale_dense(dp.ctx, _lib.ptr(y), zs), dp.ctx, "scale")
    f2 = C.c_double()
    _check(lib.gdwd_frobenius_sq(dp.ctx, C.byref(f2)), dp.ctx, "fro")
    want = float(np.sum((X / zs) ** 2))
    assert math.isclose(f2.value, want, rel_tol=1e-12), (f2.value, want, float(np.sum(X * X)))
    dp.close()


def test_reference_problem_data_is_accepted_as_is():
    """Drop-in: a ProblemData shaped like the reference's (its own dataclass
    holding a CSC with int64 colptr/rowidx, solver.py:60-71, sparse.py:20-50)
    solves without conversion by the caller, dense and sparse."""
    from dataclasses import dataclass

    @dataclass(frozen=True)
    class RefCSC:
        nrows: int
        ncols: int
        colptr: np.ndarray
        rowidx: np.ndarray
        values: np.ndarray

    @dataclass(frozen=True)
    class RefProblem:
        z_tilde: RefCSC
        y: np.ndarray
        e: np.ndarray
        weights: np.ndarray
        C: float
        q: float
        z_scale: float

    for name in ("tiny_direct", "tiny_sparse"):
        prob = problem_for(load_traj(name))
        z = prob.z_tilde
        rz = RefCSC(z.nrows, z.ncols, np.array(z.colptr), np.array(z.rowidx), np.array(z.values))
        rp = RefProblem(rz, prob.y, prob.e, prob.weights, prob.C, prob.q, prob.z_scale)
        cfg = G.SolverConfig(q=prob.q, max_iter=15)
        a = G.sgs_admm_solve(prob, cfg)
        b = G.sgs_admm_solve(rp, cfg)
        assert G.as_problem(rp) is G.as_problem(rp)  # converted once, cached
        assert a.iterations == b.iterations and a.double_count == b.double_count
        assert np.array_equal(a.final_state.w, b.final_state.w)
        assert a.train_error_pct == b.train_error_pct
        kk = G.kkt_residuals(b.final_state, rp)
        assert np.isfinite(kk.eta_p)


@pytest.mark.parametrize("pin", [True, False])
@pytest.mark.parametrize("n,d,mu", [(200, 6000, 1.0), (16, 90, 1.0), (700, 3001, 2.0), (333, 777, 0.7), (1000, 2000, 1.0)])
def test_upload_time_gram_and_inverse(n, d, mu, pin):
    """A page-locked upload in the sample-space regimes forms K = Z~^T Z~
    (subsolvers.py:109) and G^{-1} = (K/mu^2 + I)^{-1} (cholesky.py:46,60-61)
    block by block while the samples are copied (gdwd_upload_hint +
    gdwd_upload_dense): both match numpy; K is exactly symmetric."""
    torch = pytest.importorskip("torch")
    import ctypes as C

    from paper_2305_12019_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, d)) * (3.0 / np.sqrt(d))
    # page-locked source: block-wise DMA; pageable (from 8 MB): staged by host threads
    buf = torch.empty(n * d, dtype=torch.float64, pin_memory=True).numpy() if pin else np.empty(n * d)
    buf[:] = X.ravel()
    h = C.c_void_p()
    assert lib.gdwd_ctx_create(0, C.byref(h)) == 0
    try:
        assert lib.gdwd_upload_hint(h, _lib.BACKEND_CODE["smw2"], mu) == 0
        assert lib.gdwd_upload_dense(h, _lib.ptr(buf), d, n) == 0
        K, Gi, have = np.empty((n, n)), np.empty((n, n)), C.c_int32()
        assert lib.gdwd_get_upload_factor(h, _lib.ptr(K), _lib.ptr(Gi), C.byref(have)) == 0
        if not pin and n * d < (1 << 20):
            assert have.value == 0  # small pageable sources take the plain copy
            return
        assert have.value == 3
        Kr = X @ X.T
        assert np.abs(K - Kr).max() <= 1e-13 * np.abs(Kr).max()
        assert np.array_equal(K, K.T)
        Gr = np.linalg.inv(Kr / mu ** 2 + np.eye(n))
        assert np.abs(Gi - Gr).max() <= 1e-12 * np.abs(Gr).max()
        assert np.array_equal(Gi, Gi.T)
        fro2 = C.c_double()
        assert lib.gdwd_frobenius_sq(h, C.byref(fro2)) == 0
        assert abs(fro2.value - (X * X).sum()) <= 1e-12 * (X * X).sum()
        # an ITERATIVE hint (also what the shards of a multi-GPU solve pass): plain copy
        assert lib.gdwd_upload_hint(h, _lib.BACKEND_CODE["iterative"], mu) == 0
        assert lib.gdwd_upload_dense(h, _lib.ptr(buf), d, n) == 0
        assert lib.gdwd_get_upload_factor(h, None, None, C.byref(have)) == 0
        assert have.value == 0
        back = np.empty_like(X)
        assert lib.gdwd_download_dense(h, _lib.ptr(back)) == 0
        assert np.array_equal(back, X)
    finally:
        lib.gdwd_ctx_destroy(h)


@pytest.mark.parametrize("d,n", [(1001, 9000), (300, 4001)])
def test_staged_pageable_upload_round_trip(d, n, monkeypatch):
    """A pageable [n][d] source of >= 8 MB outside the sample-space regimes is
    staged by host threads through the page-locked ring, several blocks deep
    (odd d: padded rows, 2-D copies): the device copy is the source, bit for
    bit, the products match numpy and the norm equals the plain path's."""
    rng = np.random.default_rng(d + n)
    S = rng.standard_normal((n, d))
    z = G.SparseMatrixCSC.from_dense_samples(S)
    ones = np.ones(n)
    dp = G.DeviceProblem(G.ProblemData(z, ones, ones, ones, 1.0, 1.0, 1.0))
    try:
        back = np.empty_like(S)
        from paper_2305_12019_b200 import _lib

        assert dp.lib.gdwd_download_dense(dp.ctx, _lib.ptr(back)) == 0
        assert np.array_equal(back, S)
        t, w = rng.standard_normal(n), rng.standard_normal(d)
        assert relerr(dp.matvec(t), S.T @ t) < 1e-13
        assert relerr(dp.rmatvec(w), S @ w) < 1e-13
        eps = dp.eps_c()
    finally:
        dp.close()
    monkeypatch.setenv("GDWD_UPLOAD", "pageable")  # the plain pageable copy
    dp = G.DeviceProblem(G.ProblemData(z, ones, ones, ones, 1.0, 1.0, 1.0))
    try:
        assert dp.eps_c() == eps
    finally:
        dp.close()


@pytest.mark.parametrize("pin", [False, True])
def test_direct_gram_summed_during_upload(pin, monkeypatch):
    """DIRECT's own regime (n >= 4 d): the d x d Gram Z~ Z~^T is summed block
    by block while the rows are copied (page-locked: block-wise DMA; pageable:
    staged).  The solve equals the one that forms the Gram afterwards."""
    from paper_2305_12019_b200 import synth

    prob = synth.make_variant_problem("c3", 300, 40000, seed=4)
    z = prob.z_tilde
    cfg = G.SolverConfig(q=prob.q, max_iter=20, backend=G.Backend.DIRECT)

    def solve():
        vals = z.values
        if pin:
            torch = pytest.importorskip("torch")
            vals = torch.empty(z.values.size, dtype=torch.float64, pin_memory=True).numpy()
            vals[:] = z.values
        zp = G.SparseMatrixCSC.from_dense_samples(vals.reshape(z.ncols, z.nrows))
        pp = G.ProblemData(zp, prob.y, prob.e, prob.weights, prob.C, prob.q, prob.z_scale)
        out = G.sgs_admm_solve(pp, cfg)
        G.solver.device_problem(pp).close()
        return out

    a = solve()
    monkeypatch.setenv("GDWD_UPLOAD_FACTOR", "0")
    b = solve()
    assert a.iterations == b.iterations == 20 and a.double_count == b.double_count
    assert a.setup_ms < b.setup_ms  # no Gram left in the setup
    for key in ("w", "u", "rho", "r", "xi", "alpha"):
        assert relerr(getattr(a.final_state, key), getattr(b.final_state, key)) < 1e-10, key
