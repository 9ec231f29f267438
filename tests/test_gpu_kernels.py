"""GPU kernel parity through the C ABI (run on a B200: pytest -m gpu)."""

import ctypes

import numpy as np
import pytest

import paper_2305_12019_b200 as G
from conftest import load_kat, relerr
from oracle import gdwd_oracle as O
from paper_2305_12019_b200 import linalg as L

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,n", [(2000, 1000), (1001, 37), (9000, 300), (17, 5000), (64, 1)])
def test_matvec_both_directions(d, n):
    rng = np.random.default_rng(d * 7 + n)
    S = rng.standard_normal((n, d))  # sample-major [n, d] = CSC values of Z (d x n)
    z = G.SparseMatrixCSC.from_dense_samples(S)
    t = rng.standard_normal(n)
    w = rng.standard_normal(d)
    ones = np.ones(n)
    dp = G.DeviceProblem(G.ProblemData(z, ones, ones, ones, 1.0, 1.0, 1.0))
    try:
        assert relerr(dp.matvec(t), S.T @ t) < 1e-13
        assert relerr(dp.rmatvec(w), S @ w) < 1e-13
        # deterministic: same bits twice
        assert np.array_equal(dp.matvec(t), dp.matvec(t))
        assert np.array_equal(dp.rmatvec(w), dp.rmatvec(w))
    finally:
        dp.close()


@pytest.mark.parametrize("d,n,dens", [(3000, 2000, 0.001), (500, 7000, 0.02), (40, 30, 0.3)])
def test_sparse_matvec_both_directions(d, n, dens):
    import scipy.sparse as sp

    rng = np.random.default_rng(d + n)
    M = sp.random(d, n, density=dens, format="csc", random_state=rng, data_rvs=rng.standard_normal)
    z = G.sparse.csc_from_scipy(M)
    assert not z.is_dense
    ones = np.ones(n)
    dp = G.DeviceProblem(G.ProblemData(z, ones, ones, ones, 1.0, 1.0, 1.0))
    try:
        t = rng.standard_normal(n)
        w = rng.standard_normal(d)
        assert relerr(dp.matvec(t), M @ t) < 1e-13
        assert relerr(dp.rmatvec(w), M.T @ w) < 1e-13
        assert np.array_equal(dp.matvec(t), dp.matvec(t))
    finally:
        dp.close()


@pytest.mark.parametrize("d,n,dens", [(20000, 1000, 0.002), (30000, 90000, 0.0005), (8193, 297, 0.01)])
@pytest.mark.parametrize("blocked", ["1", "0"])
def test_sparse_rmatvec_feature_blocked(d, n, dens, blocked, monkeypatch):
    """Z~^T w through the feature-blocked sliced-ELL kernel (spops.cuh) and the
    plain CSC kernel: several feature blocks of 8192, fewer samples than CTA
    parts, a sample count that does not divide, empty samples."""
    import scipy.sparse as sp

    monkeypatch.setenv("GDWD_SP_BLOCKED", blocked)
    rng = np.random.default_rng(d + n)
    M = sp.random(d, n, density=dens, format="csc", random_state=rng, data_rvs=rng.standard_normal)
    z = G.sparse.csc_from_scipy(M)
    ones = np.ones(n)
    dp = G.DeviceProblem(G.ProblemData(z, ones, ones, ones, 1.0, 1.0, 1.0))
    try:
        for _ in range(2):
            w = rng.standard_normal(d)
            got = dp.rmatvec(w)
            ref = M.T @ w
            assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(M).T @ np.abs(w))
            assert np.array_equal(got, dp.rmatvec(w))
    finally:
        dp.close()


@pytest.mark.parametrize("rows,cols", [(1000, 300), (130, 2001), (5, 70)])
def test_gram_dmma(rows, cols):
    rng = np.random.default_rng(rows + cols)
    X = rng.standard_normal((rows, cols))
    g1 = L.gram(X, True, div=1.0, shift=0.5)
    assert relerr(g1, X.T @ X + 0.5 * np.eye(cols)) < 1e-13
    g2 = L.gram(X, False, div=4.0, shift=1.0)
    assert relerr(g2, X @ X.T / 4.0 + np.eye(rows)) < 1e-13
    assert np.array_equal(g1, g1.T)


@pytest.mark.parametrize("m", [2, 63, 64, 65, 300, 2001])
def test_cholesky_inverse(m):
    rng = np.random.default_rng(m)
    B = rng.standard_normal((m, m))
    S = B @ B.T + m * np.eye(m)
    inv = L.cholesky_inverse(S)
    assert relerr(inv, np.linalg.inv(S)) < 1e-12


@pytest.mark.parametrize("m,block", [(2, 128), (100, 128), (129, 128), (300, 37), (1001, 128), (2000, 128),
                                     (2000, 96), (777, 200)])
def test_cholesky_inverse_bordered(m, block):
    """The row-block chain of the pipelined upload (gram.cu bordered_chol_step):
    rows of L^{-1} block by block, G^{-1} accumulated as rank-`block` updates."""
    rng = np.random.default_rng(m)
    B = rng.standard_normal((m, m))
    S = B @ B.T + m * np.eye(m)
    inv = L.cholesky_inverse(S, block=block)
    assert relerr(inv, np.linalg.inv(S)) < 1e-12
    assert np.array_equal(inv, inv.T)
    with pytest.raises(G.IndefiniteMatrixError):
        L.cholesky_inverse(np.array([[1.0, 2.0], [2.0, 1.0]]), block=128)


@pytest.mark.parametrize("m", [64, 200, 1000])
def test_cholesky_inverse_ill_conditioned(m):
    """Eigenvalues spread over 1e0..1e8: the leaf panels' rsqrt pivots and
    rank-8 updates keep the inverse at numpy's backward-stable accuracy."""
    rng = np.random.default_rng(m + 7)
    Q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    S = (Q * np.logspace(0, 8, m)) @ Q.T
    S = (S + S.T) / 2
    inv = L.cholesky_inverse(S)
    ref = np.linalg.inv(S)
    assert relerr(inv, ref) < 1e-7
    assert relerr(inv @ S, np.eye(m)) < 1e-7


def test_cholesky_kat_and_indefinite():
    S = np.array([[4.0, 2.0], [2.0, 3.0]])
    x = L.cholesky_inverse(S) @ np.array([6.0, 5.0])
    assert np.allclose(x, load_kat()["cholesky"]["solve"], rtol=0, atol=1e-14)
    with pytest.raises(G.IndefiniteMatrixError):
        L.cholesky_inverse(np.array([[1.0, 2.0], [2.0, 1.0]]))


def test_newton_kats():
    for a, s, q, w, r0, root, its in load_kat()["newton_r"]:
        got, git = G.newton_r(a, s, q, w, r0)
        assert got == pytest.approx(root, rel=1e-15, abs=0) and git == its


@pytest.mark.parametrize("q", [1.0, 2.0, 4.0, 0.5])
def test_newton_sweep_vs_oracle(q):
    rng = np.random.default_rng(int(q * 10))
    n = 20000
    a = rng.standard_normal(n) * 3
    r0 = rng.random(n) * 2 + 0.05
    w = rng.random(n) + 0.1
    for sigma in (0.5, 10.0, 3e5):
        ref = O.newton_sweep(a, sigma, q, w, r0, tol=1e-6)
        got = G.newton_r_sweep(a, sigma, q, w, r0, tol=1e-6)
        assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-13


@pytest.mark.parametrize("q", [1.0, 2.0, 0.5])
def test_newton_sweep_bisection_regime(q):
    """Large sigma (config 2 drives it past 1e12): |foc| <= tol needs s to
    better than an ulp, Newton stalls on a fixed point or 2-cycle and the
    reference finishes in its 200-step bisection.  The device leaves both
    loops once their state repeats; the roots must not move."""
    rng = np.random.default_rng(int(q * 100))
    n = 1500
    a = rng.standard_normal(n) * 3
    r0 = rng.random(n) * 2 + 0.05
    w = rng.random(n) + 0.1
    for sigma, tol in ((1e10, 1e-7), (1e13, 1e-8), (3e15, 1e-9)):
        ref = O.newton_sweep(a, sigma, q, w, r0, tol=tol)
        got = G.newton_r_sweep(a, sigma, q, w, r0, tol=tol)
        assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-13
    for i in range(40):  # scalar form: root and the reported Newton count
        ref, rit = O.newton_scalar(float(a[i]), 1e13, q, float(w[i]), float(r0[i]), tol=1e-8)
        got, git = G.newton_r(float(a[i]), 1e13, q, float(w[i]), float(r0[i]), tol=1e-8)
        assert got == pytest.approx(ref, rel=1e-13, abs=0) and git == rit


def _newton_dev(a, sigma, q, w, r0, tol, form):
    from paper_2305_12019_b200 import _lib
    a, w, r0 = (np.ascontiguousarray(v, dtype=np.float64) for v in (a, w, r0))
    out = np.empty_like(a)
    its = np.zeros(a.size, dtype=np.int32)
    lib = _lib.load()
    assert lib.gdwd_newton_sweep(0, a.size, _lib.ptr(a), float(sigma), float(q), _lib.ptr(w), _lib.ptr(r0),
                                 float(tol), 50, form, _lib.ptr(out),
                                 its.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))) == 0
    return out, its


@pytest.mark.parametrize("q", [1.0, 2.0, 4.0, 0.5])
def test_newton_warp_form_matches(q):
    """The warp-cooperative Newton + bisection (persistent kernel) returns the
    per-thread form's roots bit for bit, and its Newton counts, in every
    regime (converging Newton, stalled Newton + bisection)."""
    rng = np.random.default_rng(int(q * 7))
    n = 4000
    a = rng.standard_normal(n) * 3
    r0 = rng.random(n) * 2 + 0.05
    w = rng.random(n) + 0.1
    for sigma, tol in ((0.5, 1e-6), (3e5, 1e-6), (1e13, 1e-8), (3e15, 1e-9)):
        for form in (0, 1):
            ref, rit = _newton_dev(a, sigma, q, w, r0, tol, form)
            got, git = _newton_dev(a, sigma, q, w, r0, tol, form | 2)
            assert np.array_equal(got, ref) and np.array_equal(git, rit)
        o = O.newton_sweep(a[:300], sigma, q, w[:300], r0[:300], tol=tol)
        assert np.max(np.abs(got[:300] - o) / np.abs(o)) < 1e-13


def test_psqmr_kats():
    k = load_kat()
    p = L.psqmr_dense(np.diag([1.0, 2.0, 3.0]), np.array([1.0, 2.0, 3.0]), tol=1e-12)
    assert p.iterations == k["psqmr_diag"]["iterations"] and p.converged
    assert np.allclose(p.x, k["psqmr_diag"]["x"], rtol=0, atol=1e-14)
    rng = np.random.default_rng(7)
    B = rng.standard_normal((50, 50))
    S = B @ B.T + 50 * np.eye(50)
    b = rng.standard_normal(50)
    M = np.diag(S).copy()
    p2 = L.psqmr_dense(S, b, precond_diag=M, tol=1e-10, max_iter=200)
    ref = k["psqmr_spd50"]
    assert p2.iterations == ref["iterations"] and p2.converged
    assert relerr(p2.x, ref["x"]) < 1e-12
