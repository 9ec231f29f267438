"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference's sGS-ADMM hot path
(``/root/reference/pkg/src/gdwd``), used as the *checker* by ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``.  Nothing in the product package imports this module;
the product path is the CUDA library and fails loudly without it.

Parity pin: ``tests/golden/make_golden.py`` runs the reference package itself
(imported from /root/reference in the build container) on seeded problems
and commits its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this restatement against those fixtures (KATs from SPEC.md and
per-iteration trajectories for all three backends).

Every routine cites the reference line range it restates.  Arithmetic order
follows the reference expression by expression so that, with the default
``operator="csc"`` (scipy sparse products, like the reference), results agree
with the reference to the last bit or close to it.  ``operator="dense"`` swaps
the X products for dense BLAS (same math, different summation order; SURVEY.md
Appendix B) so large configurations finish in seconds.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np
import scipy.linalg as sla

TINY = 1e-300  # psqmr.py:14


# --------------------------------------------------------------------------
# small scalar rules
# --------------------------------------------------------------------------

def select_backend(n: int, d: int) -> str:
    """subsolvers.py:42-55 (integer test 5n < d for n < 0.2 d)."""
    if n < 1 or d < 1:
        raise ValueError("n and d must be at least 1")
    if d > 5000:
        return "smw2" if (5 * n < d and n <= 2500) else "iterative"
    return "direct"


def sigma_rule(sigma: float, eta_p: float, eta_d: float) -> float:
    """solver.py:343-362."""
    if eta_p == 0.0 and eta_d == 0.0:
        return sigma
    chi = math.inf if eta_d == 0.0 else eta_p / eta_d
    ichi = math.inf if eta_p == 0.0 else eta_d / eta_p
    worst = max(chi, ichi)
    zeta = 2.2 if worst > 500.0 else (1.65 if worst > 50.0 else 1.1)
    if chi > 5.0:
        return sigma * zeta
    if ichi > 5.0:
        return sigma / zeta
    return sigma


def class_weights(y: np.ndarray, q: float) -> np.ndarray:
    """solver.py:235-250."""
    y = np.asarray(y, dtype=np.float64)
    n = y.size
    npos, nneg = int(np.sum(y > 0)), int(np.sum(y < 0))
    if n < 2 or npos == 0 or nneg == 0:
        raise ValueError("need two classes and n >= 2")
    k = n / math.log(n)
    tp = (npos / k) ** (1.0 / (1.0 + q))
    tn = (nneg / k) ** (1.0 / (1.0 + q))
    top = max(tp, tn)
    return np.where(y > 0, tn / top, tp / top)


# --------------------------------------------------------------------------
# margin subproblem (subsolvers.py:264-364)
# --------------------------------------------------------------------------

def bisect_margin(a: float, sigma: float, q: float, wt: float, tol: float) -> float:
    """subsolvers.py:264-280."""
    lo = 1e-12
    hi = max(a, 0.0) + (q * wt / sigma) ** (1.0 / (q + 2.0)) + 1.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        g = sigma * (mid - a) - q * wt / mid ** (q + 1.0)
        if abs(g) <= tol:
            return mid
        if g < 0.0:
            lo = mid
        else:
            hi = mid
        if hi - lo <= 1e-17 * max(1.0, hi):
            break
    return 0.5 * (lo + hi)


def newton_scalar(a, sigma, q, wt, r0, tol=1e-12, max_newton=50):
    """subsolvers.py:283-318 -> (root, iterations)."""
    if sigma <= 0 or q <= 0 or wt <= 0 or r0 <= 0:
        raise ValueError("sigma, q, weight and r_init must be positive")
    c = q * wt / sigma
    s = float(r0)
    for it in range(max_newton + 1):
        if abs(-q * wt / s ** (q + 1.0) + sigma * (s - a)) <= tol:
            return s, it
        if it == max_newton:
            break
        sp1 = s ** (q + 1.0)
        nxt = s * ((q + 2.0) * c + a * sp1) / ((q + 1.0) * c + sp1 * s)
        if not np.isfinite(nxt) or nxt <= 0.0:
            return bisect_margin(a, sigma, q, wt, tol), it
        s = nxt
    return bisect_margin(a, sigma, q, wt, tol), max_newton


def newton_sweep(a, sigma, q, wts, r0, tol, max_newton=50, stats=None):
    """subsolvers.py:321-364: vectorised sweep.  The first activity test uses
    ``/ s**(q+1)``, later ones ``* s**(-(q+1))`` (the reference's two forms)."""
    s = np.array(r0, dtype=np.float64)
    a = np.asarray(a, dtype=np.float64)
    wts = np.asarray(wts, dtype=np.float64)
    c = q * wts / sigma
    live = np.abs(-q * wts / s ** (q + 1.0) + sigma * (s - a)) > tol
    sweeps = 0
    for _ in range(max_newton):
        if not live.any():
            break
        sweeps += 1
        idx = np.flatnonzero(live)
        si, ai = s[idx], a[idx]
        sp1 = si ** (q + 1.0)
        nxt = si * ((q + 2.0) * c[idx] + ai * sp1) / ((q + 1.0) * c[idx] + sp1 * si)
        bad = ~np.isfinite(nxt) | (nxt <= 0.0)
        for i in idx[bad]:
            s[i] = bisect_margin(float(a[i]), sigma, q, float(wts[i]), tol)
        idx, nxt = idx[~bad], nxt[~bad]
        s[idx] = nxt
        foc = -q * wts[idx] * nxt ** (-(q + 1.0)) + sigma * (nxt - a[idx])
        live[:] = False
        live[idx[np.abs(foc) > tol]] = True
    else:
        for i in np.flatnonzero(live):
            s[i] = bisect_margin(float(a[i]), sigma, q, float(wts[i]), tol)
    if stats is not None:
        stats["sweeps"] = sweeps
    return s


# --------------------------------------------------------------------------
# dense Cholesky (linalg/cholesky.py:25-66)
# --------------------------------------------------------------------------

class Indefinite(ArithmeticError):
    pass


def chol_upper(s: np.ndarray) -> np.ndarray:
    """cholesky.py:25-49 (no permutation branch: the solver never passes one)."""
    s = np.asarray(s, dtype=np.float64)
    if s.ndim != 2 or s.shape[0] != s.shape[1]:
        raise ValueError("expected a square matrix")
    scale = max(1.0, float(np.abs(s).max()) if s.size else 0.0)
    if not np.allclose(s, s.T, rtol=0.0, atol=1e-8 * scale):
        raise ValueError("matrix is not symmetric")
    try:
        return sla.cholesky(s, lower=False, check_finite=False)
    except np.linalg.LinAlgError as exc:
        raise Indefinite(str(exc)) from exc


def chol_apply(rf: np.ndarray, b: np.ndarray) -> np.ndarray:
    """cholesky.py:52-66: R^T z = b, then R x = z."""
    z = sla.solve_triangular(rf, b, trans="T", check_finite=False)
    return sla.solve_triangular(rf, z, trans="N", check_finite=False)


# --------------------------------------------------------------------------
# PSQMR (linalg/psqmr.py:27-95), exact recurrence
# --------------------------------------------------------------------------

@dataclass
class KrylovOut:
    x: np.ndarray
    iterations: int
    converged: bool
    breakdown: bool
    residual_norm: float


def psqmr(apply, b, precond=None, tol=1e-8, max_iter=None, x0=None) -> KrylovOut:
    b = np.asarray(b, dtype=np.float64)
    m = b.size
    max_iter = max(2 * m, 20) if max_iter is None else max_iter
    pre = precond if precond is not None else (lambda v: v)
    x = np.zeros(m) if x0 is None else np.array(x0, dtype=np.float64)
    warm = x0 is not None and np.any(x != 0.0)
    r = b - apply(x) if warm else b - 0.0
    res = r.copy()
    rn = float(np.linalg.norm(res))
    if rn <= tol:
        return KrylovOut(x, 0, True, False, rn)
    qv = pre(r)
    tau = float(np.linalg.norm(qv))
    rho = float(r @ qv)
    theta = 0.0
    dv = np.zeros(m)
    adv = np.zeros(m)
    done = brk = False
    it = 0
    for it in range(1, max_iter + 1):
        aq = apply(qv)
        sg = float(qv @ aq)
        if abs(sg) < TINY:
            brk = True
            it -= 1
            break
        al = rho / sg
        r = r - al * aq
        u = pre(r)
        th = float(np.linalg.norm(u)) / tau if tau > TINY else 0.0
        c2 = 1.0 / (1.0 + th * th)
        tau = tau * th * np.sqrt(c2)
        dv = (c2 * theta * theta) * dv + (c2 * al) * qv
        x = x + dv
        adv = (c2 * theta * theta) * adv + (c2 * al) * aq
        res = res - adv
        rn = float(np.linalg.norm(res))
        if rn <= tol:
            done = True
            break
        if abs(rho) < TINY:
            brk = True
            break
        rnew = float(r @ u)
        qv = u + (rnew / rho) * qv
        rho = rnew
        theta = th
    return KrylovOut(x, it, done, brk, rn)


# --------------------------------------------------------------------------
# Lanczos top-k (linalg/lanczos.py:33-133)
# --------------------------------------------------------------------------

class LanczosFailed(RuntimeError):
    def __init__(self, msg, best):
        super().__init__(msg)
        self.best = best


def _orth_start(rng, basis, dim):
    for _ in range(50):
        v = rng.standard_normal(dim)
        if basis:
            qm = np.column_stack(basis)
            v -= qm @ (qm.T @ v)
            v -= qm @ (qm.T @ v)
        nv = np.linalg.norm(v)
        if nv > 1e-8:
            return v / nv
    raise RuntimeError("could not generate a direction orthogonal to the basis")


def lanczos_topk(apply, dim, k, tol=1e-10, max_iter=None, seed=0):
    """Returns (eigenvalues descending, vectors d x k)."""
    if not 1 <= k < dim:
        raise ValueError("need 1 <= k < dim")
    cap = min(dim, max(10 * k, 100)) if max_iter is None else min(max_iter, dim)
    rng = np.random.default_rng(seed)
    basis, al, be = [], [], []
    v = _orth_start(rng, basis, dim)
    nest = 0.0
    best = None
    for _ in range(cap):
        w = apply(v)
        a = float(v @ w)
        w = w - a * v
        if basis and be and be[-1] != 0.0:
            w -= be[-1] * basis[-1]
        basis.append(v)
        al.append(a)
        qm = np.column_stack(basis)
        w -= qm @ (qm.T @ w)
        w -= qm @ (qm.T @ w)
        bn = float(np.linalg.norm(w))
        th, sv = sla.eigh_tridiagonal(np.asarray(al), np.asarray(be))
        nest = max(nest, float(np.abs(th).max()))
        top = np.argsort(th)[::-1][: min(k, len(al))]
        best = (th[top].copy(), qm @ sv[:, top])
        if len(al) >= k and (np.all(np.abs(bn * sv[-1, top]) <= tol * max(nest, 1e-300)) or len(al) == dim):
            return best
        if bn <= max(nest, 1.0) * 1e-14:
            if len(al) == dim:
                return best
            v = _orth_start(rng, basis, dim)
            be.append(0.0)
        else:
            v = w / bn
            be.append(bn)
    raise LanczosFailed(f"no convergence to tol={tol} within {cap} iterations", best)


# --------------------------------------------------------------------------
# operators on Z~ (the single operator seam, solver.py:410-411)
# --------------------------------------------------------------------------

class ZOp:
    """Z~ products.  ``csc``: scipy sparse (the reference's own routine);
    ``dense``: BLAS on the sample-major dense array."""

    def __init__(self, z, mode: str = "csc", gram: str = "same"):
        self.z = z
        self.d, self.n = z.nrows, z.ncols
        self.mode = mode
        self.gram = gram  # "dense": one-time Gram by dense BLAS (bench CPU leg only)
        if mode == "dense":
            self.S = z.dense_samples() if hasattr(z, "dense_samples") else z.toarray().T.copy()
        elif mode == "csc":
            self.zs = z.scipy
            self.zst = self.zs.T
        else:
            raise ValueError(mode)

    def mv(self, t):  # Z~ t   (n -> d)
        return self.S.T @ t if self.mode == "dense" else self.zs @ t

    def rmv(self, w):  # Z~^T w (d -> n)
        return self.S @ w if self.mode == "dense" else self.zst @ w

    def _dense(self):
        if self.mode == "dense":
            return self.S
        return self.z.dense_samples() if getattr(self.z, "is_dense", False) else self.z.toarray().T

    def zzt(self):
        if self.mode == "dense" or self.gram == "dense":
            S = self._dense()
            return S.T @ S
        return (self.zs @ self.zs.T).toarray()

    def ztz(self):
        if self.mode == "dense" or self.gram == "dense":
            S = self._dense()
            return S @ S.T
        return (self.zst @ self.zs).toarray()


# --------------------------------------------------------------------------
# the three normal-system backends (subsolvers.py:63-256)
# --------------------------------------------------------------------------

class DirectSys:
    """subsolvers.py:63-86 (``ar``: sum over sample shards)."""

    def __init__(self, op: ZOp, y, mu_sq, ar=None):
        ar = ar or (lambda v: v)
        d = op.d
        a = np.empty((d + 1, d + 1))
        a[:d, :d] = ar(op.zzt())
        a[:d, :d][np.diag_indices(d)] += mu_sq
        zy = ar(op.mv(y))
        a[:d, d] = zy
        a[d, :d] = zy
        a[d, d] = float(ar(np.array([float(y @ y)]))[0])
        self.A = a
        self.R = chol_upper(a)

    def solve(self, h):
        return chol_apply(self.R, h)


class SmwSys:
    """subsolvers.py:94-151."""

    def __init__(self, op: ZOp, y, mu_sq):
        self.op, self.y, self.mu_sq = op, y, float(mu_sq)
        g = op.ztz() / mu_sq
        g[np.diag_indices(op.n)] += 1.0
        self.G = g
        self.R = chol_upper(g)
        self.yy = float(y @ y)
        self.ynorm = np.sqrt(self.yy)
        gy = chol_apply(self.R, y / self.ynorm)
        self.jy = np.concatenate([gy, [-1.0]])
        self.ys = 1.0 + float((y / self.ynorm) @ gy) - 1.0

    def solve(self, h):
        op, y, n, d = self.op, self.y, self.op.n, self.op.d
        t1 = h[:d] / self.mu_sq
        t2 = h[d] / self.yy
        s1 = op.rmv(t1) + y * t2
        s2 = self.ynorm * t2
        js = np.concatenate([chol_apply(self.R, s1), [-s2]])
        dot = float((y / self.ynorm) @ js[:n]) + js[n]
        v = js - (dot / self.ys) * self.jy
        p1 = op.mv(v[:n])
        p2 = float(y @ v[:n]) + self.ynorm * v[n]
        x = np.empty(d + 1)
        x[:d] = t1 - p1 / self.mu_sq
        x[d] = t2 - p2 / self.yy
        return x


class ProxSys:
    """subsolvers.py:159-256 (closed-form inverse of Z Z^T + P + T)."""

    def __init__(self, op: ZOp, y, mu_sq, ell, seed=0, tol=1e-12, max_iter=None):
        d = op.d
        if d < 2:
            raise ValueError("proximal backend needs d >= 2")
        self.ell = min(ell, d - 1)
        self.mu_sq = float(mu_sq)
        self.lam, self.V = lanczos_topk(lambda v: op.mv(op.rmv(v)), d, self.ell, tol=tol,
                                        max_iter=max_iter, seed=seed)
        self.zy = op.mv(y)
        self.yty = float(y @ y)
        self.schur = np.nan
        self.schur = self.yty - float(self.zy @ self.inv(self.zy))

    def inv(self, v):
        base = 1.0 / (self.mu_sq + self.lam[-1])
        out = base * v
        if self.ell > 1:
            coef = 1.0 / (self.mu_sq + self.lam[:-1]) - base
            out += self.V[:, :-1] @ (coef * (self.V[:, :-1].T @ v))
        return out

    def fwd(self, v):
        out = (self.mu_sq + self.lam[-1]) * v
        if self.ell > 1:
            out += self.V[:, :-1] @ ((self.lam[:-1] - self.lam[-1]) * (self.V[:, :-1].T @ v))
        return out

    def solve(self, h):
        d = self.zy.size
        if not self.schur > 1e-14:
            raise ArithmeticError(f"Schur scalar {self.schur:.3e} is not safely positive")
        beta = (h[d] - float(self.zy @ self.inv(h[:d])))
        beta /= self.schur
        return np.concatenate([self.inv(h[:d] - self.zy * beta), [beta]])


# --------------------------------------------------------------------------
# KKT residuals and objectives (solver.py:293-340)
# --------------------------------------------------------------------------

KKT_FIELDS = ("eta_c1", "eta_c2", "eta_c3", "eta_p1", "eta_p2", "eta_p3",
              "eta_d1", "eta_d2", "eta_gap", "obj_primal", "obj_dual")


def kkt(op: ZOp, prob, st, mu, ar=None):
    """solver.py:311-340; returns a dict with the 11 KKT fields.  ``ar``:
    sum-all-reduce over sample shards (None: unsharded)."""
    ar = ar or (lambda v: v)

    def nsum(x):  # a sum over samples
        return float(ar(np.array([x]))[0])

    q, C = prob.q, prob.C
    y, e, wl = prob.y, prob.e, prob.weights
    one_c = 1.0 + C
    if nsum(float(np.any(st["r"] <= 0.0))) > 0:
        raise AssertionError("margin iterate left the positive orthant")
    r, xi, al, w, u, beta = st["r"], st["xi"], st["alpha"], st["w"], st["u"], st["beta"]
    ztw = op.rmv(w)
    s = q * wl / r ** (q + 1.0)
    pg = ztw + beta * y + xi - r
    out = dict(
        eta_c1=abs(nsum(float(y @ al))) / one_c,
        eta_c2=abs(nsum(float(xi @ (C * e - al)))) / one_c,
        eta_c3=nsum(float(np.sum((al - s) ** 2))) / one_c,
        eta_p1=float(np.sqrt(nsum(pg.dot(pg)))) / one_c,
        eta_p2=mu * float(np.linalg.norm(w - u)) / one_c,
        eta_p3=max(float(np.linalg.norm(w)) - prob.z_scale, 0.0) / one_c,
        eta_d1=float(np.sqrt(nsum(np.minimum(al, 0.0).dot(np.minimum(al, 0.0))))) / one_c,
        eta_d2=float(np.sqrt(nsum(np.maximum(al - C * e, 0.0).dot(np.maximum(al - C * e, 0.0))))) / one_c,
    )
    op_ = nsum(float(np.sum(wl / r ** q))) + C * nsum(float(e @ xi))
    kap = (q + 1.0) / q * q ** (1.0 / (q + 1.0))
    za = ar(op.mv(al))
    od = float(kap * nsum(float(np.sum(wl ** (1.0 / (q + 1.0)) * np.maximum(al, 0.0) ** (q / (q + 1.0)))))
               - prob.z_scale * np.linalg.norm(za))
    out["obj_primal"] = op_
    out["obj_dual"] = od
    out["eta_gap"] = abs(op_ - od) / (1.0 + abs(op_) + abs(od))
    return out


def eta_p(res):
    return max(res["eta_p1"], res["eta_p2"], res["eta_p3"])


def eta_d(res):
    return max(res["eta_d1"], res["eta_d2"])


def eta_c(res):
    return max(res["eta_c1"], res["eta_c2"], res["eta_c3"])


# --------------------------------------------------------------------------
# the main loop (solver.py:392-602)
# --------------------------------------------------------------------------

@dataclass
class OracleConfig:
    """Mirror of ``SolverConfig`` defaults (solver.py:101-116)."""
    max_iter: int = 2000
    steplength: float = 1.618
    tol_feas: float = 1e-5
    tol_cgap: float = math.sqrt(1e-5)
    tol_cap: float = 0.05
    sigma0: Optional[float] = None
    epsilon_c: Optional[float] = None
    backend: str = "auto"
    use_sgs: bool = True
    ell: int = 10
    mu: float = 1.0
    psqmr_switch_steps: int = 50
    seed: int = 0


@dataclass
class OracleResult:
    state: dict
    residuals: dict
    iterations: int
    converged: bool
    backend: str
    psqmr_total: int
    double_count: int
    history: list = field(default_factory=list)
    train_error_pct: float = 0.0
    setup_s: float = 0.0
    loop_s: float = 0.0
    timed_s: float = 0.0
    timed_iters: int = 0


def solve(prob, cfg: OracleConfig, operator: str = "csc",
          callback: Optional[Callable[[dict, dict], None]] = None,
          sigma_schedule: Optional[np.ndarray] = None, record: bool = True, gram: str = "same",
          time_after: Optional[int] = None, allreduce=None, n_global: Optional[int] = None) -> OracleResult:
    """solver.py:392-602.  ``sigma_schedule[k]`` (test hook)
    replaces update_sigma's output as the sigma of iteration k (k >= 1).

    ``allreduce`` (sum over sample shards) + ``n_global`` restate the sharded
    decomposition the device path uses (paper_2305_12019_b200/parallel.py):
    ``prob`` is then this rank's block of samples, every sum over samples is
    all-reduced and feature-space work is replicated."""
    import time

    t0 = time.perf_counter()
    op = ZOp(prob.z_tilde, operator, gram)
    n, d = op.n, op.d
    ar = allreduce or (lambda v: v)
    sharded = allreduce is not None
    ng = n if n_global is None else int(n_global)

    def nsum(x):  # a scalar summed over samples
        return float(ar(np.array([x]))[0])

    def zmv(t):  # Z~ t summed over the shards
        return ar(op.mv(t))
    q, C, mu = prob.q, prob.C, cfg.mu
    mu2 = mu * mu
    y, e, wl = prob.y, prob.e, prob.weights
    zs = prob.z_scale
    tau = cfg.steplength
    rn = math.sqrt(ng)
    kind = select_backend(ng, d) if cfg.backend == "auto" else cfg.backend
    zy = zmv(y)
    yty = nsum(float(y @ y))
    sysm = None
    jac = None
    if kind == "direct":
        sysm = DirectSys(op, y, mu2, ar=allreduce)
    elif kind == "smw2":
        if sharded:
            raise ValueError("SMW2 couples all samples: not sharded")
        sysm = SmwSys(op, y, mu2)
    else:
        jac = np.concatenate([ar(prob.z_tilde.row_sq_sums()) + mu2, [max(yty, mu2)]])
        jac = np.maximum(jac, 1e-12)

    def a_apply(v):
        hd, tl = v[:d], v[d]
        top = zmv(op.rmv(hd)) + mu2 * hd + zy * tl
        return np.concatenate([top, [float(zy @ hd) + yty * tl]])

    sigma = cfg.sigma0 if cfg.sigma0 is not None else min(10.0 * C, float(ng)) ** q
    if cfg.epsilon_c is not None:
        epsc = cfg.epsilon_c
    elif sharded:
        epsc = 1.0 / max(1.0, math.sqrt(nsum(float(np.sum(prob.z_tilde.values * prob.z_tilde.values)))))
    else:
        epsc = 1.0 / max(1.0, prob.z_tilde.frobenius_norm())
    r = np.ones(n); xi = np.ones(n); al = np.zeros(n)
    w = np.zeros(d); u = np.zeros(d); rho = np.zeros(d)
    beta = 0.0
    ztw = np.zeros(n)
    ptot = dcount = 0
    conv = False
    prox = None
    setup_s = time.perf_counter() - t0
    last_steps = [0]

    def sys_solve(ht, hb, tol, x0, aw, aztw):
        nonlocal prox, ptot
        if kind == "direct" or kind == "smw2":
            return sysm.solve(np.concatenate([ht, [hb]]))
        if prox is None:
            o = psqmr(a_apply, np.concatenate([ht, [hb]]), precond=lambda v: v / jac, tol=tol,
                      max_iter=cfg.psqmr_switch_steps, x0=x0)
            ptot += o.iterations
            last_steps[0] += o.iterations
            if o.converged:
                return o.x
            prox = ProxSys(op, y, mu2, cfg.ell, seed=cfg.seed)
        shift = prox.fwd(aw) - mu2 * aw - zmv(aztw)
        return prox.solve(np.concatenate([ht + shift, [hb]]))

    hist = []
    t1 = time.perf_counter()
    res = None
    st = None
    t_mark = None
    for k in range(cfg.max_iter):
        if time_after is not None and k == time_after:
            t_mark = time.perf_counter()
        last_steps[0] = 0
        eps = epsc / (k + 1.0) ** 1.5
        rhs = xi - r - al / sigma
        ht = -zmv(rhs) + mu2 * u + (mu / sigma) * rho
        hb = -nsum(float(y @ rhs))
        x = sys_solve(ht, hb, eps, np.concatenate([w, [beta]]), w, ztw)
        wb, bb = x[:d], float(x[d])
        ztwb = op.rmv(wb)
        cvec = ztwb + y * bb + xi - al / sigma
        rnew = newton_sweep(cvec, sigma, q, wl, r, tol=eps / rn)
        reused = True
        if cfg.use_sgs:
            dr = rnew - r
            h2t = ht + zmv(dr)
            h2b = hb + nsum(float(y @ dr))
            if prox is not None:
                shift = prox.fwd(w) - mu2 * w - zmv(ztw)
                axt = prox.fwd(wb) + zy * bb
                rt = h2t + shift - axt
            else:
                axt = zmv(ztwb) + mu2 * wb + zy * bb
                rt = h2t - axt
            rb = h2b - (float(zy @ wb) + yty * bb)
            if math.hypot(float(np.linalg.norm(rt)), rb) <= 5.0 * eps:
                w, beta, ztw = wb, bb, ztwb
            else:
                reused = False
                dcount += 1
                x2 = sys_solve(h2t, h2b, 5.0 * eps, np.concatenate([wb, [bb]]), w, ztw)
                w, beta = x2[:d], float(x2[d])
                ztw = op.rmv(w)
        else:
            w, beta, ztw = wb, bb, ztwb
        r = rnew
        g = w - rho / (sigma * mu)
        gn = float(np.linalg.norm(g))
        u = g if gn <= zs else (zs / gn) * g
        xi = np.maximum(0.0, r - ztw - y * beta + al / sigma - (C / sigma) * e)
        pg = ztw + y * beta + xi - r
        al = al - (tau * sigma) * pg
        rho = rho - (tau * sigma * mu) * (w - u)
        st = dict(r=r, xi=xi, alpha=al, w=w, u=u, rho=rho, beta=beta, sigma=sigma, iter=k + 1, eps_c=epsc)
        res = kkt(op, prob, st, mu, ar=allreduce)
        if record:
            hist.append(dict(res, sigma=sigma, beta=beta, reused=reused, psqmr_steps=last_steps[0], eps=eps))
        if callback is not None:
            callback(st, res)
        if (max(eta_p(res), eta_d(res)) < cfg.tol_feas and min(eta_c(res), res["eta_gap"]) < cfg.tol_cgap
                and max(eta_c(res), res["eta_gap"]) < cfg.tol_cap):
            conv = True
            break
        if sigma_schedule is not None and k + 1 < len(sigma_schedule):
            sigma = float(sigma_schedule[k + 1])
        else:
            sigma = sigma_rule(sigma, eta_p(res), eta_d(res))
    t_end = time.perf_counter()
    loop_s = t_end - t1
    scores = beta + y * ztw
    terr = 100.0 * nsum(float(np.sum(y * np.sign(scores) <= 0.0))) / ng
    return OracleResult(state=st, residuals=res, iterations=st["iter"], converged=conv, backend=kind,
                        psqmr_total=ptot, double_count=dcount, history=hist, train_error_pct=terr,
                        setup_s=setup_s, loop_s=loop_s,
                        timed_s=(t_end - t_mark) if t_mark is not None else loop_s,
                        timed_iters=(st["iter"] - time_after) if t_mark is not None else st["iter"])


# ---------------------------------------------------------------------------
# Penalty parameter (solver.py:190-232)
# ---------------------------------------------------------------------------
def penalty_C(x_csc, y, q, seed=0, limit=2000):
    """solver.py:193-232: C from the median between-class distance; classes
    subsampled (default_rng(seed).choice, sorted) beyond `limit`; exact zero
    distances dropped.  Returns (C, dist)."""
    y = np.asarray(y, dtype=np.float64)
    n = y.size
    pos = np.flatnonzero(y > 0)
    neg = np.flatnonzero(y < 0)
    if pos.size == 0 or neg.size == 0:
        raise ValueError("single class")
    rng = np.random.default_rng(seed)
    if pos.size > limit:
        pos = np.sort(rng.choice(pos, limit, replace=False))
    if neg.size > limit:
        neg = np.sort(rng.choice(neg, limit, replace=False))
    a = x_csc[:, pos]
    b = x_csc[:, neg]
    sq_a = np.asarray(a.multiply(a).sum(axis=0)).ravel()
    sq_b = np.asarray(b.multiply(b).sum(axis=0)).ravel()
    d2 = sq_a[:, None] + sq_b[None, :] - 2.0 * (a.T @ b).toarray()
    np.maximum(d2, 0.0, out=d2)
    dists = np.sqrt(d2.ravel())
    dists = dists[dists > 0.0]
    if dists.size == 0:
        raise ValueError("all between-class distances are zero")
    dist = float(np.median(dists))
    c = 10.0 ** (q + 1.0) * max(1.0, 10.0 ** (q - 1.0) * math.log(n) * max(1000.0, float(x_csc.shape[0]))
                                ** (1.0 / 3.0) / dist ** (q + 1.0))
    return c, dist


# ---------------------------------------------------------------------------
# Applying a model (solver.py:610-642)
# ---------------------------------------------------------------------------
def decision_values(w_composite, beta, x_csc):
    """solver.py:610-629: beta + x^T w with the weights padded with zeros or
    cut to the input dimension (x: scipy CSC, features x samples)."""
    d_in, d_tr = x_csc.shape[0], w_composite.size
    if d_in == d_tr:
        w_eff = w_composite
    elif d_in > d_tr:
        w_eff = np.concatenate([w_composite, np.zeros(d_in - d_tr)])
    else:
        w_eff = w_composite[:d_in]
    return beta + x_csc.T @ w_eff


def predict(w_composite, beta, x_csc):
    """solver.py:632-636: where(score > 0, +1, -1) (zero -> -1, as the code does)."""
    return np.where(decision_values(w_composite, beta, x_csc) > 0.0, 1.0, -1.0)


def train_error(w_composite, beta, x_csc, y):
    """solver.py:639-642: y sign(score) <= 0 is wrong (zero scores included)."""
    y = np.asarray(y, dtype=np.float64)
    return 100.0 * float(np.mean(y * np.sign(decision_values(w_composite, beta, x_csc)) <= 0.0))


__all__ = ["DirectSys", "KKT_FIELDS", "KrylovOut", "OracleConfig", "OracleResult", "ProxSys",
           "SmwSys", "ZOp", "bisect_margin", "penalty_C", "chol_apply", "chol_upper", "class_weights", "decision_values", "kkt",
           "lanczos_topk", "newton_scalar", "newton_sweep", "predict", "psqmr", "select_backend", "sigma_rule",
           "solve", "train_error"]
