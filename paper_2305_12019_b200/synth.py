"""Seeded synthetic stand-ins for the five BASELINE.json configurations.

The reference ships no datasets; BASELINE.json names
five synthetic shapes.  Each generator here is a pure function of
``(config, seed)``: noise for samples ``[b*BLOCK, (b+1)*BLOCK)`` is drawn from
its own Philox stream keyed by ``(seed, salt, b)``, so a shard that starts on
a block boundary can regenerate its columns independently.

Conventions: true labels alternate +1 (even i) /
-1 (odd i); a flip fraction f flips exactly round(f*n) labels chosen without
replacement; weights = compute_weights(y, q); e = 1; mu = 1.

The returned raw matrix X is a d x n ``SparseMatrixCSC`` (dense configs use
the zero-copy sample-major layout); ``make_problem`` applies the reference's
``scale_problem`` (reference ``solver.py:253-285``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from .sparse import SparseMatrixCSC

BLOCK = 1024


@dataclass(frozen=True)
class SynthConfig:
    name: str
    kind: str  # "gauss" | "ar1" | "sparse"
    d: int
    n: int
    q: float
    C: float
    signal_k: int = 0  # number of leading coordinates carrying the class shift
    shift: float = 0.0
    flip: float = 0.0
    ar_rho: float = 0.0
    density: float = 0.0
    wstar_k: int = 0
    label_noise: float = 0.0
    max_iter: int = 2000

    def scaled(self, d: Optional[int] = None, n: Optional[int] = None, **kw) -> "SynthConfig":
        """Same generator at a different size (proxies for tests)."""
        return replace(self, d=d or self.d, n=n or self.n,
                       name=f"{self.name}@{d or self.d}x{n or self.n}", **kw)


CONFIGS = {
    # BASELINE.json configs[0..4]
    "c1": SynthConfig("c1", "gauss", d=2000, n=1000, q=1.0, C=1.0,
                      signal_k=50, shift=1.0 / math.sqrt(50.0)),
    "c2": SynthConfig("c2", "gauss", d=20000, n=2000, q=1.0, C=10.0,
                      signal_k=200, shift=2.0 / math.sqrt(200.0), flip=0.10),
    "c3": SynthConfig("c3", "ar1", d=1000, n=200000, q=2.0, C=1.0,
                      signal_k=20, shift=0.3, ar_rho=0.5),
    "c4": SynthConfig("c4", "sparse", d=50000, n=500000, q=1.0, C=1.0,
                      density=0.001, wstar_k=500, label_noise=0.1),
    "c5": SynthConfig("c5", "gauss", d=20000, n=1000000, q=4.0, C=5.0,
                      signal_k=1000, shift=1.0 / math.sqrt(1000.0), flip=0.05),
}

_SALT = {"gauss": 11, "ar1": 13, "sparse": 17, "flip": 19, "wstar": 23, "noise": 29}


def _rng(seed: int, salt: int, block: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[int(seed) & (2**64 - 1), salt * 2**32 + block]))


def true_labels(n: int) -> np.ndarray:
    y = np.ones(n)
    y[1::2] = -1.0
    return y


def flip_labels(y: np.ndarray, frac: float, seed: int) -> np.ndarray:
    m = int(round(frac * y.size))
    if m == 0:
        return y.copy()
    idx = _rng(seed, _SALT["flip"], 0).choice(y.size, m, replace=False)
    out = y.copy()
    out[idx] = -out[idx]
    return out


def _mean_vector(cfg: SynthConfig) -> np.ndarray:
    mu = np.zeros(cfg.d)
    mu[: cfg.signal_k] = cfg.shift
    return mu


def dense_samples(cfg: SynthConfig, seed: int = 0, lo: int = 0, hi: Optional[int] = None) -> np.ndarray:
    """Row-major [hi-lo, d] samples x_i = y_true_i * mu + noise_i (lo on a block boundary)."""
    hi = cfg.n if hi is None else hi
    if lo % BLOCK:
        raise ValueError("shards must start on a BLOCK boundary")
    mu = _mean_vector(cfg)
    ytrue = true_labels(cfg.n)
    out = np.empty((hi - lo, cfg.d))
    salt = _SALT[cfg.kind]
    for b0 in range(lo, hi, BLOCK):
        b1 = min(b0 + BLOCK, hi)
        z = _rng(seed, salt, b0 // BLOCK).standard_normal((b1 - b0, cfg.d))
        if cfg.kind == "ar1":
            from scipy.signal import lfilter

            a = cfg.ar_rho
            z[:, 0] /= math.sqrt(1.0 - a * a)  # x_0 = z_0 (unit-variance start)
            z = lfilter([math.sqrt(1.0 - a * a)], [1.0, -a], z, axis=1)
        z += ytrue[b0:b1, None] * mu[None, :]
        out[b0 - lo: b1 - lo] = z
    return out


def sparse_matrix(cfg: SynthConfig, seed: int = 0):
    """Bernoulli(density) pattern, |N(0,1)| values, unit-norm columns (samples);
    labels sign(w*^T x + noise*N(0,1)), 0 -> +1.  Returns (X csc d x n, y)."""
    import scipy.sparse as sp

    d, n = cfg.d, cfg.n
    cols, rows, vals = [], [], []
    for b0 in range(0, n, BLOCK):
        b1 = min(b0 + BLOCK, n)
        g = _rng(seed, _SALT["sparse"], b0 // BLOCK)
        counts = g.binomial(d, cfg.density, size=b1 - b0)
        tot = int(counts.sum())
        cidx = np.repeat(np.arange(b0, b1, dtype=np.int64), counts)
        ridx = g.integers(0, d, size=tot, dtype=np.int64)
        key = np.unique(cidx * d + ridx)  # drop repeated positions; sorted by (col,row)
        c, r = key // d, key % d
        v = np.abs(g.standard_normal(key.size))
        cols.append(c), rows.append(r), vals.append(v)
    c = np.concatenate(cols); r = np.concatenate(rows); v = np.concatenate(vals)
    colptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(colptr, c + 1, 1)
    colptr = np.cumsum(colptr)
    # unit-norm columns
    nrm = np.sqrt(np.bincount(c, weights=v * v, minlength=n))
    nrm[nrm == 0.0] = 1.0
    v = v / nrm[c]
    x = SparseMatrixCSC(d, n, colptr, r, v)
    gw = _rng(seed, _SALT["wstar"], 0)
    wstar = np.zeros(d)
    wstar[gw.choice(d, cfg.wstar_k, replace=False)] = gw.standard_normal(cfg.wstar_k)
    score = x.scipy.T @ wstar + cfg.label_noise * _rng(seed, _SALT["noise"], 0).standard_normal(n)
    y = np.where(score >= 0.0, 1.0, -1.0)
    return x, y


def raw_data(cfg: SynthConfig, seed: int = 0):
    """(X as d x n SparseMatrixCSC, labels y) for a config."""
    if cfg.kind == "sparse":
        return sparse_matrix(cfg, seed)
    x = SparseMatrixCSC.from_dense_samples(dense_samples(cfg, seed))
    y = flip_labels(true_labels(cfg.n), cfg.flip, seed)
    return x, y


def make_problem(cfg: SynthConfig, seed: int = 0):
    """ProblemData for a config: weights from compute_weights, e = 1
    (reference ``solver.py:235-285``)."""
    from .solver import compute_weights, scale_problem

    x, y = raw_data(cfg, seed)
    tau = compute_weights(y, cfg.q)
    return scale_problem(x, y, None, cfg.C, cfg.q, tau=tau)


def make_variant_problem(cfgname: str, d: int, n: int, seed: int = 0, **var):
    """A scaled config with option / edge-case variations (test fixtures):
    ``q``, ``C``, ``shift`` override the config; ``e_random`` draws a
    max-normalised e in [0.2, 1]; ``holes`` (sparse) empties every 17th
    sample and feature 3.  Other keys (solver options) are ignored here."""
    import dataclasses

    from .solver import compute_weights, scale_problem
    from .sparse import csc_from_scipy

    cfg = CONFIGS[cfgname].scaled(d=d, n=n)
    over = {k: var[k] for k in ("q", "C", "shift") if k in var}
    if over:
        cfg = dataclasses.replace(cfg, **over)
    x, y = raw_data(cfg, seed)
    if var.get("holes") and not x.is_dense:
        m = x.scipy.tolil()
        m[:, ::17] = 0.0
        m[3, :] = 0.0
        x = csc_from_scipy(m.tocsc())
    e = None
    if var.get("e_random"):
        e = np.random.default_rng(seed + 99).uniform(0.2, 1.0, size=n)
        e[0] = 1.0
    return scale_problem(x, y, e, cfg.C, cfg.q, tau=compute_weights(y, cfg.q))


class DeviceProblemData:
    """ProblemData-compatible record whose Z~ exists only in HBM (configs that
    do not fit host memory).  Fields as ProblemData (solver.py:60-71) minus
    ``z_tilde``; ``y``/``e``/``weights`` are this rank's slices."""

    def __init__(self, dp, y, e, weights, C, q, z_scale, d, n_global):
        self.y, self.e, self.weights = y, e, weights
        self.C, self.q, self.z_scale = float(C), float(q), float(z_scale)
        self._d, self.n_global = int(d), int(n_global)
        self.z_tilde = None
        self._gdwd_device = dp

    @property
    def n(self) -> int:
        return self.y.size

    @property
    def d(self) -> int:
        return self._d

    def download_samples(self) -> np.ndarray:
        """Row-major [n, d] copy of the local Z~ (tests / proxies)."""
        from . import _lib
        from .solver import _check

        out = np.empty((self.n, self.d))
        dp = self._gdwd_device
        _check(dp.lib.gdwd_download_dense(dp.ctx, _lib.ptr(out)), dp.ctx, "download")
        return out


def make_device_problem(cfg: SynthConfig, seed: int = 0, device: int = 0, rank: int = 0, nranks: int = 1,
                        allreduce=None, comm=None) -> DeviceProblemData:
    """Generate a two-Gaussian config directly in HBM (counter-based stream,
    shard-consistent), scale it like scale_problem and register it for
    sgs_admm_solve.  With nranks > 1 this rank holds samples
    [n*rank/nranks, n*(rank+1)/nranks); ``allreduce`` sums the Frobenius norm
    across ranks and ``comm`` (parallel.*Communicator) shards the solve."""
    import ctypes as C

    from . import _lib
    from .solver import DeviceProblem, _check, compute_weights

    if cfg.kind != "gauss":
        raise ValueError("device generation covers the two-Gaussian configs")
    n = cfg.n
    lo, hi = n * rank // nranks, n * (rank + 1) // nranks
    dp = DeviceProblem(None, device)
    lib = dp.lib
    _check(lib.gdwd_generate_dense(dp.ctx, 0, int(seed) * 1000003 + 17, cfg.d, hi - lo, lo, cfg.signal_k,
                                   float(cfg.shift)), dp.ctx, "generate")
    dp.n, dp.d = hi - lo, cfg.d
    fro2 = C.c_double()
    _check(lib.gdwd_frobenius_sq(dp.ctx, C.byref(fro2)), dp.ctx, "frobenius")
    f2 = fro2.value if allreduce is None else float(allreduce(np.array([fro2.value]))[0])
    z_scale = math.sqrt(math.sqrt(f2))  # sqrt(||X||_F)  (solver.py:265-268)
    y_all = flip_labels(true_labels(n), cfg.flip, seed)
    tau = compute_weights(y_all, cfg.q)
    y = np.ascontiguousarray(y_all[lo:hi])
    w = np.ascontiguousarray((tau ** cfg.q)[lo:hi])
    e = np.ones(hi - lo)
    _check(lib.gdwd_scale_dense(dp.ctx, _lib.ptr(y), z_scale), dp.ctx, "scale")
    _check(lib.gdwd_set_problem(dp.ctx, _lib.ptr(y), _lib.ptr(e), _lib.ptr(w), float(cfg.C), float(cfg.q),
                                z_scale), dp.ctx, "set_problem")
    out = DeviceProblemData(dp, y, e, w, cfg.C, cfg.q, z_scale, cfg.d, n)
    if comm is not None:
        comm.attach(dp, n)
    return out


__all__ = ["BLOCK", "CONFIGS", "DeviceProblemData", "SynthConfig", "dense_samples", "flip_labels",
           "make_device_problem", "make_problem", "raw_data", "sparse_matrix", "true_labels"]
