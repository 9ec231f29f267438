"""Full-size final-state fixtures: run the REFERENCE to its stopping rule or
max_iter on BASELINE.json configs 2-4 and a config-5 proxy.

Build container only (imports /root/reference/pkg/src; the GPU box never runs
this).  The reference is run unmodified except, for the dense configs, the
operator swap of SURVEY.md Appendix B: ``z_tilde.scipy`` is replaced by a
dense-BLAS object with the same ``@`` / ``.T`` / ``.toarray()`` surface (same
math, different summation order; the scipy CSC path would take hours to
days on c2/c3 -- SURVEY section 6).  The sparse config 4 runs as-is.

    python tests/golden/make_golden_full.py --only c2 [--threads 4]

Each ``full_<name>.npz`` holds
  hist           per-iteration scalars (reference callback, solver.py:546):
                 eta_c1..eta_gap, obj_primal, obj_dual, sigma, beta, iter,
                 ||w||, ||alpha|| -- column 11 is the sigma trace that the GPU
                 test replays
  w1, w20        the full w iterate after iterations 1 and 20
  s20_{alpha,r,xi}, idx_n   sampled n-space coordinates after iteration 20
  final_w, final_beta, obj_primal, obj_dual, iterations, converged,
  double_count, psqmr_total, train_error, backend, z_sha, solve_time
Targets: reference solver.py:548-602 (stopping rule, SolveResult).
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, "/root/reference/pkg/src")

ap = argparse.ArgumentParser()
ap.add_argument("--only", required=True)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--max-iter", type=int, default=2000)
ARGS = ap.parse_args()
if ARGS.threads:
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = str(ARGS.threads)

import numpy as np  # noqa: E402

import gdwd  # noqa: E402  (the reference)
from gdwd.linalg import SparseMatrixCSC as RefCSC  # noqa: E402

from paper_2305_12019_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent

# name -> (synth config, d, n, operator)
FULL = {
    "c2": ("c2", None, None, "dense"),
    "c3": ("c3", None, None, "dense"),
    "c4": ("c4", None, None, "csc"),
    "c5p": ("c5", 6000, 30000, "dense"),   # config-5 proxy: d > 5000, d <= n/4 -> ITERATIVE, Gram operator
}
NSAMPLE = 4096


class _Gram:
    def __init__(self, a):
        self.a = a

    def toarray(self):
        return self.a


class DenseZT:
    """Z~^T of a sample-major [n, d] array S."""

    def __init__(self, S):
        self.S = S
        self.shape = (S.shape[0], S.shape[1])

    def __matmul__(self, v):
        if isinstance(v, DenseZ):  # Z~^T Z~ (build_smw, subsolvers.py:109)
            return _Gram(self.S @ self.S.T)
        return self.S @ v


class DenseZ:
    """Stand-in for ``SparseMatrixCSC.scipy`` (sparse.py:52-57) over dense data."""

    def __init__(self, S):
        self.S = S
        self.shape = (S.shape[1], S.shape[0])

    @property
    def T(self):
        return DenseZT(self.S)

    def __matmul__(self, v):
        if isinstance(v, DenseZT):  # Z~ Z~^T (build_direct, subsolvers.py:76)
            return _Gram(self.S.T @ self.S)
        return self.S.T @ v


def z_checksum(values: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(values).tobytes()).hexdigest()[:16]


def problem(name):
    cfgname, d, n, _ = FULL[name]
    cfg = synth.CONFIGS[cfgname]
    if d is not None:
        cfg = cfg.scaled(d=d, n=n)
    return synth.make_problem(cfg, 0)


def main():
    name = ARGS.only
    cfgname, _, _, operator = FULL[name]
    t0 = time.perf_counter()
    prob = problem(name)
    z = prob.z_tilde
    print(f"{name}: generated d={z.nrows} n={z.ncols} in {time.perf_counter() - t0:.1f}s", flush=True)
    if operator == "dense":
        # the reference object keeps its (unused) index arrays small: the operator
        # seam and the two direct value reductions are all the solver touches
        rz = RefCSC.__new__(RefCSC)
        object.__setattr__(rz, "nrows", z.nrows)
        object.__setattr__(rz, "ncols", z.ncols)
        object.__setattr__(rz, "values", z.values)
        object.__setattr__(rz, "colptr", np.asarray(z.colptr, dtype=np.int64))
        object.__setattr__(rz, "rowidx", np.tile(np.arange(z.nrows, dtype=np.int64), z.ncols))
        rz.__dict__["scipy"] = DenseZ(z.dense_samples())
    else:
        rz = RefCSC(nrows=z.nrows, ncols=z.ncols, colptr=z.colptr, rowidx=z.rowidx, values=z.values)
    rp = gdwd.ProblemData(z_tilde=rz, y=prob.y, e=prob.e, weights=prob.weights, C=prob.C, q=prob.q,
                          z_scale=prob.z_scale)
    conf = gdwd.SolverConfig(q=prob.q, max_iter=ARGS.max_iter)
    rng = np.random.default_rng(1234)
    idx_n = np.sort(rng.choice(prob.n, min(NSAMPLE, prob.n), replace=False))
    rows, keep = [], {}
    tlast = [time.perf_counter()]

    def cb(st, res):
        rows.append([res.eta_c1, res.eta_c2, res.eta_c3, res.eta_p1, res.eta_p2, res.eta_p3, res.eta_d1,
                     res.eta_d2, res.eta_gap, res.obj_primal, res.obj_dual, st.sigma, st.beta, st.iter,
                     float(np.linalg.norm(st.w)), float(np.linalg.norm(st.alpha))])
        if st.iter in (1, 20):
            keep[f"w{st.iter}"] = np.array(st.w, copy=True)
        if st.iter == 20:
            for k in ("alpha", "r", "xi"):
                keep[f"s20_{k}"] = np.array(getattr(st, k))[idx_n].copy()
        if st.iter % 50 == 0:
            now = time.perf_counter()
            print(f"{name}: iter {st.iter} sigma={st.sigma:.3e} eta_p={res.eta_p:.2e} eta_d={res.eta_d:.2e} "
                  f"({(now - tlast[0]) / 50:.2f}s/it)", flush=True)
            tlast[0] = now

    t1 = time.perf_counter()
    res = gdwd.sgs_admm_solve(rp, conf, callback=cb)
    dt = time.perf_counter() - t1
    fs = res.final_state
    np.savez_compressed(
        OUT / f"full_{name}.npz", hist=np.array(rows), idx_n=idx_n, final_w=fs.w, final_beta=fs.beta,
        obj_primal=res.final_residuals.obj_primal, obj_dual=res.final_residuals.obj_dual,
        iterations=res.iterations, converged=int(res.converged), double_count=res.double_count,
        psqmr_total=res.psqmr_total, train_error=res.train_error_pct, backend=res.backend_used.value,
        z_sha=z_checksum(z.values), solve_time=dt, operator=operator, cfg=cfgname, d=prob.d, n=prob.n,
        max_iter=ARGS.max_iter, **keep)
    print(f"{name}: backend={res.backend_used.value} iters={res.iterations} conv={res.converged} "
          f"doubles={res.double_count} psqmr={res.psqmr_total} err={res.train_error_pct:.3f}% {dt:.1f}s",
          flush=True)


if __name__ == "__main__":
    main()
