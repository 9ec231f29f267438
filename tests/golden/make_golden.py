"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is importable from
/root/reference/pkg/src; it does not exist on the GPU box):

    python tests/golden/make_golden.py            # everything
    python tests/golden/make_golden.py --quick    # skip the 2000-iteration c1 run

Outputs (committed, small):
  kat.json           SPEC.md known-answer tests evaluated by the reference
  traj_<case>.npz    per-iteration trajectories of sgs_admm_solve on seeded
                     problems (all three backends; full vectors for tiny
                     cases, scalars + sampled coordinates for larger ones)
  c1_full.npz        BASELINE config 1 (d=2000, n=1000), 2000 iterations:
                     scalar history (incl. the sigma trace), first 20 iterates
                     of w and alpha, final state

Inputs are regenerated from paper_2305_12019_b200.synth (pure function of the
seed); each fixture stores a checksum of Z~ so a generator change is caught.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import gdwd  # noqa: E402  (the reference)
from gdwd.linalg import SparseMatrixCSC as RefCSC  # noqa: E402
from gdwd.linalg import cholesky_factorize, cholesky_solve, lanczos_topk, psqmr  # noqa: E402

from paper_2305_12019_b200 import synth  # noqa: E402
from make_golden_inputs import LIBSVM_CASES, big_libsvm, penalty_inputs  # noqa: E402

OUT = Path(__file__).resolve().parent

# (name, synth config, d, n, backend, max_iter, full vectors?)
CASES = [
    ("tiny_direct", "c1", 60, 40, "direct", 80, True),
    ("tiny_smw2", "c2", 90, 16, "smw2", 80, True),
    ("tiny_iter", "c1", 70, 50, "iterative", 80, True),
    ("tiny_iter_c4gen", "c2", 64, 40, "iterative", 60, True),
    ("tiny_direct_q2", "c3", 40, 120, "direct", 80, True),
    ("smw2_natural", "c2", 6000, 200, "auto", 40, False),
    ("iter_natural", "c1", 6000, 1500, "auto", 25, False),
    ("direct_q4", "c5", 300, 900, "auto", 60, False),
    ("tiny_sparse", "c4", 3000, 2000, "iterative", 40, True),
    ("sparse_natural", "c4", 8000, 30000, "auto", 25, False),
    ("sparse_direct", "c4", 1500, 4000, "auto", 40, False),
    # proximal fallback (subsolvers.py:159-256): PSQMR budget 2 steps forces the switch
    ("prox_tiny", "c1", 70, 50, "iterative", 40, True, 0, 2),
    ("prox_tiny_q2", "c3", 90, 300, "iterative", 40, True, 0, 2),
    ("prox_lanczos_fail", "c1", 6000, 1500, "auto", 12, False, 0, 3),
]
# option / edge-case variants: (name, cfg, d, n, backend, max_iter, full, variations)
VARIANTS = [
    ("var_nosgs", "c1", 61, 45, "direct", 40, True, dict(use_sgs=False)),
    ("var_q_half", "c1", 50, 41, "direct", 40, True, dict(q=0.5)),
    ("var_q3_mu2", "c1", 48, 60, "iterative", 40, True, dict(q=3.0, mu=2.0)),
    ("var_opts", "c2", 80, 15, "smw2", 40, True, dict(sigma0=3.0, epsilon_c=0.05, steplength=1.2, mu=0.7)),
    ("var_e_random", "c1", 40, 55, "direct", 40, True, dict(e_random=True, C=3.0)),
    ("var_odd", "c3", 37, 53, "direct", 40, True, dict()),
    ("var_sparse_holes", "c4", 700, 400, "iterative", 30, True, dict(holes=True)),
    ("var_min_direct", "c1", 1, 2, "direct", 30, True, dict()),
    ("var_min_smw", "c1", 3, 2, "smw2", 30, True, dict()),
    ("var_min_iter", "c1", 2, 3, "iterative", 30, True, dict()),
    ("var_d1_smw", "c1", 1, 5, "smw2", 30, True, dict()),
    # DIRECT with 2n <= d: solved in sample space on the device (same exact solve)
    ("var_direct_gram", "c1", 200, 60, "direct", 40, True, dict()),
    ("var_direct_gram_nosgs", "c1", 160, 50, "direct", 30, True, dict(use_sgs=False)),
    ("var_direct_gram_converge", "c2", 120, 20, "direct", 600, True,
     dict(C=10.0, shift=2.0, tol_feas=1e-3, tol_cgap=0.03, tol_cap=0.3)),
    ("var_converge", "c1", 30, 60, "direct", 600, True,
     dict(C=10.0, shift=2.0, tol_feas=1e-3, tol_cgap=0.03, tol_cap=0.3)),
    ("var_converge_smw", "c2", 120, 20, "smw2", 600, True,
     dict(C=10.0, shift=2.0, tol_feas=1e-3, tol_cgap=0.03, tol_cap=0.3)),
    ("var_converge_iter", "c1", 30, 60, "iterative", 600, True,
     dict(C=10.0, shift=2.0, tol_feas=1e-3, tol_cgap=0.03, tol_cap=0.3)),
]
SAMPLE = 64  # sampled coordinates per vector for the non-full cases


def z_checksum(values: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(values).tobytes()).hexdigest()[:16]


def to_ref(prob):
    z = prob.z_tilde
    rz = RefCSC(nrows=z.nrows, ncols=z.ncols, colptr=z.colptr, rowidx=z.rowidx, values=z.values)
    return gdwd.ProblemData(z_tilde=rz, y=prob.y, e=prob.e, weights=prob.weights, C=prob.C, q=prob.q,
                            z_scale=prob.z_scale)


variant_problem = synth.make_variant_problem


SOLVER_KEYS = ("use_sgs", "mu", "sigma0", "epsilon_c", "steplength", "tol_feas", "tol_cgap", "tol_cap")


def run_case(name, cfgname, d, n, backend, max_iter, full, seed=0, switch=50, **var):
    prob = variant_problem(cfgname, d, n, seed, **var)
    rp = to_ref(prob)
    conf = gdwd.SolverConfig(q=prob.q, max_iter=max_iter, backend=gdwd.Backend(backend),
                             psqmr_switch_steps=switch, **{k: var[k] for k in SOLVER_KEYS if k in var})
    rows, vecs = [], {k: [] for k in ("w", "u", "rho", "r", "xi", "alpha")}
    rng = np.random.default_rng(1234)
    idx_d = np.sort(rng.choice(d, min(SAMPLE, d), replace=False))
    idx_n = np.sort(rng.choice(n, min(SAMPLE, n), replace=False))

    def cb(st, res):
        rows.append([res.eta_c1, res.eta_c2, res.eta_c3, res.eta_p1, res.eta_p2, res.eta_p3, res.eta_d1,
                     res.eta_d2, res.eta_gap, res.obj_primal, res.obj_dual, st.sigma, st.beta, st.iter,
                     float(np.linalg.norm(st.w)), float(np.linalg.norm(st.alpha))])
        for k in vecs:
            v = np.array(getattr(st, k), copy=True)
            if not full:
                v = v[idx_d] if k in ("w", "u", "rho") else v[idx_n]
            vecs[k].append(v)

    t0 = time.perf_counter()
    try:
        res = gdwd.sgs_admm_solve(rp, conf, callback=cb)
    except Exception as exc:  # the reference's own error behaviour is part of the fixture
        np.savez_compressed(OUT / f"traj_{name}.npz", hist=np.array(rows), idx_d=idx_d, idx_n=idx_n,
                            error=type(exc).__name__, iterations_before_error=len(rows), variant=json.dumps(var),
                            z_sha=z_checksum(prob.z_tilde.values), d=d, n=n, seed=seed, cfg=cfgname,
                            max_iter=max_iter, full=int(full), switch=switch,
                            **{"it_" + k: np.array(v) for k, v in vecs.items()})
        print(f"{name}: reference raised {type(exc).__name__} after {len(rows)} iterations", flush=True)
        return
    dt = time.perf_counter() - t0
    out = dict(hist=np.array(rows), idx_d=idx_d, idx_n=idx_n, iterations=res.iterations,
               converged=int(res.converged), double_count=res.double_count, psqmr_total=res.psqmr_total,
               backend=res.backend_used.value, final_w=res.final_state.w, final_beta=res.final_state.beta,
               z_sha=z_checksum(prob.z_tilde.values), d=d, n=n, seed=seed, cfg=cfgname, max_iter=max_iter,
               full=int(full), train_error=res.train_error_pct, switch=switch,
               variant=json.dumps(var))
    for k, v in vecs.items():
        out["it_" + k] = np.array(v)
    np.savez_compressed(OUT / f"traj_{name}.npz", **out)
    print(f"{name}: backend={res.backend_used.value} iters={res.iterations} doubles={res.double_count} "
          f"psqmr={res.psqmr_total} conv={res.converged} {dt:.1f}s", flush=True)


def run_c1_full():
    prob = synth.make_problem(synth.CONFIGS["c1"], 0)
    rp = to_ref(prob)
    conf = gdwd.SolverConfig(q=1.0, max_iter=2000)
    rows, w20, a20 = [], [], []

    def cb(st, res):
        rows.append([res.eta_c1, res.eta_c2, res.eta_c3, res.eta_p1, res.eta_p2, res.eta_p3, res.eta_d1,
                     res.eta_d2, res.eta_gap, res.obj_primal, res.obj_dual, st.sigma, st.beta, st.iter,
                     float(np.linalg.norm(st.w)), float(np.linalg.norm(st.alpha))])
        if st.iter <= 20:
            w20.append(np.array(st.w, copy=True))
            a20.append(np.array(st.alpha, copy=True))

    t0 = time.perf_counter()
    res = gdwd.sgs_admm_solve(rp, conf, callback=cb)
    dt = time.perf_counter() - t0
    fs = res.final_state
    np.savez_compressed(OUT / "c1_full.npz", hist=np.array(rows), w20=np.array(w20), alpha20=np.array(a20),
                        final_w=fs.w, final_beta=fs.beta, final_r=fs.r, final_xi=fs.xi, final_alpha=fs.alpha,
                        iterations=res.iterations, converged=int(res.converged), double_count=res.double_count,
                        z_sha=z_checksum(prob.z_tilde.values), solve_time=dt,
                        obj_primal=res.final_residuals.obj_primal)
    print(f"c1_full: iters={res.iterations} conv={res.converged} doubles={res.double_count} {dt:.1f}s", flush=True)


def kats():
    """SPEC.md KATs evaluated by the reference."""
    k = {}
    k["newton_r"] = [[a, s, q, w, r0] + list(gdwd.newton_r(a, s, q, w, r0))
                     for (a, s, q, w, r0) in [(0.0, 1.0, 1.0, 1.0, 1.0), (0.0, 2.0, 1.0, 1.0, 1.0),
                                              (10.0, 1.0, 1.0, 1.0, 1.0), (-3.0, 5.0, 2.0, 0.5, 1.0),
                                              (2.0, 100.0, 4.0, 0.3, 0.5), (0.5, 1e6, 1.0, 1.0, 1.0)]]
    k["select_solver"] = [[n, d, gdwd.select_solver(n, d).value] for (n, d) in
                          [(100, 100), (1000, 10000), (30000, 300000), (1000, 5000), (1000, 5001), (1000, 5000 + 1),
                           (2500, 12501), (2501, 20000), (1000, 5005), (1001, 5005), (1, 1)]]
    k["update_sigma"] = [[s, p, dd, gdwd.update_sigma(s, p, dd)] for (s, p, dd) in
                         [(1.0, 10.0, 1.0), (1.0, 1.0, 1.0), (1.0, 600.0, 1.0), (1.0, 1.0, 10.0), (2.0, 0.0, 0.0),
                          (3.0, 1e-9, 0.0), (3.0, 0.0, 1e-9), (1.0, 60.0, 1.0), (1.0, 1.0, 60.0)]]
    y = np.array([1.0] * 90 + [-1.0] * 10)
    k["compute_weights"] = {"q1": gdwd.compute_weights(y, 1.0).tolist()[:1] + gdwd.compute_weights(y, 1.0).tolist()[-1:],
                            "q2": gdwd.compute_weights(y, 2.0).tolist()[:1] + gdwd.compute_weights(y, 2.0).tolist()[-1:]}
    f = cholesky_factorize(np.array([[4.0, 2.0], [2.0, 3.0]]))
    k["cholesky"] = {"R": f.r_factor.tolist(), "solve": cholesky_solve(f, np.array([6.0, 5.0])).tolist()}
    pr = psqmr(lambda v: np.array([1.0, 2.0, 3.0]) * v, np.array([1.0, 2.0, 3.0]), tol=1e-12)
    k["psqmr_diag"] = {"x": pr.x.tolist(), "iterations": pr.iterations, "converged": pr.converged}
    rng = np.random.default_rng(7)
    B = rng.standard_normal((50, 50))
    S = B @ B.T + 50 * np.eye(50)
    b = rng.standard_normal(50)
    M = np.diag(S).copy()
    pr2 = psqmr(lambda v: S @ v, b, precond=lambda v: v / M, tol=1e-10, max_iter=200)
    k["psqmr_spd50"] = {"seed": 7, "x": pr2.x.tolist(), "iterations": pr2.iterations,
                        "converged": pr2.converged, "residual_norm": pr2.residual_norm}
    pe = lanczos_topk(lambda v: np.array([5.0, 4.0, 3.0, 2.0, 1.0]) * v, 5, 2)
    k["lanczos_diag"] = {"eigenvalues": pe.eigenvalues.tolist()}
    (OUT / "kat.json").write_text(json.dumps(k, indent=1))
    print("kat.json written")


def make_scoring():
    """Reference decision_values / predict / train_error (solver.py:610-642)
    on raw dense and sparse matrices, with models trained by the reference;
    test matrices wider and narrower than the training dimension."""
    out = {}
    for tag, cfgname, d, n in (("dense", "c1", 60, 40), ("sparse", "c4", 3000, 500)):
        cfg = synth.CONFIGS[cfgname].scaled(d=d, n=n)
        x, y = synth.raw_data(cfg, 5)
        rx = RefCSC(nrows=x.nrows, ncols=x.ncols, colptr=x.colptr, rowidx=x.rowidx, values=x.values)
        tau = gdwd.compute_weights(y, cfg.q)
        prob = gdwd.scale_problem(rx, y, None, cfg.C, cfg.q, tau=tau)
        res = gdwd.sgs_admm_solve(prob, gdwd.SolverConfig(q=cfg.q, max_iter=60))
        model = res.model
        out[f"{tag}_w"] = model.w
        out[f"{tag}_beta"] = model.beta
        out[f"{tag}_y"] = y
        out[f"{tag}_scores"] = gdwd.solver.decision_values(model, rx)
        out[f"{tag}_pred"] = gdwd.predict(model, rx)
        out[f"{tag}_err"] = gdwd.train_error(model, rx, y)
        for extra, dd in (("wide", d + 7), ("narrow", d - 5)):
            cfg2 = synth.CONFIGS[cfgname].scaled(d=dd, n=n // 2)
            x2, y2 = synth.raw_data(cfg2, 6)
            rx2 = RefCSC(nrows=x2.nrows, ncols=x2.ncols, colptr=x2.colptr, rowidx=x2.rowidx, values=x2.values)
            out[f"{tag}_{extra}_scores"] = gdwd.solver.decision_values(model, rx2)
            out[f"{tag}_{extra}_err"] = gdwd.train_error(model, rx2, y2)
            out[f"{tag}_{extra}_d"] = dd
        out[f"{tag}_n"] = n
        out[f"{tag}_d"] = d
    np.savez_compressed(OUT / "scoring.npz", **out)
    print("scoring.npz:", {k: float(v) for k, v in out.items() if k.endswith("_err")})


def make_penalty():
    """Reference compute_penalty_C (solver.py:193-232) values."""
    out = {}
    for name, (x, y, q, seed) in penalty_inputs().items():
        rx = RefCSC(nrows=x.nrows, ncols=x.ncols, colptr=x.colptr, rowidx=x.rowidx, values=x.values)
        c, dist = gdwd.compute_penalty_C(rx, y, q, seed=seed)
        out[name] = {"C": c, "dist": dist, "q": q, "seed": seed}
    (OUT / "penalty.json").write_text(json.dumps(out, indent=1))
    print("penalty.json:", out)


def make_ingest():
    """Reference parse_libsvm / preprocess (ingest.py:102-211) outputs and
    error messages on the LIBSVM_CASES texts and a large seeded text."""
    import io

    out = {}
    for name, text, req in LIBSVM_CASES + [("big", big_libsvm(), True)]:
        rec = {"require_labels": req}
        try:
            raw = gdwd.parse_libsvm(io.StringIO(text, newline=None), require_labels=req)
        except gdwd.ParseError as exc:
            rec["error"] = str(exc)
            rec["line_no"] = exc.line_no
            out[name] = rec
            continue
        x = raw.X
        arrays = {"colptr": x.colptr, "rowidx": x.rowidx, "values": x.values}
        rec.update({"n": x.ncols, "d": x.nrows, "nnz": int(x.values.size),
                    "labels": None if raw.labels is None else raw.labels.tolist()})
        try:
            xc, _, meta = gdwd.preprocess(raw)
            arrays.update({"pcolptr": xc.colptr, "prowidx": xc.rowidx, "pvalues": xc.values,
                           "kept": meta.kept_ids, "scales": meta.scales})
        except ValueError as exc:
            rec["preprocess_error"] = str(exc)
        if name == "big":
            rec["sha"] = {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for k, v in arrays.items()}
            rec["labels"] = hashlib.sha256(np.asarray(raw.labels).tobytes()).hexdigest()
        else:
            rec.update({k: v.tolist() for k, v in arrays.items()})
        out[name] = rec
    (OUT / "ingest.json").write_text(json.dumps(out, indent=1))
    print("ingest.json:", {k: v.get("error", v.get("n")) for k, v in out.items()})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    if a.only in (None, "kat"):
        kats()
    for c in CASES:
        if a.only in (None, c[0]):
            run_case(*c)
    for name, cfgname, d, n, backend, mi, full, var in VARIANTS:
        if a.only in (None, name, "variants"):
            run_case(name, cfgname, d, n, backend, mi, full, **var)
    if a.only in (None, "scoring"):
        make_scoring()
    if a.only in (None, "penalty"):
        make_penalty()
    if a.only in (None, "ingest"):
        make_ingest()
    if not a.quick and a.only in (None, "c1"):
        run_c1_full()


if __name__ == "__main__":
    main()
