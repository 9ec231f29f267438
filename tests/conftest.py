import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (str(ROOT),):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libgdwd_b200.so")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def load_traj(name):
    return dict(np.load(GOLDEN / f"traj_{name}.npz", allow_pickle=False))


def load_kat():
    return json.loads((GOLDEN / "kat.json").read_text())


TRAJ_CASES = ["tiny_direct", "tiny_smw2", "tiny_iter", "tiny_iter_c4gen", "tiny_direct_q2", "smw2_natural",
              "iter_natural", "direct_q4", "tiny_sparse", "sparse_natural", "sparse_direct", "prox_tiny",
              "prox_tiny_q2"]
# option / edge-case variants (make_golden.py VARIANTS): backend requested explicitly
VAR_CASES = ["var_nosgs", "var_q_half", "var_q3_mu2", "var_opts", "var_e_random", "var_odd", "var_sparse_holes",
             "var_min_direct", "var_min_smw", "var_min_iter", "var_d1_smw", "var_direct_gram",
             "var_direct_gram_nosgs", "var_direct_gram_converge", "var_converge", "var_converge_smw", "var_converge_iter"]
SOLVER_KEYS = ("use_sgs", "mu", "sigma0", "epsilon_c", "steplength", "tol_feas", "tol_cgap", "tol_cap")


def variant_of(tr) -> dict:
    return json.loads(str(tr["variant"])) if "variant" in tr else {}


def solver_options(tr) -> dict:
    """SolverConfig keyword overrides the fixture was generated with."""
    var = variant_of(tr)
    return {k: var[k] for k in SOLVER_KEYS if k in var}


def problem_for(tr):
    from paper_2305_12019_b200 import synth

    var = variant_of(tr)
    if var:
        return synth.make_variant_problem(str(tr["cfg"]), int(tr["d"]), int(tr["n"]), int(tr["seed"]), **var)
    cfg = synth.CONFIGS[str(tr["cfg"])].scaled(d=int(tr["d"]), n=int(tr["n"]))
    return synth.make_problem(cfg, int(tr["seed"]))


def relerr(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    den = max(np.linalg.norm(b), 1e-300)
    return float(np.linalg.norm(a - b) / den)
