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


def problem_for(tr):
    from paper_2305_12019_b200 import synth

    cfg = synth.CONFIGS[str(tr["cfg"])].scaled(d=int(tr["d"]), n=int(tr["n"]))
    return synth.make_problem(cfg, int(tr["seed"]))


def relerr(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    den = max(np.linalg.norm(b), 1e-300)
    return float(np.linalg.norm(a - b) / den)
