"""Gram builds of configs 2 and 3 on the FP64 tensor cores (DMMA), timed
end to end through gdwd_gram (includes the H2D copy) -- for ncu captures."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2305_12019_b200 import linalg as L

rng = np.random.default_rng(0)
for name, rows, cols, over_rows in (("c3 ZZ^T", 200000, 1000, True), ("c2 Z^TZ", 2000, 20000, False)):
    X = rng.standard_normal((rows, cols))
    for rep in range(2):
        t = time.perf_counter()
        G = L.gram(X, over_rows)
        dt = time.perf_counter() - t
    M = cols if over_rows else rows
    K = rows if over_rows else cols
    print(f"{name}: M={M} K={K} {2*M*M*K/1e9:.0f} GFLOP (full), wall incl. upload {dt*1e3:.1f} ms", flush=True)
