"""Device-generated problems (config 5 is 160 GB: generated in HBM).
A column-subsampled config-5 proxy is generated on the device, downloaded,
and the device solve is checked against the oracle on the same Z~."""

import numpy as np
import pytest

import paper_2305_12019_b200 as G
from oracle import gdwd_oracle as O
from paper_2305_12019_b200 import synth

pytestmark = pytest.mark.gpu


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def test_generator_statistics_and_sharding():
    cfg = synth.CONFIGS["c5"].scaled(d=3000, n=4000)
    full = synth.make_device_problem(cfg, seed=3)
    Z = full.download_samples()  # rows: y_i x_i / z_scale
    X = Z * (full.z_scale / full.y[:, None])
    ytrue = synth.true_labels(cfg.n)
    noise = X - ytrue[:, None] * np.where(np.arange(cfg.d) < cfg.signal_k, cfg.shift, 0.0)[None, :]
    assert abs(noise.mean()) < 3e-3 and abs(noise.std() - 1.0) < 3e-3
    assert abs(np.sqrt(np.sqrt(np.sum(X * X))) - full.z_scale) < 1e-9 * full.z_scale
    # shards regenerate their columns exactly
    parts = [synth.make_device_problem(cfg, seed=3, rank=r, nranks=3) for r in range(3)]
    Xp = np.concatenate([p.download_samples() * (p.z_scale / p.y[:, None]) for p in parts])
    assert np.allclose(Xp, X, rtol=1e-14, atol=1e-14)


# (6000, 30000): d > 5000 and d <= n/4 -- ITERATIVE with the Gram operator and
# q = 4, the path config 5 itself takes (iter_gram automatic)
@pytest.mark.parametrize("d,n", [(2000, 9000), (6000, 12000), (6000, 30000)])
def test_c5_proxy_first20(d, n):
    cfg = synth.CONFIGS["c5"].scaled(d=d, n=n)
    dev = synth.make_device_problem(cfg, seed=0)
    S = dev.download_samples()
    host = G.ProblemData(G.SparseMatrixCSC.from_dense_samples(S), dev.y, dev.e, dev.weights, dev.C, dev.q, dev.z_scale)
    ref = []
    O.solve(host, O.OracleConfig(max_iter=20), operator="dense", record=False,
            callback=lambda st, res: ref.append((st["w"].copy(), st["alpha"].copy(), st["r"].copy())))
    got = []
    out = G.sgs_admm_solve(dev, G.SolverConfig(q=dev.q, max_iter=20),
                           callback=lambda st, res: got.append((st.w.copy(), st.alpha.copy(), st.r.copy())))
    assert out.backend_used.value == O.select_backend(n, d)
    for i in range(20):
        for a, b in zip(got[i], ref[i]):
            assert relerr(a, b) < 1e-9, i
