"""CPU tests: host-side mirror of the reference API, the synthetic generators
and the C ABI surface (no compute calls without a GPU)."""

import ctypes
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2305_12019_b200 as G
from conftest import ROOT, load_kat
from paper_2305_12019_b200 import _lib, synth


def test_select_solver_matches_kat():
    for n, d, kind in load_kat()["select_solver"]:
        assert G.select_solver(n, d).value == kind
    with pytest.raises(ValueError):
        G.select_solver(0, 5)


def test_update_sigma_matches_kat():
    for s, p, d, out in load_kat()["update_sigma"]:
        assert G.update_sigma(s, p, d) == out


def test_compute_weights():
    y = np.array([1.0] * 90 + [-1.0] * 10)
    k = load_kat()["compute_weights"]
    w = G.compute_weights(y, 1.0)
    assert [w[0], w[-1]] == k["q1"]
    assert w[0] == pytest.approx(1.0 / 3.0)
    with pytest.raises(G.SingleClassError):
        G.compute_weights(np.ones(5), 1.0)


def test_solver_config_validation():
    G.SolverConfig()
    with pytest.raises(ValueError):
        G.SolverConfig(steplength=1.7)
    with pytest.raises(ValueError):
        G.SolverConfig(tol_feas=0.0)
    with pytest.raises(ValueError):
        G.SolverConfig(mu=-1.0)


def test_problem_data_validation():
    x = G.csc_from_dense(np.arange(1.0, 7.0).reshape(2, 3))
    y = np.array([1.0, -1.0, 1.0])
    p = G.scale_problem(x, y, None, 1.0, 1.0)
    assert p.n == 3 and p.d == 2
    assert p.z_scale == pytest.approx(math.sqrt(math.sqrt(91.0)))
    with pytest.raises(ValueError):
        G.ProblemData(p.z_tilde, np.array([1.0, 2.0, 1.0]), p.e, p.weights, 1.0, 1.0, 1.0)
    with pytest.raises(ValueError):
        G.ProblemData(p.z_tilde, y, p.e * 2, p.weights, 1.0, 1.0, 1.0)
    with pytest.raises(ValueError):
        G.ProblemData(p.z_tilde, y, p.e, p.weights, -1.0, 1.0, 1.0)


def test_dense_csc_layout_is_sample_major():
    a = np.random.default_rng(0).standard_normal((5, 3)) + 10.0  # d=5, n=3, no zeros
    z = G.csc_from_dense(a)
    assert z.is_dense and z.nnz == 15
    assert np.array_equal(z.dense_samples(), a.T)
    assert np.array_equal(z.toarray(), a)
    assert np.array_equal(z.scipy.toarray(), a)
    assert np.allclose(z.row_sq_sums(), (a * a).sum(axis=1))


def test_scale_problem_matches_reference_formula():
    x, y = synth.raw_data(synth.CONFIGS["c1"].scaled(d=30, n=20))
    p = G.scale_problem(x, y, None, 1.0, 1.0)
    ref = x.values * np.repeat(y, np.diff(x.colptr)) / math.sqrt(x.frobenius_norm())
    assert np.array_equal(p.z_tilde.values, ref)


def test_synth_generators_shapes_and_labels():
    for name in ("c1", "c2", "c3", "c5"):
        cfg = synth.CONFIGS[name].scaled(d=50, n=64)
        x, y = synth.raw_data(cfg)
        assert x.is_dense and x.nrows == 50 and x.ncols == 64
        assert set(np.unique(y)) <= {-1.0, 1.0}
        assert np.sum(y != synth.true_labels(64)) == round(cfg.flip * 64)
    cfg = synth.CONFIGS["c4"].scaled(d=2000, n=3000)
    x, y = synth.raw_data(cfg)
    assert not x.is_dense
    colnorm = np.sqrt(np.add.reduceat(x.values ** 2, x.colptr[:-1]))
    assert np.allclose(colnorm[np.diff(x.colptr) > 0], 1.0)
    assert abs(x.nnz / (2000 * 3000) - 0.001) < 2e-4
    # shard regeneration: block-aligned slices reproduce the full matrix
    cfg = synth.CONFIGS["c2"].scaled(d=40, n=3 * synth.BLOCK)
    full = synth.dense_samples(cfg, 5)
    part = synth.dense_samples(cfg, 5, lo=synth.BLOCK, hi=2 * synth.BLOCK)
    assert np.array_equal(full[synth.BLOCK:2 * synth.BLOCK], part)


def _header_symbols():
    txt = (ROOT / "include" / "gdwd_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(gdwd_\w+)\(", txt, re.M)))


def test_header_declares_binding_symbols():
    assert _header_symbols() == sorted(_lib.SYMBOLS)


def test_library_loads_and_exports_every_symbol():
    lib = _lib.load()
    for s in _header_symbols():
        assert hasattr(lib, s), s
    assert lib.gdwd_version() == 1
    # struct layouts agree with the compiled header (sizes, no compute)
    cb, rb = ctypes.c_int64(), ctypes.c_int64()
    lib.gdwd_abi_sizes(ctypes.byref(cb), ctypes.byref(rb))
    assert ctypes.sizeof(_lib.GdwdConfig) == cb.value == 11 * 4 + 4 + 7 * 8
    assert ctypes.sizeof(_lib.GdwdResult) == rb.value == 6 * 4 + 5 * 8 + 11 * 8


def test_no_cpu_fallback_in_product_package():
    pkg = ROOT / "paper_2305_12019_b200"
    for f in pkg.glob("*.py"):
        src = f.read_text()
        assert "oracle" not in src.replace("oracle/", ""), f"{f.name} references the oracle"


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(_lib.GdwdLibraryError):
        _lib._lib_saved = _lib._lib
        _lib._lib = None
        try:
            _lib.load(tmp_path / "nope.so")
        finally:
            _lib._lib = _lib._lib_saved
