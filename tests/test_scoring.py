"""Model application (decision_values / predict / train_error,
solver.py:610-642): the oracle pinned against the reference's own outputs
(tests/golden/scoring.npz), then the device scoring pass against both."""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import gdwd_oracle as O
from paper_2305_12019_b200 import synth


def _fixture():
    return dict(np.load(GOLDEN / "scoring.npz"))


def _inputs(fx, tag):
    cfgname = {"dense": "c1", "sparse": "c4"}[tag]
    d, n = int(fx[f"{tag}_d"]), int(fx[f"{tag}_n"])
    x, _ = synth.raw_data(synth.CONFIGS[cfgname].scaled(d=d, n=n), 5)
    out = {"train": x}
    for extra in ("wide", "narrow"):
        dd = int(fx[f"{tag}_{extra}_d"])
        out[extra] = synth.raw_data(synth.CONFIGS[cfgname].scaled(d=dd, n=n // 2), 6)
    return out


@pytest.mark.parametrize("tag", ["dense", "sparse"])
def test_oracle_scoring_matches_reference(tag):
    fx = _fixture()
    inp = _inputs(fx, tag)
    w, b = fx[f"{tag}_w"], float(fx[f"{tag}_beta"])
    x = inp["train"].scipy
    assert np.array_equal(O.decision_values(w, b, x), fx[f"{tag}_scores"])
    assert np.array_equal(O.predict(w, b, x), fx[f"{tag}_pred"])
    assert O.train_error(w, b, x, fx[f"{tag}_y"]) == float(fx[f"{tag}_err"])
    for extra in ("wide", "narrow"):
        x2, y2 = inp[extra]
        assert np.array_equal(O.decision_values(w, b, x2.scipy), fx[f"{tag}_{extra}_scores"])
        assert O.train_error(w, b, x2.scipy, y2) == float(fx[f"{tag}_{extra}_err"])


def _model(w, beta):
    from paper_2305_12019_b200 import ModelFile, identity_meta

    return ModelFile(q=1.0, C=1.0, z_scale=1.0, mu=1.0, feature_meta=identity_meta(w.size), w=w, beta=beta)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["dense", "sparse"])
def test_device_scoring_matches_reference(tag):
    from paper_2305_12019_b200 import scoring

    fx = _fixture()
    inp = _inputs(fx, tag)
    w, b = fx[f"{tag}_w"], float(fx[f"{tag}_beta"])
    model = _model(w, b)
    x = inp["train"]
    s = scoring.decision_values(model, x)
    ref = fx[f"{tag}_scores"]
    # the device sums each sample's products in a different (tree) order
    assert np.allclose(s, ref, rtol=1e-12, atol=1e-13 * np.abs(ref).max())
    assert np.array_equal(scoring.predict(model, x), fx[f"{tag}_pred"])
    assert scoring.train_error(model, x, fx[f"{tag}_y"]) == float(fx[f"{tag}_err"])
    for extra in ("wide", "narrow"):
        x2, y2 = inp[extra]
        r2 = fx[f"{tag}_{extra}_scores"]
        assert np.allclose(scoring.decision_values(model, x2), r2, rtol=1e-12, atol=1e-13 * np.abs(r2).max())
        assert scoring.train_error(model, x2, y2) == float(fx[f"{tag}_{extra}_err"])


@pytest.mark.gpu
def test_zero_scores_follow_reference_conventions():
    """w = 0, beta = 0: every score is 0 -> every sample wrong
    (solver.py:639-642), and predict gives -1: the reference's code is
    ``np.where(scores > 0, 1, -1)`` (its docstring's "zero maps to +1" is not
    what it does; the code is the behaviour mirrored)."""
    from paper_2305_12019_b200 import scoring

    x, y = synth.raw_data(synth.CONFIGS["c1"].scaled(d=30, n=25), 1)
    model = _model(np.zeros(30), 0.0)
    assert np.array_equal(scoring.decision_values(model, x), np.zeros(25))
    assert np.array_equal(scoring.predict(model, x), -np.ones(25))
    assert np.array_equal(O.predict(np.zeros(30), 0.0, x.scipy), -np.ones(25))
    assert scoring.train_error(model, x, y) == 100.0
    assert O.train_error(np.zeros(30), 0.0, x.scipy, y) == 100.0


@pytest.mark.gpu
def test_scoring_rejects_bad_labels():
    from paper_2305_12019_b200 import scoring

    x, _ = synth.raw_data(synth.CONFIGS["c1"].scaled(d=10, n=8), 1)
    dm = scoring.device_matrix(x)
    with pytest.raises(ValueError):
        dm.score(np.zeros(11), 0.0)
    with pytest.raises(ValueError):
        dm.score(np.zeros(10), 0.0, y=np.ones(7))
