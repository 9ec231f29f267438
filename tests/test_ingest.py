"""LIBSVM ingest / preprocess / model files (reference ingest.py) against the
reference's own outputs and messages (tests/golden/ingest.json).  The parser
and preprocess are native host code in the library: these run on CPU."""

import hashlib
import io
import json
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_golden_inputs import LIBSVM_CASES, big_libsvm  # noqa: E402

import paper_2305_12019_b200 as G  # noqa: E402

REF = json.loads((GOLDEN / "ingest.json").read_text())


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("from_file", [False, True])
@pytest.mark.parametrize("name,text,req", LIBSVM_CASES, ids=[c[0] for c in LIBSVM_CASES])
def test_parse_and_preprocess_match_reference(name, text, req, from_file, tmp_path):
    """Streams (Python's universal-newline text) and files (raw bytes with
    \r\n and lone \r, read natively) parse alike."""
    ref = REF[name]
    if from_file:
        src = tmp_path / "in.svm"
        src.write_bytes(text.encode())
    else:
        src = io.StringIO(text, newline=None)
    if "error" in ref:
        with pytest.raises(G.ParseError) as ei:
            G.parse_libsvm(src, require_labels=req)
        assert str(ei.value) == ref["error"] and ei.value.line_no == ref["line_no"]
        return
    raw = G.parse_libsvm(src, require_labels=req)
    x = raw.X
    assert (x.ncols, x.nrows) == (ref["n"], ref["d"])
    assert x.colptr.tolist() == ref["colptr"] and x.rowidx.tolist() == ref["rowidx"]
    assert x.values.tolist() == ref["values"]
    assert (raw.labels is None and ref["labels"] is None) or raw.labels.tolist() == ref["labels"]
    xc, _, meta = G.preprocess(raw)
    assert xc.colptr.tolist() == ref["pcolptr"] and xc.rowidx.tolist() == ref["prowidx"]
    assert xc.values.tolist() == ref["pvalues"]
    assert meta.kept_ids.tolist() == ref["kept"] and meta.scales.tolist() == ref["scales"]


@pytest.mark.parametrize("threads", ["1", "0"])
def test_large_text_multithreaded_matches_reference(threads, monkeypatch, tmp_path):
    """40k lines with CRLF and comment lines: every chunk seam, file and
    stream inputs, 1 thread and all cores give the reference's arrays."""
    monkeypatch.setenv("GDWD_INGEST_THREADS", threads)
    ref = REF["big"]
    text = big_libsvm()
    p = tmp_path / "big.svm"
    p.write_bytes(text.encode())
    for raw in (G.parse_libsvm(p), G.parse_libsvm(io.StringIO(text, newline=None))):
        x = raw.X
        got = {"colptr": x.colptr, "rowidx": x.rowidx, "values": x.values}
        xc, _, meta = G.preprocess(raw)
        got.update({"pcolptr": xc.colptr, "prowidx": xc.rowidx, "pvalues": xc.values, "kept": meta.kept_ids,
                    "scales": meta.scales})
        for k, v in got.items():
            assert _sha(v) == ref["sha"][k], k
        assert _sha(raw.labels) == ref["labels"]


def test_errors_at_chunk_seams_report_the_first_line(monkeypatch):
    """An error late in a multi-chunk text and another earlier: the earliest
    line wins, as in the reference's single pass."""
    monkeypatch.setenv("GDWD_INGEST_THREADS", "8")
    lines = big_libsvm().splitlines(keepends=True)
    lines[30000] = "1 5:1 2:1\n"
    lines[12345] = "1 0:1\n"
    with pytest.raises(G.ParseError) as ei:
        G.parse_libsvm(io.StringIO("".join(lines), newline=None))
    assert ei.value.line_no == 12346 and "not positive" in str(ei.value)


def test_preprocess_all_zero_and_file_errors(tmp_path):
    raw = G.RawDataset(X=G.SparseMatrixCSC(3, 2, [0, 0, 0], [], []), labels=np.array([1.0, -1.0]), source_path="x")
    with pytest.raises(ValueError, match="all features are zero"):
        G.preprocess(raw)
    with pytest.raises(FileNotFoundError):
        G.parse_libsvm(tmp_path / "missing.svm")


def test_model_file_round_trip(tmp_path):
    meta = G.FeatureMeta(kept_ids=np.array([0, 2, 5]), scales=np.array([1.5, 2.0, 0.25]), d_original=7)
    m = G.ModelFile(q=1.0, C=12.5, z_scale=3.0, mu=1.0, feature_meta=meta, w=np.array([0.1, -1 / 3, 2e-17]),
                    beta=-0.75, solver_info={"iterations": 10, "converged": False})
    p = tmp_path / "m.json"
    G.write_model(m, p)
    r = G.read_model(p)
    assert r.w.tolist() == m.w.tolist() and r.beta == m.beta and r.C == m.C
    assert r.feature_meta.kept_ids.tolist() == [0, 2, 5] and r.solver_info == m.solver_info
    assert np.array_equal(r.composite_weights(), m.composite_weights())
    doc = json.loads(p.read_text())
    doc["format_version"] = 2
    p.write_text(json.dumps(doc))
    with pytest.raises(G.ModelFormatError, match="unsupported model format_version"):
        G.read_model(p)
    del doc["format_version"]
    doc.pop("w")
    doc["format_version"] = 1
    p.write_text(json.dumps(doc))
    with pytest.raises(G.ModelFormatError, match="missing field 'w'"):
        G.read_model(p)
