"""Interchange formats: the native text writer / reader
against the reference's own polmat_to_text / polmat_from_text outputs
(tests/golden/textio.json, tests/golden/make_golden_textio.py), the binary
format round trip, and the PolMat-level mirror.  Host code only: runs on CPU."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1905_04356_b200 as F
from golden_util import GOLDEN, dense
from paper_1905_04356_b200 import textio


def _golden():
    with open(os.path.join(GOLDEN, "textio.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("idx", range(7))
def test_to_text_matches_reference(idx):
    g = _golden()["to_text"][idx]
    p, m, n = g["p"], g["m"], g["n"]
    dt = np.uint32 if p < (1 << 32) else np.uint64
    M = dense(g["rows"], m, n, dtype=dt) if m else np.zeros((0, n, 0), dtype=dt)
    txt = textio.dense_to_text(M, p)
    assert hashlib.sha256(txt.encode()).hexdigest() == g["sha256"]
    if "text" in g:
        assert txt == g["text"]
    # and the PolMat-level mirror (polmat.py:617-623)
    if m:
        A = F.PolMat(F.field_new(p), [[list(e) for e in r] for r in g["rows"]], ncols=n)
        A = F.polmat.from_dense(A.ctx, M, ncols=n)
        assert F.polmat_to_text(A) == txt


@pytest.mark.parametrize("idx", range(10))
def test_from_text_matches_reference(idx):
    g = _golden()["from_text"][idx]
    p, M = textio.dense_from_text(g["text"])
    assert p == g["p"] and M.shape[:2] == (g["m"], g["n"])
    got = [[[int(c) for c in np.trim_zeros(M[i, j], "b")] for j in range(g["n"])]
           for i in range(g["m"])]
    assert got == g["rows"]
    A = F.polmat_from_text(g["text"])
    assert A.rows == g["rows"]


def test_from_text_errors_match_reference():
    for g in _golden()["errors"]:
        assert g["error"] == "ValueError"
        with pytest.raises(ValueError):
            textio.dense_from_text(g["text"])
        with pytest.raises(ValueError):
            F.polmat_from_text(g["text"])


@pytest.mark.parametrize("p,eb", [(2013265921, 4), ((1 << 60) - 93, 8)])
def test_text_and_binary_round_trip(tmp_path, p, eb):
    rng = np.random.default_rng(5)
    dt = np.uint32 if eb == 4 else np.uint64
    M = rng.integers(0, p, size=(9, 7, 301), dtype=np.uint64).astype(dt)
    M[2, 3] = 0
    M[4, 1, 150:] = 0
    p2, back = textio.dense_from_text(textio.dense_to_text(M, p))
    assert p2 == p and np.array_equal(back, M[:, :, : back.shape[2]])
    assert not M[:, :, back.shape[2]:].any()
    path = str(tmp_path / "m.fpmb")
    textio.save_binary(path, M, p)
    p3, back2, lens = textio.load_binary(path)
    assert p3 == p and np.array_equal(back2, M)
    assert lens[2, 3] == 0 and lens[4, 1] <= 150
    _, mm, _ = textio.load_binary(path, mmap=True)
    assert np.array_equal(np.asarray(mm), M)
