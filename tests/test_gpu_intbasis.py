"""Interpolant bases on the GPU against the reference's
own outputs (tests/golden/intbasis.json, make_golden_intbasis.py)."""
import hashlib
import json
import os
import random

import numpy as np
import pytest

import paper_1905_04356_b200 as F
from golden_util import GOLDEN

pytestmark = pytest.mark.gpu


def _golden():
    with open(os.path.join(GOLDEN, "intbasis.json")) as f:
        return json.load(f)


def draw_case(seed, p, m, n, order, geometric=False, zero_every=0):
    """Same draw order as tests/golden/make_golden_intbasis.py:draw_case."""
    rng = random.Random(seed)
    E = []
    for t in range(order):
        if zero_every and t % zero_every == 0:
            E.append([[0] * n for _ in range(m)])
        else:
            E.append([[rng.randrange(p) for _ in range(n)] for _ in range(m)])
    if geometric:
        a0, r = rng.randrange(1, p), rng.randrange(2, p)
        alpha, cur = [], a0
        for _ in range(order):
            alpha.append(cur)
            cur = cur * r % p
    else:
        alpha = rng.sample(range(p), order)
    return E, alpha


@pytest.mark.parametrize("idx", range(14))
def test_intbasis_matches_reference(idx):
    g = _golden()["cases"][idx]
    ctx = F.field_new(g["p"])
    E, alpha = draw_case(g["seed"], g["p"], g["m"], g["n"], g["order"], g["geometric"],
                         g["zero_every"])
    fn = F.m_intbasis if g["flavor"] == "m" else F.pm_intbasis
    P = fn(E, alpha, list(g["shift"]), ctx)
    txt = F.polmat_to_text(P)
    assert hashlib.sha256(txt.encode()).hexdigest() == g["sha256"]
    if "rows" in g:
        assert P.rows == g["rows"]


def test_intbasis_duplicate_points():
    ctx = F.field_new(97)
    E = [[[1], [2]], [[3], [4]]]
    with pytest.raises(F.errors.DuplicatePoints):
        F.pm_intbasis(E, [5, 5], [0, 0], ctx)


def test_intbasis_is_an_interpolant_basis():
    """P(alpha_t) E_t = 0 for every point (the defining property)."""
    p = 2013265921
    ctx = F.field_new(p)
    E, alpha = draw_case(42, p, 10, 4, 90)
    P = F.pm_intbasis(E, alpha, [0] * 10, ctx)
    vals = F.eval_polmat_points(P, alpha, ctx)
    for t in range(len(alpha)):
        A = np.array(vals[t], dtype=object)
        R = A.dot(np.array(E[t], dtype=object)) % p
        assert not R.any()


@pytest.mark.parametrize("idx", range(3))
def test_eval_points_matches_reference(idx):
    g = _golden()["evals"][idx]
    ctx = F.field_new(g["p"])
    P = F.PolMat(ctx, g["rows"])
    assert F.eval_polmat_points(P, g["pts"], ctx) == g["vals"]
