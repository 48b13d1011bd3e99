"""Callers one level above the hot path against the
reference's own outputs (tests/golden/make_golden_callers.py): fraction
reconstruction from a series and kernel bases, each one PM-Basis (+ one
product) on the B200."""
import json
import os

import pytest

import paper_1905_04356_b200 as F

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "callers.json")) as f:
    CALLERS = json.load(f)


def _pm(p, rows, ncols):
    return F.PolMat(F.field_new(p), rows, ncols=ncols)


@pytest.mark.parametrize("idx", range(len(CALLERS["fracrec"])))
def test_fracrec_series_matches_reference(idx):
    rec = CALLERS["fracrec"][idx]
    H = _pm(rec["p"], rec["H"], rec["n"])
    if "error" in rec:
        with pytest.raises(getattr(F.errors, rec["error"])):
            F.fraction.fracrec_series(H, rec["D"])
        return
    d = F.fraction.fracrec_series(H, rec["D"])
    assert d.Q.rows == rec["Q"] and d.R.rows == rec["R"]


@pytest.mark.parametrize("idx", range(len(CALLERS["kernel"])))
def test_kernel_direct_matches_reference(idx):
    rec = CALLERS["kernel"][idx]
    Fm = _pm(rec["p"], rec["F"], rec["n"])
    kb = F.kernel.kernel_direct(Fm, rec["s"])
    assert kb.K.rows == rec["K"]
    if kb.K.m:
        assert F.pm_mul(kb.K, Fm).is_zero()


@pytest.mark.parametrize("idx", range(len(CALLERS["fracrec_points"])))
def test_fracrec_points_matches_reference(idx):
    """fracrec_points (fraction.py:72-97): one GPU PM-IntBasis at 2D points."""
    rec = CALLERS["fracrec_points"][idx]
    ctx = F.field_new(rec["p"])
    d = F.fraction.fracrec_points(ctx, rec["Hvals"], rec["pts"], rec["D"])
    assert d.Q.rows == rec["Q"] and d.R.rows == rec["R"]


@pytest.mark.parametrize("idx", range(len(CALLERS["kernel_interp"])))
def test_kernel_direct_interp_matches_reference(idx):
    """kernel_direct(flavor="interp") (kernel.py:58-70): evaluation on a
    geometric progression + GPU PM-IntBasis."""
    rec = CALLERS["kernel_interp"][idx]
    Fm = _pm(rec["p"], rec["F"], rec["n"])
    kb = F.kernel.kernel_direct(Fm, rec["s"], flavor="interp")
    assert kb.K.rows == rec["K"]
    if kb.K.m:
        assert F.pm_mul(kb.K, Fm).is_zero()
