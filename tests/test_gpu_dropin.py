"""The drop-in, run for real: the UNMODIFIED reference package `fpmat`
with its hot-path names rebound to the B200 library
(bridge.install_into_reference), then the reference's OWN
callers executed -- fraction reconstruction (fraction.py:54-97), kernel
bases (kernel.py:42-76), and pm_mul / pmbasis through the reference module
attributes -- on the inputs of tests/golden/callers.json, compared with the
outputs the unmodified reference produced (make_golden_callers.py).

The reference must be present (tests/refpkg.py resolution order); these
tests fail rather than skip when it is not.
"""
import json
import os

import pytest

from paper_1905_04356_b200 import _lib
from paper_1905_04356_b200.bridge import install_into_reference, uninstall
from refpkg import import_reference

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "callers.json")) as f:
    CALLERS = json.load(f)


@pytest.fixture(scope="module")
def fpmat():
    ref = import_reference()
    assert ref is not None, ("reference fpmat not found ($FPMAT_REF, /root/reference/pkg/src, "
                             "baseline/_ref): the drop-in cannot be checked")
    import fpmat.fraction  # noqa: F401  (modules bind the names at import)
    import fpmat.kernel  # noqa: F401
    import fpmat.solve  # noqa: F401

    saved = install_into_reference(ref)
    yield ref
    uninstall(saved)


def _ref_pm(fpmat, p, rows, ncols):
    return fpmat.polmat.PolMat(fpmat.modring.field_new(p), rows, ncols=ncols)


def _gpu_launches(fn):
    n0 = _lib.launch_count()
    out = fn()
    return out, _lib.launch_count() - n0


@pytest.mark.parametrize("idx", range(len(CALLERS["fracrec"])))
def test_reference_fracrec_series_on_gpu(fpmat, idx):
    rec = CALLERS["fracrec"][idx]
    H = _ref_pm(fpmat, rec["p"], rec["H"], rec["n"])
    if "error" in rec:
        with pytest.raises(getattr(fpmat.errors, rec["error"])):
            fpmat.fraction.fracrec_series(H, rec["D"])
        return
    d, launched = _gpu_launches(lambda: fpmat.fraction.fracrec_series(H, rec["D"]))
    assert launched > 0, "the reference caller did not reach the B200 library"
    assert isinstance(d.Q, fpmat.polmat.PolMat)
    assert d.Q.rows == rec["Q"] and d.R.rows == rec["R"]


@pytest.mark.parametrize("idx", range(len(CALLERS["kernel"])))
def test_reference_kernel_direct_on_gpu(fpmat, idx):
    rec = CALLERS["kernel"][idx]
    F = _ref_pm(fpmat, rec["p"], rec["F"], rec["n"])
    kb, launched = _gpu_launches(lambda: fpmat.kernel.kernel_direct(F, rec["s"]))
    assert launched > 0
    assert kb.K.rows == rec["K"]
    if kb.K.m:
        assert fpmat.polmat.pm_mul(kb.K, F).is_zero()


@pytest.mark.parametrize("idx", range(len(CALLERS["fracrec_points"])))
def test_reference_fracrec_points_on_gpu(fpmat, idx):
    rec = CALLERS["fracrec_points"][idx]
    ctx = fpmat.modring.field_new(rec["p"])
    d = fpmat.fraction.fracrec_points(ctx, rec["Hvals"], rec["pts"], rec["D"])
    assert d.Q.rows == rec["Q"] and d.R.rows == rec["R"]


@pytest.mark.parametrize("idx", range(len(CALLERS["kernel_interp"])))
def test_reference_kernel_direct_interp_on_gpu(fpmat, idx):
    rec = CALLERS["kernel_interp"][idx]
    F = _ref_pm(fpmat, rec["p"], rec["F"], rec["n"])
    kb = fpmat.kernel.kernel_direct(F, rec["s"], flavor="interp")
    assert kb.K.rows == rec["K"]


def test_reference_pm_mul_and_pmbasis_attributes_on_gpu(fpmat):
    """fpmat.polmat.pm_mul / fpmat.appint.pmbasis as the reference exposes
    them: goldens of the unmodified reference (small.json)."""
    from golden_util import small

    for rec in small()["mul"][:40]:
        A = _ref_pm(fpmat, rec["p"], rec["A"], rec["k"])
        B = _ref_pm(fpmat, rec["p"], rec["B"], rec["n"])
        C, launched = _gpu_launches(lambda: fpmat.polmat.pm_mul(A, B))
        assert C.rows == rec["C"]
        assert launched > 0 or A.degree < 0 or B.degree < 0 or A.n == 0
    for rec in small()["pmbasis"][:12]:
        F = _ref_pm(fpmat, rec["p"], rec["F"], rec["n"])
        P = fpmat.appint.pmbasis(F, rec["sigma"], rec["s"])
        assert P.rows == rec["P"]
        assert fpmat.forms.is_owp(P, rec["s"])
