"""CPU-only tests: the C-ABI library loads and exports every header symbol,
host-side mirror logic (strategies, errors, PolMat views, text I/O), and the
product path fails loudly without a GPU (no CPU fallback)."""
import ctypes
import random

import pytest

import paper_1905_04356_b200 as F
from paper_1905_04356_b200 import _lib, errors, forms
from golden_util import small


def test_library_exports_all_header_symbols():
    L = _lib.lib()
    names = _lib.exported_symbols()
    assert "fpm_polmat_mul" in names and "fpm_pmbasis" in names
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert L.fpm_version() >= 100


def test_field_info_matches_reference_convention():
    L = _lib.lib()
    for rec in small()["primes"]:
        k = ctypes.c_int()
        r = ctypes.c_uint64()
        assert L.fpm_field_info(rec["p"], ctypes.byref(k), ctypes.byref(r)) == 0
        assert k.value == rec["two_adicity"] and r.value == rec["ntt_root"]
    assert L.fpm_field_info(91, None, None) == 9  # CompositeModulus
    assert L.fpm_field_info(2, None, None) == 8   # OutOfRange


def test_field_new_mirror():
    for rec in small()["primes"]:
        ctx = F.field_new(rec["p"])
        assert (ctx.two_adicity, ctx.ntt_root) == (rec["two_adicity"], rec["ntt_root"])
    with pytest.raises(errors.CompositeModulus):
        F.field_new(91)
    with pytest.raises(errors.OutOfRange):
        F.field_new(1 << 62)


def _pm(p, rows, n):
    return F.PolMat(F.field_new(p), rows, ncols=n)


def test_applicable_strategies_match_reference():
    for rec in small()["mul"]:
        A = _pm(rec["p"], rec["A"], rec["k"])
        B = _pm(rec["p"], rec["B"], rec["n"])
        assert F.applicable_strategies(A, B) == rec["strategies"]


def test_forced_strategy_errors_without_gpu():
    ctx = F.field_new(3)
    A = F.PolMat(ctx, [[[1, 2, 1, 1]]])
    B = F.PolMat(ctx, [[[1, 1, 2, 1, 1]]])
    with pytest.raises(ValueError):
        F.pm_mul(A, B, strategy="bogus")
    with pytest.raises(errors.OrderTooSmall):
        F.pm_mul(A, B, strategy="ntt")          # two-adicity 1 < log2(8)
    with pytest.raises(errors.OrderTooSmall):
        F.pm_mul(A, B, strategy="geometric")    # 8 points > p - 1
    with pytest.raises(errors.FieldTooSmall):
        F.pm_mul(A, B, strategy="vandermonde")  # 8 points > p
    with pytest.raises(errors.DimMismatch):
        F.pm_mul(A, F.PolMat(ctx, [[[1]], [[1]]]))
    with pytest.raises(errors.CtxMismatch):
        F.pm_mul(A, F.PolMat(F.field_new(5), [[[1]]]))


def test_zero_shortcut_needs_no_device():
    ctx = F.field_new(97)
    Z = F.PolMat.zeros(ctx, 2, 3)
    B = F.PolMat(ctx, [[[1, 2]], [[3]], [[4, 5, 6]]])
    assert F.pm_mul(Z, B).rows == [[[]], [[]]]


def test_product_path_has_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    ctx = F.field_new(97)
    A = F.PolMat(ctx, [[[1, 2]]])
    with pytest.raises(_lib.FpmBackendError):
        F.pm_mul(A, A)


def test_middle_product_precondition_errors():
    ctx = F.field_new(97)
    A = F.PolMat(ctx, [[[1, 2, 3]]])
    B = F.PolMat(ctx, [[[1] * 5]])
    with pytest.raises(errors.DegreeTooLarge):
        F.pm_middle_product(A, B, 2, 4)   # deg A = 2 >= c = 2
    with pytest.raises(errors.DegreeTooLarge):
        F.pm_middle_product(A, B, 3, 1)   # deg B = 4 >= c + d


def test_polmat_views_and_text_roundtrip():
    ctx = F.field_new(97)
    rng = random.Random(1)
    M = F.random_polmat(ctx, 3, 2, 5, rng)
    assert F.PolMat.from_matpoly(ctx, M.to_matpoly()) == M
    assert F.polmat_from_text(F.polmat_to_text(M)) == M
    assert M.transpose().transpose() == M
    assert M.truncate(2).degree <= 1
    assert M.slice_coeffs(1, 3).degree <= 1
    D = M.to_dense()
    assert F.polmat.from_dense(ctx, D) == M


def test_random_polmat_matches_reference_draw_order():
    # fpmat.polmat.random_polmat draws rng.randrange(p) entry by entry
    ctx = F.field_new(2013265921)
    a = F.random_polmat(ctx, 2, 2, 3, random.Random(9))
    rng = random.Random(9)
    flat = [rng.randrange(ctx.p) for _ in range(16)]
    assert [c for r in a.rows for e in r for c in e] == [c for c in flat]


def test_forms_predicates_on_reference_outputs():
    for rec in small()["pmbasis"]:
        P = _pm(rec["p"], rec["P"], rec["m"])
        assert forms.is_owp(P, rec["s"])
        assert forms.rdeg(P, rec["s"]) == rec["rdeg"]


def test_bridge_rebinds_and_restores(tmp_path, monkeypatch):
    """install_into_reference rebinds the names reference modules imported
     and uninstall restores them; uses a stand-in package."""
    pkg = tmp_path / "fakefpmat"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    (pkg / "polmat.py").write_text(
        "class PolMat:\n"
        "    def __init__(self, ctx, rows, ncols=None):\n"
        "        self.ctx, self.rows = ctx, rows\n"
        "def pm_mul(A, B, strategy=None):\n    return 'ref'\n"
        "def _pm_middle(A, B, c, d):\n    return 'ref'\n")
    (pkg / "appint.py").write_text(
        "from .polmat import pm_mul, _pm_middle\n"
        "def pmbasis(F, o, s):\n    return 'ref'\n")
    (pkg / "kernel.py").write_text("from .polmat import pm_mul\nfrom .appint import pmbasis\n")
    monkeypatch.syspath_prepend(str(tmp_path))
    import importlib

    fake = importlib.import_module("fakefpmat")
    from paper_1905_04356_b200.bridge import install_into_reference, uninstall

    saved = install_into_reference(fake)
    kern = importlib.import_module("fakefpmat.kernel")
    app = importlib.import_module("fakefpmat.appint")
    assert kern.pm_mul is not saved[("fakefpmat.kernel", "pm_mul")]
    assert app.pmbasis is not saved[("fakefpmat.appint", "pmbasis")]
    assert app._pm_middle is not saved[("fakefpmat.appint", "_pm_middle")]
    uninstall(saved)
    assert kern.pm_mul(None, None) == "ref" and app.pmbasis(None, 1, [0]) == "ref"


def test_polmat_entrywise_arithmetic():
    ctx = F.field_new(97)
    A = F.PolMat(ctx, [[[1, 96], [5]], [[], [3, 4, 90]]])
    B = F.PolMat(ctx, [[[96, 1], []], [[2], [94, 93, 7]]])
    assert (A + B).rows == [[[], [5]], [[2], []]]  # 3+94, 4+93, 90+7 = 0 mod 97
    assert (A - A).is_zero()
    assert (A + B - B) == A
    assert A.scale(-1) == F.PolMat.zeros(ctx, 2, 2) - A
    assert (A + B).rows[0][0] == []  # 1+96 = 0, 96+1 = 0 -> trimmed


def test_caller_goldens_present():
    import json
    import os

    d = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "callers.json")))
    assert len(d["fracrec"]) >= 10 and len(d["kernel"]) >= 6
