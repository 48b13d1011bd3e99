"""Approximant bases (mirror of fpmat/appint.py:24-196), GPU resident.

``pmbasis(F, order, s)`` returns exactly the matrix the reference returns:
the reference output is the product of its canonical order-1 steps
(appint.py:24-60) and does not depend on the base threshold or on how the
products are computed, so the whole recursion
-- M-Basis leaves, middle products, shift updates and the final products --
runs in libfpm_b200.so (csrc/pmbasis.cu) with data kept on the device.
"""
from . import config, dense
from .polmat import PolMat, _pm_middle, from_dense, pm_mul, to_dense  # noqa: F401


def _run(kind, F, order, s, T=None):
    if len(s) != F.m:
        raise ValueError("shift length must match the row count")
    p = F.ctx.p
    # F.truncate(order) (appint.py:186): only the first `order` coefficients matter
    L = max(min(F.degree + 1, order), 1)
    f = dense.to_device(to_dense(F, L), p)
    if kind == "pmbasis":
        P, _ = dense.pmbasis_dense(f, order, s, p, T=T if T is not None else config.PMBASIS_BASE_ORDER)
    else:
        P, _ = dense.mbasis_dense(f, order, s, p)
    return from_dense(F.ctx, dense.to_numpy(P, p), ncols=F.m)


def mbasis(F, order, s):
    """Iterative s-ordered weak Popov approximant basis (appint.py:143-180)."""
    return _run("mbasis", F, order, s)


def pmbasis(F, order, s):
    """Divide-and-conquer approximant basis (appint.py:183-196)."""
    return _run("pmbasis", F, order, s)


def mbasis1(R, s, ctx):
    """s-Popov order-1 basis of a constant matrix (appint.py:63-76).

    Equal to mbasis of R viewed as a constant polynomial matrix at order 1
    (same canonical step; R = 0 gives the identity in both)."""
    F = PolMat.from_const(ctx, R)
    if F.m == 0:
        return PolMat(ctx, [])
    return mbasis(F, 1, s)
