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


# ---- interpolant bases (appint.py:200-319) -----------------------------------

def _check_points(alpha, p=None):
    """appint._check_points: pairwise distinct points (appint.py:203-205)."""
    from .errors import DuplicatePoints

    if len(set(alpha)) != len(alpha):
        raise DuplicatePoints("interpolation points must be pairwise distinct")


def _intbasis(E, alpha, s, ctx):
    _check_points(alpha)
    p = ctx.p
    m = len(E[0]) if E else len(s)
    if len(s) != m:
        raise ValueError("shift length must match the row count")
    n = len(E[0][0]) if E and E[0] else 0
    import numpy as np

    Ed = np.zeros((len(E), m, n), dtype=np.uint64)
    for t, mat in enumerate(E):
        for i, row in enumerate(mat):
            Ed[t, i, : len(row)] = [int(x) % p for x in row]
    P, _ = dense.intbasis_dense(dense.to_device(Ed, p), [int(a) for a in alpha], s, p)
    return from_dense(ctx, dense.to_numpy(P, p), ncols=m)


def m_intbasis(E, alpha, s, ctx):
    """Iterative s-ordered weak Popov interpolant basis (appint.py:208-238).

    E: list of m x n constant matrices, one per point of alpha; pivot rows of
    each order-1 step are multiplied by (x - alpha_k)."""
    return _intbasis(E, alpha, s, ctx)


def pm_intbasis(E, alpha, s, ctx):
    """Divide-and-conquer interpolant basis (appint.py:290-319); equal to
    m_intbasis (product of the same canonical steps)."""
    return _intbasis(E, alpha, s, ctx)


def eval_polmat_points(P, pts, ctx):
    """[P(x) for x in pts] as constant matrices (appint.py:262-287)."""
    p = ctx.p
    if not pts:
        return []
    L = max(P.degree + 1, 1)
    d = dense.to_device(to_dense(P, L), p)
    vals = dense.to_numpy(dense.eval_points_dense(d, [int(x) for x in pts], p), p)
    return [[[int(vals[t, i, j]) for j in range(P.n)] for i in range(P.m)]
            for t in range(len(pts))]
