"""Left kernel bases from one approximant basis (the `kernel_direct` route of
the reference `kernel.py`, one level above the hot path: a single PM-Basis
on the B200).

kernel_direct(F, s) follows ref:kernel.py:42-76 (flavor "approx"): with
d = deg F and the shift normalised to minimum 0, the order d + delta basis
(delta = n d + max(s0) + 1) contains the kernel rows as its rows of s0-degree
below delta; they are returned sorted by pivot (ref:kernel.py:35-40).  The
"interp" flavor evaluates F on a geometric progression of that length
(modring.order_at_least) and takes the GPU PM-IntBasis instead
(ref:kernel.py:58-70).
"""
from .appint import eval_polmat_points, pm_intbasis, pmbasis
from .errors import NoGeometricGrid, NoSuchElement
from .forms import NEG_INF, pivot_profile, rdeg
from .modring import order_at_least


class KernelBasis:
    """Rows K with K F = 0, the shift, and a form certificate."""

    __slots__ = ("K", "shift", "certificate")

    def __init__(self, K, shift, certificate):
        self.K, self.shift, self.certificate = K, shift, certificate

    def __repr__(self):
        return f"KernelBasis({self.K.m}x{self.K.n}, {self.certificate})"


def _by_pivot(M, s):
    if M.m == 0:
        return M
    prof = pivot_profile(M, s)
    order = sorted(range(M.m), key=lambda i: (prof[i][1], i))
    return M.submatrix(order, range(M.n))


def kernel_direct(F, s, flavor="approx"):
    if any(si < 0 for si in s):
        raise ValueError("kernel_direct expects a nonnegative shift")
    ctx = F.ctx
    m, n = F.m, F.n
    d = max(F.degree, 0)
    s0 = [si - min(s) for si in s] if s else []
    delta = n * d + (max(s0) if s0 else 0) + 1
    order = d + delta
    if flavor == "approx":
        P = pmbasis(F, order, s0)
    elif flavor == "interp":
        try:
            alpha = order_at_least(ctx, order)
        except NoSuchElement:
            raise NoGeometricGrid(f"field has no geometric progression of length {order}")
        pts = [1] * order
        for i in range(1, order):
            pts[i] = pts[i - 1] * alpha % ctx.p
        E = eval_polmat_points(F, pts, ctx)  # pm_eval at every point (polmat.py:539-543)
        P = pm_intbasis(E, pts, s0, ctx)
    else:
        raise ValueError(f"unknown flavor {flavor!r}")
    degs = rdeg(P, s0)
    keep = [i for i in range(m) if degs[i] != NEG_INF and degs[i] < delta]
    return KernelBasis(_by_pivot(P.submatrix(keep, range(m)), s), list(s), "owp")
