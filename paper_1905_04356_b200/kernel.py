"""Left kernel bases from one approximant basis (the `kernel_direct` route of
the reference `kernel.py`, one level above the hot path: a single PM-Basis
on the B200).

kernel_direct(F, s) follows ref:kernel.py:42-76 (flavor "approx"): with
d = deg F and the shift normalised to minimum 0, the order d + delta basis
(delta = n d + max(s0) + 1) contains the kernel rows as its rows of s0-degree
below delta; they are returned sorted by pivot (ref:kernel.py:35-40).  The
"interp" flavor needs PM-IntBasis, outside this repository's scope.
"""
from .appint import pmbasis
from .forms import NEG_INF, pivot_profile, rdeg


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
    if flavor != "approx":
        raise ValueError(f"unsupported flavor {flavor!r} (only 'approx' is provided here)")
    m, n = F.m, F.n
    d = max(F.degree, 0)
    s0 = [si - min(s) for si in s] if s else []
    delta = n * d + (max(s0) if s0 else 0) + 1
    P = pmbasis(F, d + delta, s0)
    degs = rdeg(P, s0)
    keep = [i for i in range(m) if degs[i] != NEG_INF and degs[i] < delta]
    return KernelBasis(_by_pivot(P.submatrix(keep, range(m)), s), list(s), "owp")
