"""Polynomial matrices over F_p and their product (mirror of fpmat/polmat.py).

``PolMat`` keeps the reference storage (row-major lists of trimmed coefficient
lists, polmat.py:48-58) and the same view helpers, so reference callers can
switch modules unchanged.  The arithmetic entry points -- ``pm_mul``,
``pm_middle_product`` / ``_pm_middle`` and ``Multiplier`` -- convert to the
dense device layout and run the sm_100a kernels of libfpm_b200.so; there is
no CPU implementation behind them.
"""
import numpy as np

from . import dense
from .errors import (
    CtxMismatch,
    DegreeTooLarge,
    DimMismatch,
    EnvelopeExceeded,
    FieldTooSmall,
    NoSuchElement,
    OrderTooSmall,
)
from .modring import field_new, order_at_least

STRATEGIES = ("naive", "ntt", "geometric", "vandermonde")


def _trim(c):
    while c and c[-1] == 0:
        c.pop()
    return c


class PolMat:
    """Dense m x n matrix of polynomials, immutable by convention (polmat.py:48)."""

    __slots__ = ("ctx", "m", "n", "rows", "_deg")

    def __init__(self, ctx, rows, ncols=None):
        self.ctx = ctx
        self.m = len(rows)
        self.n = len(rows[0]) if self.m else (ncols or 0)
        self.rows = rows
        self._deg = None

    @classmethod
    def from_entries(cls, ctx, entries):
        p = ctx.p
        rows = []
        for row in entries:
            out = []
            for e in row:
                coeffs = getattr(e, "coeffs", e)
                out.append(_trim([int(c) % p for c in coeffs]))
            rows.append(out)
        return cls(ctx, rows)

    @classmethod
    def zeros(cls, ctx, m, n):
        return cls(ctx, [[[] for _ in range(n)] for _ in range(m)], ncols=n)

    @classmethod
    def identity(cls, ctx, n):
        rows = [[[] for _ in range(n)] for _ in range(n)]
        for i in range(n):
            rows[i][i] = [1]
        return cls(ctx, rows, ncols=n)

    @classmethod
    def from_const(cls, ctx, mat):
        p = ctx.p
        return cls(ctx, [[([v % p] if v % p else []) for v in row] for row in mat])

    @property
    def degree(self):
        """Max entry degree; -1 for the zero matrix (polmat.py:95-104)."""
        if self._deg is None:
            d = -1
            for row in self.rows:
                for e in row:
                    if len(e) - 1 > d:
                        d = len(e) - 1
            self._deg = d
        return self._deg

    def coefficient(self, k):
        return [[e[k] if k < len(e) else 0 for e in row] for row in self.rows]

    def to_matpoly(self):
        return [self.coefficient(k) for k in range(self.degree + 1)]

    @classmethod
    def from_matpoly(cls, ctx, coeffs, m=None, n=None):
        if not coeffs:
            return cls.zeros(ctx, m or 0, n or 0)
        m = len(coeffs[0])
        n = len(coeffs[0][0]) if m else 0
        return cls(ctx, [[_trim([c[i][j] for c in coeffs]) for j in range(n)]
                         for i in range(m)], ncols=n)

    def transpose(self):
        return PolMat(self.ctx, [[self.rows[i][j][:] for i in range(self.m)]
                                 for j in range(self.n)], ncols=self.m)

    def truncate(self, k):
        return PolMat(self.ctx, [[_trim(e[:k]) for e in row] for row in self.rows],
                      ncols=self.n)

    def slice_coeffs(self, lo, hi):
        return PolMat(self.ctx, [[_trim(e[lo:hi]) for e in row] for row in self.rows],
                      ncols=self.n)

    def shift(self, k):
        return PolMat(self.ctx, [[([0] * k + e if e else []) for e in row]
                                 for row in self.rows], ncols=self.n)

    def submatrix(self, rows, cols):
        cols = list(cols)
        return PolMat(self.ctx, [[self.rows[i][j][:] for j in cols] for i in rows],
                      ncols=len(cols))

    def vstack(self, other):
        _same_ctx(self, other)
        if self.n != other.n:
            raise DimMismatch("column counts differ")
        return PolMat(self.ctx, [r[:] for r in self.rows] + [r[:] for r in other.rows],
                      ncols=self.n)

    def hstack(self, other):
        _same_ctx(self, other)
        if self.m != other.m:
            raise DimMismatch("row counts differ")
        return PolMat(self.ctx, [a[:] + b[:] for a, b in zip(self.rows, other.rows)])

    def is_zero(self):
        return all(not e for row in self.rows for e in row)

    # ---- entrywise arithmetic (host; polmat.py:199-231) ----------------------
    def _entrywise(self, other, sign):
        _same_ctx(self, other)
        if (self.m, self.n) != (other.m, other.n):
            raise DimMismatch(f"shapes {self.m}x{self.n} and {other.m}x{other.n} differ")
        p = self.ctx.p

        def comb(a, b):
            L = max(len(a), len(b))
            a = a + [0] * (L - len(a))
            b = b + [0] * (L - len(b))
            return _trim([(x + sign * y) % p for x, y in zip(a, b)])

        return PolMat(self.ctx, [[comb(a, b) for a, b in zip(ra, rb)]
                                 for ra, rb in zip(self.rows, other.rows)], ncols=self.n)

    def __add__(self, other):
        return self._entrywise(other, 1)

    def __sub__(self, other):
        return self._entrywise(other, -1)

    def scale(self, c):
        p = self.ctx.p
        c %= p
        return PolMat(self.ctx, [[_trim([x * c % p for x in e]) for e in row]
                                 for row in self.rows], ncols=self.n)

    def __eq__(self, other):
        # duck-typed so reference PolMat values compare equal (polmat.py:184-189)
        return (hasattr(other, "rows") and hasattr(other, "ctx")
                and self.ctx.p == other.ctx.p and self.rows == other.rows)

    def __hash__(self):
        return hash((self.ctx.p, tuple(tuple(tuple(e) for e in r) for r in self.rows)))

    def __repr__(self):
        return f"PolMat(p={self.ctx.p}, {self.m}x{self.n}, deg={self.degree})"

    # ---- dense conversion --------------------------------------------------
    def to_dense(self, length=None):
        """(m, n, L) uint64 numpy array, L = degree + 1 unless given."""
        return to_dense(self, length)


def _same_ctx(A, B):
    if A.ctx.p != B.ctx.p:
        raise CtxMismatch("matrices live in different prime fields")


def _mul_dims(A, B):
    _same_ctx(A, B)
    if A.n != B.m:
        raise DimMismatch(f"cannot multiply {A.m}x{A.n} by {B.m}x{B.n}")


def to_dense(M, length=None):
    L = (M.degree + 1) if length is None else length
    out = np.zeros((M.m, M.n, max(L, 0)), dtype=np.uint64)
    for i, row in enumerate(M.rows):
        for j, e in enumerate(row):
            if e:
                le = min(len(e), L)
                out[i, j, :le] = e[:le]
    return out


def from_dense(ctx, D, ncols=None):
    """Dense (m, n, L) -> PolMat with trimmed entries (upoly.py:34-37)."""
    D = np.asarray(D)
    m, n = D.shape[0], D.shape[1]
    L = D.shape[2] if D.ndim == 3 else 0
    if L == 0:
        return PolMat(ctx, [[[] for _ in range(n)] for _ in range(m)], ncols=n)
    nz = D != 0
    lens = np.where(nz.any(axis=2), L - np.argmax(nz[:, :, ::-1], axis=2), 0)
    rows = [[D[i, j, : lens[i, j]].tolist() for j in range(n)] for i in range(m)]
    return PolMat(ctx, rows, ncols=n)


def _device_mul(A, B):
    p = A.ctx.p
    a = dense.to_device(to_dense(A), p)
    b = dense.to_device(to_dense(B), p)
    c = dense.pm_mul_dense(a, b, p)
    return from_dense(A.ctx, dense.to_numpy(c, p), ncols=B.n)


def applicable_strategies(A, B):
    """Strategies valid for this product, in dispatch order (polmat.py:431-444)."""
    ctx = A.ctx
    out = ["naive"]
    if A.degree < 0 or B.degree < 0:
        return out
    npts = A.degree + B.degree + 1
    if max(1, (npts - 1).bit_length()) <= ctx.two_adicity:
        out.append("ntt")
    if npts <= ctx.p - 1:
        out.append("geometric")
    if npts <= ctx.p:
        out.append("vandermonde")
    return out


def _check_forced(A, B, strategy):
    """Preconditions a forced reference strategy would raise on."""
    ctx = A.ctx
    npts = A.degree + B.degree + 1
    if strategy == "ntt":
        if max(1, (npts - 1).bit_length()) > ctx.two_adicity:  # polmat.py:293-296
            raise OrderTooSmall("no long enough root of unity for this product")
    elif strategy == "geometric":
        try:  # polmat.py:311-315
            order_at_least(ctx, npts)
        except NoSuchElement:
            raise OrderTooSmall(f"field too small for {npts} geometric points")
    elif strategy == "vandermonde":
        if npts > ctx.p:  # polmat.py:397-398
            raise FieldTooSmall(f"need {npts} distinct points, field has {ctx.p}")


def pm_mul(A, B, strategy=None):
    """Exact product A*B (polmat.py:447-467).

    Every reference strategy returns the same unique product; the
    strategy argument keeps its validation semantics (ValueError on unknown
    names, the forced strategy's applicability errors) and the product itself
    always runs on the GPU."""
    _mul_dims(A, B)
    if strategy is not None:
        if strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {strategy!r}")
        _check_forced(A, B, strategy)
    if A.degree < 0 or B.degree < 0 or A.n == 0:
        return PolMat.zeros(A.ctx, A.m, B.n)
    return _device_mul(A, B)


def pm_middle_product(A, B, c, d):
    """Coefficient slice c..c+d-1 of A*B with the reference contract
    (polmat.py:470-481)."""
    _mul_dims(A, B)
    if A.degree >= c and c > 0:
        raise DegreeTooLarge(f"deg A = {A.degree} must be < c = {c}")
    if B.degree >= c + d:
        raise DegreeTooLarge(f"deg B = {B.degree} must be < c+d = {c + d}")
    return _pm_middle(A, B, c, d)


def _pm_middle(A, B, c, d, exact=False):
    """Slice [c, c+d) of A*B (polmat.py:484-536).

    exact=False reproduces the reference bit for bit, including the aliasing
    of its cyclic fold; exact=True returns the
    true slice promised by SPEC S:219."""
    ctx = A.ctx
    if A.degree < 0 or B.degree < 0 or d <= 0:
        return PolMat.zeros(ctx, A.m, B.n)
    p = ctx.p
    a = dense.to_device(to_dense(A), p)
    b = dense.to_device(to_dense(B), p)
    r = dense.pm_middle_dense(a, b, c, d, p, exact=exact)
    return from_dense(ctx, dense.to_numpy(r, p), ncols=B.n)


class Multiplier:
    """Fixed left factor A for repeated products (polmat.py:550-602).

    apply(B) == pm_mul(A, B) for deg B <= max_rhs_degree, else
    EnvelopeExceeded.  A stays resident on the device between calls."""

    __slots__ = ("A", "max_rhs_degree", "_dev")

    def __init__(self, A, max_rhs_degree):
        self.A = A
        self.max_rhs_degree = max_rhs_degree
        self._dev = None

    def apply(self, B):
        if B.degree > self.max_rhs_degree:
            raise EnvelopeExceeded(f"deg B = {B.degree} exceeds envelope {self.max_rhs_degree}")
        _mul_dims(self.A, B)
        A = self.A
        if A.degree < 0 or B.degree < 0 or A.n == 0:
            return PolMat.zeros(A.ctx, A.m, B.n)
        p = A.ctx.p
        if self._dev is None:
            # A's forward transforms are computed once and cached on the device
            self._dev = dense.DenseMultiplier(dense.to_device(to_dense(A), p), p,
                                              self.max_rhs_degree + 1)
        b = dense.to_device(to_dense(B), p)
        c = self._dev.apply(b)
        return from_dense(A.ctx, dense.to_numpy(c, p), ncols=B.n)


def multiplier_precompute(A, max_rhs_degree):
    return Multiplier(A, max_rhs_degree)


def multiplier_apply(mult, B):
    return mult.apply(B)


# ---- text interchange (polmat.py:617-647) -----------------------------------
# The reference's text format, written and parsed natively (csrc/textio.cu via
# textio.dense_to_text / dense_from_text), byte for byte the same.

def polmat_to_text(A):
    from . import textio

    L = max(A.degree + 1, 0)
    return textio.dense_to_text(to_dense(A, L), A.ctx.p)


def polmat_from_text(text, ctx=None):
    from . import textio

    p, D = textio.dense_from_text(text)
    if ctx is None or ctx.p != p:
        ctx = field_new(p)
    return from_dense(ctx, D, ncols=D.shape[1])


def random_polmat(ctx, m, n, deg, rng):
    """Same draw order as polmat.py:650-659 (rng.randrange per coefficient)."""
    p = ctx.p
    return PolMat(ctx, [[_trim([rng.randrange(p) for _ in range(deg + 1)]) for _ in range(n)]
                        for _ in range(m)], ncols=n)
