"""Tensor-level API over libfpm_b200.so (device-resident dense operands).

Dense layout (include/fpmat_b200.h): a polynomial matrix is a CUDA tensor of
shape (rows, cols, L), coefficient t of entry (i, j) at [i, j, t], low degree
first.  Elements are stored in int32 (p < 2^31) or int64 tensors and read
bit-for-bit as uint32 / uint64.  Every function here launches sm_100a
kernels through the C ABI; there is no CPU path.
"""
import ctypes

import numpy as np

from . import _lib


def elem_bytes_for(p):
    """uint32 storage for p < 2^31 (direct or multi-prime), uint64 otherwise."""
    return 4 if p < (1 << 31) else 8


def torch_dtype(p):
    import torch

    return torch.int32 if elem_bytes_for(p) == 4 else torch.int64


def to_device(arr, p, device=None):
    """numpy (uint) array -> CUDA tensor in the storage dtype for p."""
    import torch

    if not torch.cuda.is_available():
        raise _lib.FpmBackendError(
            "no CUDA device: the B200 product path has no CPU fallback")
    eb = elem_bytes_for(p)
    a = np.ascontiguousarray(arr, dtype=np.uint32 if eb == 4 else np.uint64)
    t = torch.from_numpy(a.view(np.int32 if eb == 4 else np.int64))
    return t.to(device or "cuda", non_blocking=False)


def to_numpy(t, p):
    eb = elem_bytes_for(p)
    a = t.detach().cpu().numpy()
    return a.view(np.uint32 if eb == 4 else np.uint64)


def _check_tensor(t, p, name):
    import torch

    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != torch_dtype(p):
        raise ValueError(f"{name} must be {torch_dtype(p)} for p={p}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def pm_mul_dense(A, B, p, out=None):
    """C = A * B over F_p; A (m,k,la), B (k,n,lb) -> C (m,n,la+lb-1).

    Replaces polmat.pm_mul (polmat.py:447-467) on dense device operands."""
    import torch

    _check_tensor(A, p, "A")
    _check_tensor(B, p, "B")
    m, k, la = A.shape
    k2, n, lb = B.shape
    if k != k2:
        from .errors import DimMismatch

        raise DimMismatch(f"cannot multiply {m}x{k} by {k2}x{n}")
    lc = la + lb - 1 if la > 0 and lb > 0 else 0
    if out is None:
        out = torch.empty((m, n, lc), dtype=A.dtype, device=A.device)
    elif tuple(out.shape) != (m, n, lc):
        raise ValueError("out has the wrong shape")
    h = _lib.context(A.device.index)
    _lib.check(_lib.lib().fpm_polmat_mul(h, p, elem_bytes_for(p), A.data_ptr(), m, k, la,
                                          B.data_ptr(), n, lb, out.data_ptr()),
               "fpm_polmat_mul")
    return out


def pm_middle_dense(A, B, c, d, p, exact=False, checked=False):
    """Coefficients [c, c+d) of A*B: reference `_pm_middle` semantics
    (polmat.py:484-536) unless exact=True (true slice)."""
    import torch

    _check_tensor(A, p, "A")
    _check_tensor(B, p, "B")
    m, k, la = A.shape
    k2, n, lb = B.shape
    if k != k2:
        from .errors import DimMismatch

        raise DimMismatch(f"cannot multiply {m}x{k} by {k2}x{n}")
    out = torch.zeros((m, n, max(d, 0)), dtype=A.dtype, device=A.device)
    if d <= 0:
        return out
    h = _lib.context(A.device.index)
    L = _lib.lib()
    if checked:
        st = L.fpm_pm_middle_product(h, p, elem_bytes_for(p), A.data_ptr(), m, k, la,
                                     B.data_ptr(), n, lb, c, d, out.data_ptr())
        _lib.check(st, "fpm_pm_middle_product")
    else:
        st = L.fpm_polmat_middle(h, p, elem_bytes_for(p), A.data_ptr(), m, k, la,
                                 B.data_ptr(), n, lb, c, d, 1 if exact else 0, out.data_ptr())
        _lib.check(st, "fpm_polmat_middle")
    return out


def _basis(fn, F, order, s, p, T=None):
    import torch

    _check_tensor(F, p, "F")
    m, n, lf = F.shape
    s_arr = (ctypes.c_int64 * max(m, 1))(*[int(x) for x in s])
    P = torch.empty((m, m, order + 1), dtype=F.dtype, device=F.device)
    lp = ctypes.c_int(0)
    rd = (ctypes.c_int64 * max(m, 1))()
    h = _lib.context(F.device.index)
    L = _lib.lib()
    if T is not None:
        _lib.check(L.fpm_set_pmbasis_threshold(h, int(T)), "fpm_set_pmbasis_threshold")
    try:
        st = getattr(L, fn)(h, p, elem_bytes_for(p), F.data_ptr(), m, n, lf, order, s_arr,
                            P.data_ptr(), ctypes.byref(lp), rd)
        _lib.check(st, fn)
    finally:
        if T is not None:
            L.fpm_set_pmbasis_threshold(h, 32)
    return P[:, :, : lp.value], [int(rd[i]) for i in range(m)]


def pmbasis_dense(F, order, s, p, T=None):
    """appint.pmbasis (appint.py:183-196) -> (P (m,m,deg+1), rdeg_s(P))."""
    return _basis("fpm_pmbasis", F, order, s, p, T)


def mbasis_dense(F, order, s, p):
    """appint.mbasis (appint.py:143-180) -> (P (m,m,deg+1), rdeg_s(P))."""
    return _basis("fpm_mbasis", F, order, s, p)


def intbasis_dense(E, alpha, s, p):
    """appint.pm_intbasis / m_intbasis (appint.py:208-319) on device data:
    E (order, m, n) point-major constant matrices, alpha (order,) host points.
    -> (P (m, m, deg+1), rdeg_s(P))."""
    import torch

    _check_tensor(E, p, "E")
    order, m, n = E.shape
    if len(alpha) != order:
        from .errors import LengthMismatch

        raise LengthMismatch("one point per constant matrix")
    s_arr = (ctypes.c_int64 * max(m, 1))(*[int(x) for x in s])
    # appint._check_points compares the integers as given (appint.py:203-205);
    # the C ABI does the same on uint64 values, so residues that repeat among
    # distinct integers (1 and 1 + p) are passed as distinct representatives
    if len(set(int(x) for x in alpha)) != len(alpha):
        from .errors import DuplicatePoints

        raise DuplicatePoints("interpolation points must be pairwise distinct")
    seen = {}
    reps = []
    for x in alpha:
        r = int(x) % p
        c = seen.get(r, 0)
        seen[r] = c + 1
        reps.append(r + c * p)
    a_arr = (ctypes.c_uint64 * max(order, 1))(*reps)
    P = torch.zeros((m, m, order + 1), dtype=E.dtype, device=E.device)
    lp = ctypes.c_int(0)
    rd = (ctypes.c_int64 * max(m, 1))()
    h = _lib.context(E.device.index)
    _lib.check(_lib.lib().fpm_pm_intbasis(h, p, elem_bytes_for(p), E.data_ptr(), m, n, order,
                                          a_arr, s_arr, P.data_ptr(), ctypes.byref(lp), rd),
               "fpm_pm_intbasis")
    return P[:, :, : lp.value], [int(rd[i]) for i in range(m)]


def eval_points_dense(P, pts, p):
    """appint.eval_polmat_points (appint.py:262-287): P (m, n, L) device ->
    (npts, m, n) values P(x) for x in pts."""
    import torch

    _check_tensor(P, p, "P")
    m, n, L = P.shape
    out = torch.empty((len(pts), m, n), dtype=P.dtype, device=P.device)
    if not pts:
        return out
    a_arr = (ctypes.c_uint64 * len(pts))(*[int(x) % p for x in pts])
    h = _lib.context(P.device.index)
    _lib.check(_lib.lib().fpm_polmat_eval_points(h, p, elem_bytes_for(p), P.data_ptr(), m, n, L,
                                                 a_arr, len(pts), out.data_ptr()),
               "fpm_polmat_eval_points")
    return out


def ntt_dense(x, p, log_len, inverse=False):
    """Batched modring.ntt_forward / ntt_inverse on a (batch, 2^log_len) tensor."""
    import torch

    h = _lib.context(x.device.index)
    L = _lib.lib()
    batch = x.shape[0]
    if p < (1 << 31):
        if x.dtype != torch.int32:
            raise ValueError("int32 storage expected for p < 2^31")
        out = torch.empty_like(x)
        _lib.check(L.fpm_ntt_u32(h, p, log_len, batch, x.data_ptr(), out.data_ptr(),
                                 1 if inverse else 0), "fpm_ntt_u32")
        return out
    x64 = x.to(torch.int64) if x.dtype != torch.int64 else x
    if x.dtype == torch.int32:
        x64 = x64 & 0xFFFFFFFF
    x64 = x64.contiguous()
    out = torch.empty_like(x64)
    _lib.check(L.fpm_ntt_u64(h, p, log_len, batch, x64.data_ptr(), out.data_ptr(),
                             1 if inverse else 0), "fpm_ntt_u64")
    return out.to(x.dtype) if x.dtype != torch.int64 else out


class DenseMultiplier:
    """Fixed left factor on the device with cached forward transforms
    (fpm_multiplier_*; reference polmat.Multiplier, polmat.py:550-610)."""

    def __init__(self, A, p, max_rhs_len):
        _check_tensor(A, p, "A")
        self.p = p
        self.m, self.k, self.la = A.shape
        self.max_rhs_len = int(max_rhs_len)
        self._h = _lib.context(A.device.index)
        self._mu = ctypes.c_void_p()
        _lib.check(_lib.lib().fpm_multiplier_create(self._h, p, elem_bytes_for(p), A.data_ptr(),
                                                     self.m, self.k, self.la, self.max_rhs_len,
                                                     ctypes.byref(self._mu)),
                   "fpm_multiplier_create")
        self.device = A.device
        self.dtype = A.dtype

    def apply(self, B, out=None):
        import torch

        _check_tensor(B, self.p, "B")
        k2, n, lb = B.shape
        if k2 != self.k:
            from .errors import DimMismatch

            raise DimMismatch(f"cannot multiply {self.m}x{self.k} by {k2}x{n}")
        lc = self.la + lb - 1 if self.la > 0 and lb > 0 else 0
        if out is None:
            out = torch.empty((self.m, n, lc), dtype=self.dtype, device=self.device)
        _lib.check(_lib.lib().fpm_multiplier_apply(self._mu, B.data_ptr(), n, lb, out.data_ptr()),
                   "fpm_multiplier_apply")
        return out

    def close(self):
        if self._mu:
            _lib.lib().fpm_multiplier_destroy(self._mu)
            self._mu = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- multi-prime pieces (parallel.pm_mul_prime_split) -------------

def product_primes(p, k, la, lb):
    """Word primes fpm_polmat_mul uses for A (.., k, la) * B (k, .., lb) mod p
    ([p] for a direct 31-bit NTT prime)."""
    buf = (ctypes.c_uint32 * 8)()
    cnt = ctypes.c_int(0)
    _lib.check(_lib.lib().fpm_product_primes(p, k, la, lb, buf, 8, ctypes.byref(cnt)),
               "fpm_product_primes")
    return [int(buf[i]) for i in range(cnt.value)]


def split_residues(X, p, primes):
    """X (device tensor of values mod p) -> (len(primes), *X.shape) int32
    residues X mod q (fpm_split_residues)."""
    import torch

    _check_tensor(X, p, "X")
    X = X.contiguous()
    out = torch.empty((len(primes),) + tuple(X.shape), dtype=torch.int32, device=X.device)
    qs = (ctypes.c_uint32 * len(primes))(*primes)
    h = _lib.context(X.device.index)
    _lib.check(_lib.lib().fpm_split_residues(h, elem_bytes_for(p), X.data_ptr(), X.numel(), qs,
                                             len(primes), out.data_ptr()), "fpm_split_residues")
    return out


def crt_combine(R, p, primes):
    """Residues R (len(primes), m, n, L) int32 on the device -> (m, n, L) mod p
    (fpm_crt_combine, the Garner step of the multi-prime product)."""
    import torch

    r, m, n, L = R.shape
    R = R.contiguous()
    out = torch.empty((m, n, L), dtype=torch_dtype(p), device=R.device)
    qs = (ctypes.c_uint32 * r)(*primes)
    h = _lib.context(R.device.index)
    _lib.check(_lib.lib().fpm_crt_combine(h, p, elem_bytes_for(p), qs, r, R.data_ptr(), m * n, L,
                                          out.data_ptr()), "fpm_crt_combine")
    return out
