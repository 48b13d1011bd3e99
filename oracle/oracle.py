"""ctypes wrapper around the CPU oracle (oracle/fpm_oracle.c).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py -- never by the product
package ``paper_1905_04356_b200``.  Every function restates the reference
(`fpmat`, /root/reference/pkg/src/fpmat) on dense numpy arrays; see the
file:line anchors in fpm_oracle.c.

Dense layout: uint64 arrays of shape (rows, cols, len), coefficient t of entry
(i, j) at [i, j, t]; trailing zeros allowed (the reference trims, equality is
on trimmed lists, polmat.py:184-189).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfpm_oracle.so")
_lib = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_ip = ctypes.POINTER(ctypes.c_int)


def build(force=False):
    """Compile the oracle with the committed Makefile (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(os.path.join(_HERE, f))
                                          for f in ("fpm_oracle.c", "fpm_port.c"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.fpo_two_adicity.restype = ctypes.c_int
        L.fpo_two_adicity.argtypes = [ctypes.c_uint64]
        L.fpo_ntt_root.restype = ctypes.c_uint64
        L.fpo_ntt_root.argtypes = [ctypes.c_uint64]
        L.fpo_ntt.restype = ctypes.c_int
        L.fpo_ntt.argtypes = [ctypes.c_uint64, ctypes.c_int, _u64p, ctypes.c_int]
        L.fpo_pm_mul.restype = ctypes.c_int
        L.fpo_pm_mul.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, _u64p, ctypes.c_int, ctypes.c_int, _u64p]
        L.fpo_pm_middle.restype = ctypes.c_int
        L.fpo_pm_middle.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, _u64p, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_long, ctypes.c_int, _u64p]
        L.fpo_mbasis1_struct.restype = None
        L.fpo_mbasis1_struct.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_int, ctypes.c_int,
                                         _i64p, _ip, _u64p]
        L.fpo_mbasis.restype = ctypes.c_int
        L.fpo_mbasis.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_int, _i64p, _u64p, _ip, _i64p]
        L.fpo_pmbasis.restype = ctypes.c_int
        L.fpo_pmbasis.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, _i64p, ctypes.c_int, _u64p, _ip]
        _u32p = ctypes.POINTER(ctypes.c_uint32)
        L.fpo_port_mul31.restype = ctypes.c_int
        L.fpo_port_mul31.argtypes = [ctypes.c_uint32, _u32p, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, _u32p, ctypes.c_int, ctypes.c_int, _u32p,
                                     ctypes.c_int]
        L.fpo_set_threads.argtypes = [ctypes.c_int]
        L.fpo_get_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def set_threads(n):
    lib().fpo_set_threads(int(n))


def _p64(a):
    return a.ctypes.data_as(_u64p)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def two_adicity(p):
    return lib().fpo_two_adicity(p)


def ntt_root(p):
    return lib().fpo_ntt_root(p)


def ntt(p, v, inverse=False):
    """modring.ntt_forward / ntt_inverse (modring.py:272-286) on a length-2^k vector."""
    v = _c64(v).copy()
    n = v.shape[0]
    log_len = n.bit_length() - 1
    assert 1 << log_len == n
    rc = lib().fpo_ntt(p, log_len, _p64(v), 1 if inverse else 0)
    if rc:
        raise ValueError("log_len exceeds two-adicity")
    return v


def pm_mul(p, A, B):
    """Dense (m,k,la) x (k,n,lb) -> (m,n,la+lb-1); unique product (polmat.py:447)."""
    A = _c64(A)
    B = _c64(B)
    m, k, la = A.shape
    k2, n, lb = B.shape
    assert k == k2
    C = np.zeros((m, n, max(la + lb - 1, 0)), dtype=np.uint64)
    if la and lb:
        lib().fpo_pm_mul(p, _p64(A), m, k, la, _p64(B), n, lb, _p64(C))
    return C


def pm_middle(p, A, B, c, d):
    """Reference _pm_middle semantics, including its cyclic fold (polmat.py:484-536)."""
    A = _c64(A)
    B = _c64(B)
    m, k, la = A.shape
    _, n, lb = B.shape
    out = np.zeros((m, n, max(d, 0)), dtype=np.uint64)
    if d > 0 and la and lb:
        lib().fpo_pm_middle(p, _p64(A), m, k, la, _p64(B), n, lb, c, d, _p64(out))
    return out


def mbasis1_struct(p, R, s):
    """(is_pivot[m] bool, kern[m,m]) of appint._mbasis1_struct (appint.py:24-60)."""
    R = _c64(R)
    m, n = R.shape
    s = np.ascontiguousarray(s, dtype=np.int64)
    isp = np.zeros(m, dtype=np.int32)
    kern = np.zeros((m, m), dtype=np.uint64)
    lib().fpo_mbasis1_struct(p, _p64(R), m, n, s.ctypes.data_as(_i64p),
                             isp.ctypes.data_as(_ip), _p64(kern))
    return isp.astype(bool), kern


def mbasis(p, F, order, s):
    """appint.mbasis (appint.py:143-180) -> (P dense (m,m,L), final shift)."""
    F = _c64(F)
    m, n, lf = F.shape
    if lf == 0:
        F = np.zeros((m, n, 1), dtype=np.uint64)
        lf = 1
    s = np.ascontiguousarray(s, dtype=np.int64)
    P = np.zeros((m, m, order + 1), dtype=np.uint64)
    lp = ctypes.c_int(0)
    sh = np.zeros(m, dtype=np.int64)
    lib().fpo_mbasis(p, _p64(F), m, n, lf, order, s.ctypes.data_as(_i64p), _p64(P),
                     ctypes.byref(lp), sh.ctypes.data_as(_i64p))
    return P[:, :, : lp.value].copy(), sh


def pmbasis(p, F, order, s, T=32):
    """appint.pmbasis (appint.py:183-196) with base threshold T -> P dense (m,m,deg+1)."""
    F = _c64(F)
    m, n, lf = F.shape
    if lf == 0:
        F = np.zeros((m, n, 1), dtype=np.uint64)
        lf = 1
    s = np.ascontiguousarray(s, dtype=np.int64)
    P = np.zeros((m, m, order + 1), dtype=np.uint64)
    lp = ctypes.c_int(0)
    lib().fpo_pmbasis(p, _p64(F), m, n, lf, order, s.ctypes.data_as(_i64p), T, _p64(P),
                      ctypes.byref(lp))
    return P[:, :, : lp.value].copy()


# ---- PolMat-text helpers (polmat.py:617-623) used for golden checksums ------

def to_text(p, M):
    """polmat_to_text of a dense (m, n, L) array (entries trimmed)."""
    M = np.asarray(M)
    m, n = M.shape[0], M.shape[1]
    lines = [f"{p} {m} {n}"]
    for i in range(m):
        for j in range(n):
            e = M[i, j]
            nz = np.flatnonzero(e)
            L = int(nz[-1]) + 1 if nz.size else 0
            lines.append(" ".join(str(int(c)) for c in e[:L]))
    return "\n".join(lines) + "\n"


def sha16(p, M):
    import hashlib

    return hashlib.sha256(to_text(p, M).encode()).hexdigest()[:16]


def port_mul31(p, A, B, threads=None, out=None):
    """Multi-threaded CPU port of polmat._pm_mul_ntt for 31-bit NTT primes
    (oracle/fpm_port.c): the bench's CPU baseline / reference arm.
    A (m, k, la), B (k, n, lb) uint32 in [0, p) -> C (m, n, la+lb-1) uint32."""
    A = np.ascontiguousarray(A, dtype=np.uint32)
    B = np.ascontiguousarray(B, dtype=np.uint32)
    m, k, la = A.shape
    k2, n, lb = B.shape
    assert k == k2
    lc = la + lb - 1
    if out is None:
        out = np.empty((m, n, lc), dtype=np.uint32)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    rc = lib().fpo_port_mul31(p, A.ctypes.data_as(u32p), m, k, la, B.ctypes.data_as(u32p), n,
                              lb, out.ctypes.data_as(u32p), int(threads or os.cpu_count() or 1))
    if rc != 0:
        raise ValueError(f"fpo_port_mul31: status {rc} (needs a 31-bit NTT prime)")
    return out
