"""tcgen05 kind::i8 plumbing self-test (descriptors, TMEM, commit) vs torch."""
import ctypes

import pytest
import torch

from paper_1905_04356_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,K", [(256, 128), (128, 64), (16, 32), (256, 256)])
def test_tc_gemm_u8(N, K):
    L = _lib.selftest_lib()
    L.fpm_selftest_tc_gemm.restype = ctypes.c_int
    L.fpm_selftest_tc_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3
    _lib.selftest_context()
    g = torch.Generator().manual_seed(N + K)
    A = torch.randint(0, 256, (128, K), generator=g, dtype=torch.int32)
    B = torch.randint(0, 256, (N, K), generator=g, dtype=torch.int32)
    Ad = A.to(torch.uint8).cuda()
    Bd = B.to(torch.uint8).cuda()
    D = torch.zeros((128, N), dtype=torch.int32, device="cuda")
    _lib.check(L.fpm_selftest_tc_gemm(Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), 128, N, K),
               "selftest")
    ref = A.to(torch.int64) @ B.to(torch.int64).T
    assert torch.equal(D.cpu().to(torch.int64), ref)


def _matmul_mod_np(A, B, p):
    import numpy as np

    lo = B & np.uint64(0xFFFF)
    hi = B >> np.uint64(16)
    return ((A @ lo) % np.uint64(p) + ((A @ hi) % np.uint64(p)) * np.uint64(1 << 16)) % np.uint64(p)


@pytest.mark.parametrize("m,k,n", [(256, 256, 256), (128, 64, 64), (200, 100, 72), (64, 512, 32)])
def test_tc_pointwise_exact(m, k, n):
    import numpy as np

    p = 2013265921
    L = _lib.selftest_lib()
    L.fpm_selftest_tc_pointwise.restype = ctypes.c_int
    L.fpm_selftest_tc_pointwise.argtypes = [ctypes.c_void_p, ctypes.c_uint32] + \
        [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4
    h = _lib.selftest_context()
    npts = 3
    rng = np.random.default_rng(m + k + n)
    A = rng.integers(0, p, size=(npts, m, k), dtype=np.uint64)
    B = rng.integers(0, p, size=(npts, k, n), dtype=np.uint64)
    A[0, 0, :] = p - 1  # extreme values
    B[0, :, 0] = p - 1
    Ad = torch.from_numpy(A.astype(np.uint32).view(np.int32)).cuda()
    Bd = torch.from_numpy(B.astype(np.uint32).view(np.int32)).cuda()
    Cd = torch.zeros((npts, m, n), dtype=torch.int32, device="cuda")
    _lib.check(L.fpm_selftest_tc_pointwise(h, p, Ad.data_ptr(), Bd.data_ptr(), Cd.data_ptr(),
                                           m, k, n, npts), "tc_pointwise")
    C = Cd.cpu().numpy().view(np.uint32).astype(np.uint64)
    for t in range(npts):
        assert np.array_equal(C[t], _matmul_mod_np(A[t], B[t], p)), t


GROUPED_SHAPES = [(32, 32, 32, 13), (16, 16, 16, 40), (64, 64, 32, 9), (128, 64, 64, 3),
                  (20, 36, 44, 11), (100, 100, 72, 3), (8, 4, 4, 33), (64, 256, 96, 5),
                  (256, 256, 64, 2), (200, 68, 36, 3), (129, 32, 8, 2)]


@pytest.mark.parametrize("m,k,n,npts", GROUPED_SHAPES)
def test_tc_grouped_exact(m, k, n, npts):
    """Grouped kernel (G = 128/mp points per UMMA tile): ragged point counts,
    m not a power of two, k/n tails, two primes (CRT layout), extreme values."""
    import numpy as np

    primes = [2013265921, 2130706433, 1107296257]
    L = _lib.selftest_lib()
    L.fpm_selftest_tc_grouped.restype = ctypes.c_int
    L.fpm_selftest_tc_grouped.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int] + \
        [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4
    h = _lib.selftest_context()
    rng = np.random.default_rng(7 * m + 3 * k + n + npts)
    A = np.stack([rng.integers(0, q, size=(npts, m, k), dtype=np.uint64) for q in primes])
    B = np.stack([rng.integers(0, q, size=(npts, k, n), dtype=np.uint64) for q in primes])
    for z, q in enumerate(primes):
        A[z, 0, 0, :] = q - 1
        B[z, 0, :, 0] = q - 1
        if npts > 1:  # a point of all p-1: largest limb sums
            A[z, 1] = q - 1
            B[z, 1] = q - 1
    Ad = torch.from_numpy(A.astype(np.uint32).view(np.int32)).cuda()
    Bd = torch.from_numpy(B.astype(np.uint32).view(np.int32)).cuda()
    Cd = torch.full((len(primes), npts, m, n), -1, dtype=torch.int32, device="cuda")
    pr = (ctypes.c_uint32 * len(primes))(*primes)
    _lib.check(L.fpm_selftest_tc_grouped(h, pr, len(primes), Ad.data_ptr(), Bd.data_ptr(), Cd.data_ptr(),
                                         m, k, n, npts), "tc_grouped")
    C = Cd.cpu().numpy().view(np.uint32).astype(np.uint64)
    for z, q in enumerate(primes):
        for t in range(npts):
            assert np.array_equal(C[z, t], _matmul_mod_np(A[z, t], B[z, t], q)), (z, t)


def _to_pq(X):
    """(z, t, r, c) point-major -> eval layout (z, t/4, r, c, 4)."""
    z, t, r, c = X.shape
    return X.reshape(z, t // 4, 4, r, c).transpose(0, 1, 3, 4, 2).copy()


def _from_pq(Y):
    z, tq, r, c, four = Y.shape
    return Y.transpose(0, 1, 4, 2, 3).reshape(z, tq * 4, r, c)


PQ_SHAPES = [(32, 32, 32, 16), (16, 16, 16, 24), (17, 5, 9, 8), (1, 1, 1, 8), (32, 64, 32, 8),
             (24, 100, 40, 16), (8, 4, 4, 32), (32, 33, 70, 8)]


@pytest.mark.parametrize("m,k,n,npts", PQ_SHAPES)
def test_tc_pq_exact(m, k, n, npts):
    """Point-quad kernel: k / n tails, m not a power of two, several n-blocks,
    three primes, a point of all p-1 (largest limb sums)."""
    import numpy as np

    primes = [2013265921, 2130706433, 1107296257]
    kernel = "fpm_selftest_tc_pq"
    L = _lib.selftest_lib()
    fn = getattr(L, kernel)
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int] + \
        [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4
    h = _lib.selftest_context()
    rng = np.random.default_rng(11 * m + 5 * k + n + npts)
    A = np.stack([rng.integers(0, q, size=(npts, m, k), dtype=np.uint64) for q in primes])
    B = np.stack([rng.integers(0, q, size=(npts, k, n), dtype=np.uint64) for q in primes])
    for z, q in enumerate(primes):
        A[z, 1] = q - 1
        B[z, 1] = q - 1
    Ad = torch.from_numpy(_to_pq(A).astype(np.uint32).view(np.int32)).cuda()
    Bd = torch.from_numpy(_to_pq(B).astype(np.uint32).view(np.int32)).cuda()
    Cd = torch.full((len(primes), npts // 4, m, n, 4), -1, dtype=torch.int32, device="cuda")
    pr = (ctypes.c_uint32 * len(primes))(*primes)
    _lib.check(fn(h, pr, len(primes), Ad.data_ptr(), Bd.data_ptr(), Cd.data_ptr(), m, k, n,
                  npts), kernel)
    C = _from_pq(Cd.cpu().numpy().view(np.uint32).astype(np.uint64))
    for z, q in enumerate(primes):
        for t in range(npts):
            assert np.array_equal(C[z, t], _matmul_mod_np(A[z, t], B[z, t], q)), (z, t)
