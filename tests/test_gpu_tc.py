"""tcgen05 kind::i8 plumbing self-test (descriptors, TMEM, commit) vs torch."""
import ctypes

import pytest
import torch

from paper_1905_04356_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,K", [(256, 128), (128, 64), (16, 32), (256, 256)])
def test_tc_gemm_u8(N, K):
    L = _lib.lib()
    L.fpm_selftest_tc_gemm.restype = ctypes.c_int
    L.fpm_selftest_tc_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3
    _lib.context()
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
    L = _lib.lib()
    L.fpm_selftest_tc_pointwise.restype = ctypes.c_int
    L.fpm_selftest_tc_pointwise.argtypes = [ctypes.c_void_p, ctypes.c_uint32] + \
        [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4
    h = _lib.context()
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
