"""Pointwise products for 128 < m <= 256 (csrc/tc_pair.cu: both M tiles of a
point share one built B tile).  Bit-exact against the oracle (restatement of
polmat._pm_mul_ntt, /root/reference/pkg/src/fpmat/polmat.py:290-308) on
sampled entries and against tc_grouped (option tc_no_pair) on every entry."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_04356_b200 import _lib, dense

pytestmark = pytest.mark.gpu

P31 = 2013265921
P60 = 1152921504606846883


def _mul(p, A, B):
    C = dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p)
    return dense.to_numpy(C, p).astype(np.uint64)


@pytest.mark.parametrize("p,m,k,n,deg,seed", [
    (P31, 256, 256, 256, 255, 1),    # cfg5 shape class (N = 512)
    (P31, 129, 36, 40, 700, 2),      # one row into the second M tile, ragged column block
    (P31, 200, 516, 100, 60, 3),     # K chunks with a partial last chunk (k % 32 = 4)
    (P31, 256, 8, 4, 2047, 4),       # N = 4096: the tensor-core forward NTT feeds it
    (P60, 136, 24, 36, 40, 5),       # 60-bit prime: 4 CRT primes, blockIdx.z = prime
])
def test_tc_pair_vs_oracle_and_grouped(p, m, k, n, deg, seed):
    rng = np.random.default_rng(seed)
    A = rng.integers(0, p, size=(m, k, deg + 1), dtype=np.uint64)
    B = rng.integers(0, p, size=(k, n, deg + 1), dtype=np.uint64)
    got = _mul(p, A, B)
    for (i, j) in [(0, 0), (m - 1, n - 1), (128, n // 2), (m // 2, 1)]:
        ref = O.pm_mul(p, A[i:i + 1], B[:, j:j + 1])
        assert np.array_equal(got[i:i + 1, j:j + 1], ref), (i, j)
    _lib.set_option("tc_no_pair", 1)
    try:
        ref_all = _mul(p, A, B)
    finally:
        _lib.set_option("tc_no_pair", 0)
    assert np.array_equal(got, ref_all)


def test_tc_pair_extreme_operands():
    """all coefficients p - 1 and k = 8192 (the largest limb sums the s32
    accumulators take)"""
    p = P31
    A = np.full((130, 8192, 2), p - 1, dtype=np.uint64)
    B = np.full((8192, 4, 2), p - 1, dtype=np.uint64)
    got = _mul(p, A, B)
    ref = O.pm_mul(p, A[:1], B[:, :1])
    assert np.all(got == ref[0, 0][None, None, :])
