"""Tensor-core NTT path (csrc/ntt_mma64.cu, and ntt_mma.cu behind option ntt_mma_r16): products whose transforms have
N = 4096 points in the point-major layout (m > 32, 2^30 < p < 2^31) run all
three transforms on tcgen05.  Bit-exact against the oracle (restatement of
polmat._pm_mul_ntt, /root/reference/pkg/src/fpmat/polmat.py:290-308) and
against the DIF-ordered Shoup kernels (option ntt_no_mma)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_04356_b200 import _lib, dense

pytestmark = pytest.mark.gpu

P31 = 2013265921      # 15 * 2^27 + 1 (cfg5)
P31B = 2113929217     # 63 * 2^25 + 1


def _rand(p, shape, seed, extreme=False):
    rng = np.random.default_rng(seed)
    if extreme:
        return np.full(shape, p - 1, dtype=np.uint64)
    return rng.integers(0, p, size=shape, dtype=np.uint64)


def _mul(p, A, B):
    C = dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p)
    return dense.to_numpy(C, p).astype(np.uint64)


@pytest.mark.parametrize("p,m,k,n,la,lb,seed", [
    (P31, 64, 64, 64, 2048, 2048, 1),      # cfg5 shape class, P1 with K' = 32
    (P31, 40, 36, 48, 2048, 2000, 2),      # ragged entry counts (tiles of 8)
    (P31, 33, 35, 37, 1500, 2049, 3),      # la + lb - 1 > 2048: N = 4096, P1 K' = 64
    (P31, 48, 64, 40, 3000, 1097, 4),      # A longer than N/2
    (P31B, 64, 32, 64, 2048, 2048, 5),     # another NTT prime
])
def test_mma_ntt_products_vs_oracle(p, m, k, n, la, lb, seed):
    A = _rand(p, (m, k, la), seed)
    B = _rand(p, (k, n, lb), seed + 100)
    got = _mul(p, A, B)
    # full oracle on a few rows / columns (the oracle is O(m k n N log N))
    for (i, j) in [(0, 0), (m - 1, n - 1), (m // 2, 3)]:
        ref = O.pm_mul(p, A[i:i + 1], B[:, j:j + 1])
        assert np.array_equal(got[i:i + 1, j:j + 1], ref), (i, j)


def test_mma_ntt_extreme_operands():
    """all coefficients p - 1: largest limb sums in every pass"""
    p = P31
    A = _rand(p, (64, 64, 2048), 0, extreme=True)
    B = _rand(p, (64, 64, 2048), 0, extreme=True)
    got = _mul(p, A, B)
    ref = O.pm_mul(p, A[:1], B[:, :1])
    assert np.array_equal(got[:1, :1], ref)
    assert np.all(got == got[0, 0][None, None, :])


def test_mma_ntt_matches_dif_kernels():
    p = P31
    A = _rand(p, (64, 48, 2048), 7)
    B = _rand(p, (48, 72, 1800), 8)
    got = _mul(p, A, B)
    _lib.set_option("ntt_no_mma", 1)
    try:
        ref = _mul(p, A, B)
    finally:
        _lib.set_option("ntt_no_mma", 0)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("la,lb", [(2048, 2048), (3000, 1097)])
def test_mma_ntt_radix16_option_matches(la, lb):
    """the three-pass radix-16 kernel (option ntt_mma_r16) and the default
    two-pass radix-64 kernel produce the same product"""
    p = P31
    A = _rand(p, (40, 24, la), 11)
    B = _rand(p, (24, 48, lb), 12)
    got = _mul(p, A, B)
    _lib.set_option("ntt_mma_r16", 1)
    try:
        ref = _mul(p, A, B)
    finally:
        _lib.set_option("ntt_mma_r16", 0)
    assert np.array_equal(got, ref)
    assert np.array_equal(got[:1, :1], O.pm_mul(p, A[:1], B[:, :1]))


def test_mma_ntt_extreme_operands_long():
    """all coefficients p - 1 with more than 2048 coefficients: the first pass
    runs with K' = 256 (largest byte-plane sums D_r = 256 * 255 * byte)"""
    p = P31
    A = _rand(p, (40, 16, 3000), 0, extreme=True)
    B = _rand(p, (16, 40, 1097), 0, extreme=True)
    got = _mul(p, A, B)
    assert np.array_equal(got[:1, :1], O.pm_mul(p, A[:1], B[:, :1]))
    assert np.all(got == got[0, 0][None, None, :])
    # 0x77FFFFFF < p: three 0xFF bytes in every input word
    A[:] = 0x77FFFFFF
    B[:] = 0x77FFFFFF
    got = _mul(p, A, B)
    assert np.array_equal(got[:1, :1], O.pm_mul(p, A[:1], B[:, :1]))
    assert np.all(got == got[0, 0][None, None, :])
