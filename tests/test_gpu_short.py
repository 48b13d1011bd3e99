"""Short operands (<= 17 coefficients: the PM-Basis nodes of order 16 and
32) through the product and true-slice middle-product entry points, against
the oracle, bit-exact: tiny primes, a 31-bit prime with no NTT root (multi-
prime route), bases allocated at twice their degree, ragged shapes."""
import numpy as np
import pytest

from paper_1905_04356_b200 import dense
from oracle import oracle as O

pytestmark = pytest.mark.gpu

P31 = 2013265921


def _rand(p, shape, seed, deg=None, extreme=False):
    rng = np.random.default_rng(seed)
    M = rng.integers(0, p, size=shape, dtype=np.uint64)
    if extreme:
        M[:] = p - 1
    if deg is not None:
        M[:, :, deg + 1:] = 0  # allocated at a bound, like the PM-Basis bases
    return M


@pytest.mark.parametrize("p", [P31, 469762049, 3, 2147483629])  # the last: not an NTT prime
@pytest.mark.parametrize("m,k,n,la,lb,dega", [(64, 64, 64, 9, 9, 4), (64, 64, 64, 17, 17, 8),
                                              (64, 64, 64, 17, 17, None), (3, 5, 37, 1, 7, None),
                                              (1, 1, 1, 17, 17, None), (8, 200, 33, 6, 12, None),
                                              (5, 7, 70, 17, 3, None)])
def test_short_products(p, m, k, n, la, lb, dega):
    A = _rand(p, (m, k, la), m + la, deg=dega)
    B = _rand(p, (k, n, lb), k + lb, deg=dega)
    Ad, Bd = dense.to_device(A, p), dense.to_device(B, p)
    got = dense.to_numpy(dense.pm_mul_dense(Ad, Bd, p), p)
    assert np.array_equal(got.astype(np.uint64), O.pm_mul(p, A, B))


def test_short_product_extreme_operands():
    p = 2147483647  # 2^31 - 1: the largest sums
    A = _rand(p, (4, 4096, 17), 1, extreme=True)
    B = _rand(p, (4096, 3, 17), 2, extreme=True)
    C = dense.to_numpy(dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p), p)
    assert np.array_equal(C.astype(np.uint64), O.pm_mul(p, A, B))


@pytest.mark.parametrize("m,k,n,la,lb,c,d,dega", [(64, 64, 32, 9, 16, 8, 8, 4),
                                                  (64, 64, 32, 17, 32, 16, 16, 8),
                                                  (64, 64, 32, 17, 32, 16, 16, None),
                                                  (5, 3, 40, 7, 50, 20, 33, None),
                                                  (2, 9, 2, 12, 9, 15, 10, None),
                                                  (4, 4, 4, 3, 30, 0, 5, None)])
def test_short_true_slices(m, k, n, la, lb, c, d, dega):
    p = P31
    A = _rand(p, (m, k, la), c + la, deg=dega)
    B = _rand(p, (k, n, lb), d + lb)
    Ad, Bd = dense.to_device(A, p), dense.to_device(B, p)
    got = dense.to_numpy(dense.pm_middle_dense(Ad, Bd, c, d, p, exact=True), p)
    full = O.pm_mul(p, A, B)
    want = np.zeros((m, n, d), dtype=np.uint64)
    hi = min(c + d, full.shape[2])
    if hi > c:
        want[:, :, : hi - c] = full[:, :, c:hi]
    assert np.array_equal(got.astype(np.uint64), want)


@pytest.mark.parametrize("m,n,order", [(16, 8, 128), (6, 5, 64)])
def test_pmbasis_small_nodes_vs_oracle(m, n, order):
    """PM-Basis whose tree is mostly nodes of order 16 and 32."""
    p = P31
    F = _rand(p, (m, n, order), 9)
    got = dense.to_numpy(dense.pmbasis_dense(dense.to_device(F, p), order, [0] * m, p)[0], p)
    assert np.array_equal(got.astype(np.uint64), O.pmbasis(p, F, order, [0] * m))
