"""Transforms and products beyond one CTA (N > 2^15): the multi-pass NTT of
csrc/ntt_big.cu and the generic u64 transform, against the CPU oracle and
the reference's own outputs.  The reference accepts every length up to
2^two_adicity (polmat.py:290-296, modring.py:212-250); so must the GPU."""
import hashlib

import numpy as np
import pytest

import paper_1905_04356_b200 as F
from paper_1905_04356_b200 import dense
from golden_util import big_goldens, rows_from_dense
from oracle import oracle as O

pytestmark = pytest.mark.gpu

P31 = 2013265921
P60 = (1 << 60) - 93
P60NTT = 1152921493869428737  # 60-bit, two-adicity 31


def _rand(p, shape, seed):
    return np.random.default_rng(seed).integers(0, p, size=shape, dtype=np.uint64)


@pytest.mark.parametrize("p,lg", [(P31, 16), (P31, 17), (P31, 20), (1811939329, 18),
                                  (1107296257, 21), (786433, 18), (P60NTT, 16),
                                  (P31, 3), (P60NTT, 4)])
def test_long_ntt_api_vs_oracle(p, lg):
    """Natural-order forward and inverse (modring.ntt_forward / ntt_inverse)
    at lengths past the single-CTA limit, u32 and u64 storage."""
    x = _rand(p, (2, 1 << lg), lg)
    x[1, :] = p - 1
    t = dense.to_device(x, p)
    y = dense.ntt_dense(t, p, lg)
    got = dense.to_numpy(y, p).astype(np.uint64)
    for r in range(2):
        assert np.array_equal(got[r], O.ntt(p, x[r])), (p, lg, r)
    z = dense.to_numpy(dense.ntt_dense(y, p, lg, inverse=True), p).astype(np.uint64)
    assert np.array_equal(z, x)
    inv = dense.to_numpy(dense.ntt_dense(t, p, lg, inverse=True), p).astype(np.uint64)
    assert np.array_equal(inv[0], O.ntt(p, x[0], inverse=True))


def test_ntt_full_two_adicity_p31():
    """N = 2^27 = 2^two_adicity(p31): the longest transform the reference's
    NttPlan admits; round trip plus a DC / delta check."""
    lg = 27
    n = 1 << lg
    x = np.zeros((1, n), dtype=np.uint64)
    x[0, 0] = 5
    x[0, 1] = 7
    y = dense.to_numpy(dense.ntt_dense(dense.to_device(x, P31), P31, lg), P31).astype(np.uint64)
    # F(w^j) = 5 + 7 w^j: j = 0 gives 12, and j = N/2 (w^(N/2) = -1) gives -2
    assert y[0, 0] == 12 and y[0, n // 2] == (5 - 7) % P31
    plan = F.NttPlan(F.field_new(P31), lg)
    assert y[0, 1] == (5 + 7 * plan.omega) % P31
    back = dense.ntt_dense(dense.to_device(y, P31), P31, lg, inverse=True)
    assert np.array_equal(dense.to_numpy(back, P31).astype(np.uint64), x)


@pytest.mark.parametrize("p,m,k,n,la,lb", [
    (P31, 2, 2, 2, 40000, 40000),        # N = 2^17 (two passes)
    (P31, 1, 3, 2, 1 << 19, 1 << 19),    # N = 2^20
    (P31, 3, 1, 1, 600000, 70000),       # N = 2^20, ragged lengths
    (P31, 1, 1, 1, 5000000, 3000000),    # N = 2^23 (three passes)
    (P31, 2, 2, 1, 3000, 70000),         # N = 2^17, one short operand
    (P60, 2, 2, 2, 17000, 17000),        # multi-prime (5 CRT primes) at N = 2^16
    (786433, 2, 3, 2, 40000, 30000),     # 20-bit prime, two-adicity 18: direct at 2^17
])
def test_long_products_vs_oracle(p, m, k, n, la, lb):
    A = _rand(p, (m, k, la), la)
    B = _rand(p, (k, n, lb), lb + 1)
    A[0, 0, :100] = p - 1
    C = dense.to_numpy(dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p), p)
    assert np.array_equal(C.astype(np.uint64), O.pm_mul(p, A, B))


@pytest.mark.parametrize("c,d,la,lb", [(40000, 40000, 40001, 80000), (65536, 30000, 60000, 95536),
                                       (120001, 20000, 50000, 140000)])  # last: B folded mod x^N
def test_long_middle_products_vs_oracle(c, d, la, lb):
    """_pm_middle (reference semantics, cyclic fold) and the true slice at
    N = 2^17."""
    p = P31
    A = _rand(p, (2, 2, la), c)
    B = _rand(p, (2, 1, lb), d)
    Ad, Bd = dense.to_device(A, p), dense.to_device(B, p)
    R = dense.to_numpy(dense.pm_middle_dense(Ad, Bd, c, d, p), p).astype(np.uint64)
    assert np.array_equal(R, O.pm_middle(p, A, B, c, d))
    full = O.pm_mul(p, A, B)
    Rx = dense.to_numpy(dense.pm_middle_dense(Ad, Bd, c, d, p, exact=True), p).astype(np.uint64)
    want = np.zeros_like(Rx)
    hi = min(c + d, full.shape[2])
    want[:, :, : hi - c] = full[:, :, c:hi]
    assert np.array_equal(Rx, want)


def test_pmbasis_order_32768_vs_oracle():
    """PM-Basis 4x2 at sigma = 32768 (the paper's PM-Basis row):
    the top middle product needs N = 2^16."""
    p = P31
    Fm = _rand(p, (4, 2, 32768), 32768)
    P, _ = dense.pmbasis_dense(dense.to_device(Fm, p), 32768, [0] * 4, p)
    got = dense.to_numpy(P, p).astype(np.uint64)
    O.set_threads(16)
    want = O.pmbasis(p, Fm, 32768, [0] * 4)
    assert got.shape == want.shape and np.array_equal(got, want)


@pytest.mark.parametrize("key,args", [
    ("mul_s21_p2013265921_2x2x2_d39999", (21, P31, 2, 2, 2, 39999)),
    ("mul_s22_p1152921504606846883_2x2x2_d16999", (22, P60, 2, 2, 2, 16999)),
    ("mul_s23_p2013265921_8x8x8_d131071", (23, P31, 8, 8, 8, 131071)),
])
def test_long_products_reference_checksums(key, args):
    """sha256 of polmat_to_text of the unmodified reference's own product
    (tests/golden/make_golden_big.py), N = 2^17, 2^16 (5 primes), 2^18 (the
    paper's m = 8, d = 131072 row)."""
    import random

    gold = big_goldens().get(key)
    assert gold is not None, f"golden {key} missing"
    seed, p, m, k, n, deg = args
    rng = random.Random(seed)
    A = np.array([[[rng.randrange(p) for _ in range(deg + 1)] for _ in range(k)]
                  for _ in range(m)], dtype=np.uint64)
    B = np.array([[[rng.randrange(p) for _ in range(deg + 1)] for _ in range(n)]
                  for _ in range(k)], dtype=np.uint64)
    C = dense.to_numpy(dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p), p)
    txt = F.polmat_to_text(F.polmat.from_dense(F.field_new(p), C.astype(np.uint64), ncols=n))
    assert hashlib.sha256(txt.encode()).hexdigest()[:16] == gold["sha16"]
