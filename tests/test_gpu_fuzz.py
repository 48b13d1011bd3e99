"""Seeded differential sweep: random shapes, lengths, shifts and primes
through the C ABI (products, middle products in both semantics, M-Basis,
PM-Basis) against the CPU oracle, bit-exact.  The fixed cases elsewhere pin
the kernel families; this sweep walks the dispatch boundaries between them
(ragged tiles, lengths around the powers of two, tiny and non-NTT primes)."""
import numpy as np
import pytest

from paper_1905_04356_b200 import dense
from oracle import oracle as O

pytestmark = pytest.mark.gpu

# 31-bit NTT primes, a 31-bit prime without a usable root, small primes, a
# 20-bit NTT prime, 40 / 60 / 62-bit primes (multi-prime route)
PRIMES = [2013265921, 469762049, 2147483629, 2147483647, 5, 3, 97, 786433,
          (1 << 40) - 87, (1 << 60) - 93, 1152921493869428737, (1 << 62) - 57]


def _len(rng, hi):
    """Log-uniform length in [1, hi], often right at a power of two +- 1."""
    if rng.random() < 0.3:
        e = int(rng.integers(0, int(np.log2(hi)) + 1))
        return int(min(hi, max(1, (1 << e) + int(rng.integers(-1, 2)))))
    return int(max(1, min(hi, round(float(np.exp(rng.uniform(0, np.log(hi))))))))


def _mat(rng, p, shape, sparse):
    M = rng.integers(0, p, size=shape, dtype=np.uint64)
    if sparse == 1:      # ragged degrees, some zero entries
        for idx in np.ndindex(shape[:2]):
            d = int(rng.integers(0, shape[2] + 1))
            M[idx][d:] = 0
    elif sparse == 2:    # extreme operands
        M[:] = p - 1
    return M


@pytest.mark.parametrize("seed", range(60))
def test_products_sweep(seed):
    rng = np.random.default_rng(1000 + seed)
    p = PRIMES[seed % len(PRIMES)]
    big = seed % 5 == 0
    m, k, n = (int(rng.integers(1, 140 if big else 40)) for _ in range(3))
    cap = max(2, min(6000, int(3e6 / (m * k * n))))   # keeps the oracle in seconds
    la, lb = _len(rng, cap), _len(rng, cap)
    A = _mat(rng, p, (m, k, la), int(rng.integers(0, 3)))
    B = _mat(rng, p, (k, n, lb), int(rng.integers(0, 3)))
    C = dense.to_numpy(dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p), p)
    assert np.array_equal(C.astype(np.uint64), O.pm_mul(p, A, B)), (p, m, k, n, la, lb)


@pytest.mark.parametrize("seed", range(24))
def test_tensor_core_tiles_sweep(seed):
    """Shapes around the tile edges of the int8 tensor-core pointwise kernels
    (m, n around 32 / 64 / 128 / 256, k with and without the multiple-of-4
    contraction), lengths on both sides of the 2048-coefficient tensor-core
    NTT; checked against the multi-threaded C port (pinned to the oracle in
    tests/test_oracle_golden.py)."""
    rng = np.random.default_rng(4000 + seed)
    p = [2013265921, 469762049][seed % 2]
    edge = [31, 32, 33, 63, 64, 65, 127, 128, 129, 136, 200, 255, 256, 257]
    m, n = (int(edge[int(rng.integers(0, len(edge)))]) for _ in range(2))
    k = int(rng.integers(1, 70)) * (4 if seed % 3 else 1)
    hi = [40, 300, 2048][seed % 3]
    la, lb = _len(rng, hi), _len(rng, hi)
    A = _mat(rng, p, (m, k, la), int(rng.integers(0, 3)))
    B = _mat(rng, p, (k, n, lb), int(rng.integers(0, 3)))
    C = dense.to_numpy(dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p), p)
    want = O.port_mul31(p, A.astype(np.uint32), B.astype(np.uint32))
    assert np.array_equal(C.astype(np.uint32), want), (p, m, k, n, la, lb)


def test_modulus_two_is_out_of_range():
    """field_new rejects p = 2 (modring.py:157-158); so does the C ABI."""
    from paper_1905_04356_b200.errors import OutOfRange

    A = np.ones((1, 1, 2), dtype=np.uint32)
    with pytest.raises(OutOfRange):
        dense.pm_mul_dense(dense.to_device(A, 3), dense.to_device(A, 3), 2)


@pytest.mark.parametrize("seed", range(40))
def test_middle_products_sweep(seed):
    rng = np.random.default_rng(2000 + seed)
    p = PRIMES[seed % 4] if seed % 3 else PRIMES[seed % len(PRIMES)]
    m, k, n = (int(rng.integers(1, 20)) for _ in range(3))
    la, lb = _len(rng, 1500), _len(rng, 3000)
    c = int(rng.integers(0, la + lb + 3))
    d = _len(rng, 2000)
    A = _mat(rng, p, (m, k, la), int(rng.integers(0, 2)))
    B = _mat(rng, p, (k, n, lb), int(rng.integers(0, 2)))
    Ad, Bd = dense.to_device(A, p), dense.to_device(B, p)
    R = dense.to_numpy(dense.pm_middle_dense(Ad, Bd, c, d, p), p).astype(np.uint64)
    assert np.array_equal(R, O.pm_middle(p, A, B, c, d)), (p, m, k, n, la, lb, c, d)
    Rx = dense.to_numpy(dense.pm_middle_dense(Ad, Bd, c, d, p, exact=True), p).astype(np.uint64)
    full = O.pm_mul(p, A, B)
    want = np.zeros((m, n, d), dtype=np.uint64)
    hi = min(c + d, full.shape[2])
    if hi > c:
        want[:, :, : hi - c] = full[:, :, c:hi]
    assert np.array_equal(Rx, want), (p, m, k, n, la, lb, c, d)


@pytest.mark.parametrize("seed", range(30))
def test_bases_sweep(seed):
    rng = np.random.default_rng(3000 + seed)
    p = [2013265921, 469762049, 97, 2147483629, (1 << 60) - 93][seed % 5]
    m = int(rng.integers(1, 24))
    n = int(rng.integers(1, m + 1)) if seed % 4 else int(rng.integers(1, 30))
    order = _len(rng, 300)
    lf = order if seed % 3 else _len(rng, order)
    F = _mat(rng, p, (m, n, lf), int(rng.integers(0, 2)))
    if seed % 6 == 1:
        F[:, :, 0] = 0                     # singular constant term: degenerate steps
    if seed % 6 == 2 and m > 1:
        F[1] = F[0]                        # dependent rows
    s = [int(x) for x in rng.integers(-5, 6, size=m)] if seed % 2 else [0] * m
    Fd = dense.to_device(F, p)
    P, rd = dense.pmbasis_dense(Fd, order, s, p)
    want = O.pmbasis(p, F, order, s)
    got = dense.to_numpy(P, p).astype(np.uint64)
    assert got.shape == want.shape and np.array_equal(got, want), (p, m, n, order, lf, s)
    if order <= 64:
        Pm, rdm = dense.mbasis_dense(Fd, order, s, p)
        wm, sh = O.mbasis(p, F, order, s)
        gm = dense.to_numpy(Pm, p).astype(np.uint64)
        assert gm.shape == wm.shape and np.array_equal(gm, wm), (p, m, n, order, lf, s)
        assert rdm == [int(x) for x in sh], (p, m, n, order, lf, s)
