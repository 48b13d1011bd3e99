"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
fixtures and the CPU oracle.  Bit-exact equality everywhere (integer work)."""
import random

import numpy as np
import pytest

import paper_1905_04356_b200 as F
from paper_1905_04356_b200 import dense
from golden_util import big_goldens, dense as to_dense_rows, random_polmat_dense, rows_from_dense, small
from oracle import oracle as O

pytestmark = pytest.mark.gpu

P31 = 2013265921
P60 = (1 << 60) - 93


def _pm(p, rows, m, n):
    ctx = F.field_new(p)
    return F.PolMat(ctx, [[list(e) for e in r] for r in rows], ncols=n)


def test_ntt_golden():
    for rec in small()["ntt"]:
        p = rec["p"]
        ctx = F.field_new(p)
        plan = F.NttPlan(ctx, len(rec["v"]).bit_length() - 1)
        assert F.ntt_forward(plan, rec["v"]) == rec["fwd"], (p, len(rec["v"]))
        assert F.ntt_inverse(plan, rec["v"]) == rec["inv"], (p, len(rec["v"]))


def test_ntt_batched_roundtrip_all_sizes():
    rng = np.random.default_rng(1)
    for lg in range(5, 16):
        x = rng.integers(0, P31, size=(3, 1 << lg), dtype=np.uint64)
        t = dense.to_device(x, P31)
        y = dense.ntt_dense(t, P31, lg)
        z = dense.ntt_dense(y, P31, lg, inverse=True)
        assert np.array_equal(dense.to_numpy(z, P31), x.astype(np.uint32)), lg
        # one row against the oracle's restatement of modring.ntt_forward
        assert np.array_equal(dense.to_numpy(y, P31)[1].astype(np.uint64), O.ntt(P31, x[1])), lg


def test_pm_mul_golden_all_primes():
    for rec in small()["mul"]:
        A = _pm(rec["p"], rec["A"], rec["m"], rec["k"])
        B = _pm(rec["p"], rec["B"], rec["k"], rec["n"])
        C = F.pm_mul(A, B)
        assert C.rows == rec["C"], (rec["p"], rec["m"], rec["k"], rec["n"])
        for st in rec["strategies"]:
            assert F.pm_mul(A, B, strategy=st).rows == rec["C"]


def test_middle_golden_reference_semantics():
    for rec in small()["middle"]:
        A = _pm(rec["p"], rec["A"], rec["m"], rec["k"])
        B = _pm(rec["p"], rec["B"], rec["k"], rec["n"])
        R = F._pm_middle(A, B, rec["c"], rec["d"])
        assert R.rows == rec["R"], (rec["p"], rec["c"], rec["d"])
        T = F._pm_middle(A, B, rec["c"], rec["d"], exact=True)
        assert T.rows == rec["true_slice"]
        if "public" in rec:
            assert F.pm_middle_product(A, B, rec["c"], rec["d"]).rows == rec["public"]
        else:
            with pytest.raises(F.errors.DegreeTooLarge):
                F.pm_middle_product(A, B, rec["c"], rec["d"])


def test_mbasis1_golden():
    for rec in small()["mbasis1"]:
        ctx = F.field_new(rec["p"])
        assert F.mbasis1(rec["R"], rec["s"], ctx).rows == rec["P"]


def test_mbasis_golden():
    for rec in small()["mbasis"]:
        Fm = _pm(rec["p"], rec["F"], rec["m"], rec["n"])
        assert F.mbasis(Fm, rec["sigma"], rec["s"]).rows == rec["P"]


@pytest.mark.parametrize("T", [32, 8, 1])
def test_pmbasis_golden(T):
    from paper_1905_04356_b200 import config

    old = config.PMBASIS_BASE_ORDER
    config.PMBASIS_BASE_ORDER = T
    try:
        for rec in small()["pmbasis"]:
            Fm = _pm(rec["p"], rec["F"], rec["m"], rec["n"])
            assert F.pmbasis(Fm, rec["sigma"], rec["s"]).rows == rec["P"], (rec["p"], rec["sigma"])
    finally:
        config.PMBASIS_BASE_ORDER = old


def _dense_rand(p, shape, seed):
    return np.random.default_rng(seed).integers(0, p, size=shape, dtype=np.uint64)


@pytest.mark.parametrize("p,m,k,n,la,lb", [
    (P31, 5, 7, 3, 1000, 37),
    (P31, 32, 32, 32, 511, 513),
    (P31, 1, 64, 1, 4096, 4096),
    (P31, 3, 2, 4, 16384, 100),
    (P60, 4, 5, 3, 300, 700),
    (1152921493869428737, 3, 3, 3, 200, 200),
    (786433, 6, 6, 6, 2000, 2000),
    (97, 4, 4, 4, 500, 500),
    # tensor-core pointwise path (m >= 64, k >= 64, n >= 32), incl. ragged shapes
    (P31, 72, 128, 40, 300, 200),
    (P31, 64, 64, 64, 1000, 1000),
    (P31, 130, 68, 33, 40, 90),
    (P60, 64, 64, 64, 100, 100),
    (1152921493869428737, 64, 96, 32, 64, 64),
])
def test_pm_mul_vs_oracle(p, m, k, n, la, lb):
    A = _dense_rand(p, (m, k, la), 10 + m)
    B = _dense_rand(p, (k, n, lb), 20 + n)
    C = dense.to_numpy(dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p), p)
    assert np.array_equal(C.astype(np.uint64), O.pm_mul(p, A, B))


@pytest.mark.parametrize("p,m,k,la,env", [
    (P31, 32, 32, 1000, 1500),      # point-quad tensor-core layout cached
    (P31, 4, 3, 300, 300),          # CUDA-core blocked layout
    (P31, 72, 64, 100, 200),        # point-major (grouped TC) layout
    (P60, 5, 4, 200, 250),          # multi-prime: cache keyed by the prime set
    (97, 3, 3, 10, 12),             # tiny two-adicity
])
def test_multiplier_cached_evaluations(p, m, k, la, env):
    """Multiplier (polmat.py:550-610): A's transforms cached on the device; every
    apply equals the product, layouts switch when n changes the kernel choice."""
    A = _dense_rand(p, (m, k, la), 31 + m)
    mu = dense.DenseMultiplier(dense.to_device(A, p), p, env)
    for idx, (n, lb) in enumerate([(m, env), (3, env // 2), (m, 1), (40, env)]):
        B = _dense_rand(p, (k, n, lb), 50 + idx)
        C = dense.to_numpy(mu.apply(dense.to_device(B, p)), p)
        assert np.array_equal(C.astype(np.uint64), O.pm_mul(p, A, B)), (n, lb)
    with pytest.raises(F.errors.EnvelopeExceeded):
        mu.apply(dense.to_device(_dense_rand(p, (k, 2, env + 1), 9), p))
    mu.close()


def test_multiplier_polmat_api():
    ctx = F.field_new(P31)
    rng = random.Random(4)
    A = F.random_polmat(ctx, 3, 4, 40, rng)
    mu = F.polmat.multiplier_precompute(A, 60)
    for d in (60, 10, 0):
        B = F.random_polmat(ctx, 4, 2, d, rng)
        assert F.polmat.multiplier_apply(mu, B) == F.pm_mul(A, B)
    with pytest.raises(F.errors.EnvelopeExceeded):
        F.polmat.multiplier_apply(mu, F.random_polmat(ctx, 4, 2, 61, rng))


def test_host_abi_matches_device():
    import ctypes

    from paper_1905_04356_b200 import _lib

    p = P31
    A = _dense_rand(p, (4, 3, 200), 1).astype(np.uint32)
    B = _dense_rand(p, (3, 2, 300), 2).astype(np.uint32)
    C = np.zeros((4, 2, 499), dtype=np.uint32)
    h = _lib.context()
    _lib.check(_lib.lib().fpm_polmat_mul_host(
        h, p, 4, A.ctypes.data, 4, 3, 200, B.ctypes.data, 2, 300, C.ctypes.data), "host")
    assert np.array_equal(C.astype(np.uint64), O.pm_mul(p, A, B))
    _ = ctypes


@pytest.mark.parametrize("p,m,k,n,la,lb,blocks", [
    (P31, 9, 3, 11, 16000, 16000, 0),   # C >= 8 MB: 4 x 4 pipelined blocks, uneven edges
    (P60, 8, 2, 9, 9000, 9000, 0),      # u64 CRT path through the same pipeline
    (P31, 64, 48, 72, 2048, 2048, 8),   # 8 x 8 blocks (the >= 512 MB rule), tensor-core NTT
    (P31, 200, 40, 136, 1500, 600, 2),  # 2 x 2: 100-row blocks on tc_grouped, 68-column B blocks
])
def test_host_abi_pipelined_blocks(p, m, k, n, la, lb, blocks):
    """fpm_polmat_mul_host on a product large enough for the block pipeline
    (copy-in / compute / copy-out streams) equals the device entry point."""
    import torch

    from paper_1905_04356_b200 import _lib

    _lib.set_option("host_blocks", blocks)
    try:
        _host_blocks_case(p, m, k, n, la, lb)
    finally:
        _lib.set_option("host_blocks", 0)
    _ = torch


def _host_blocks_case(p, m, k, n, la, lb):
    from paper_1905_04356_b200 import _lib

    eb = dense.elem_bytes_for(p)
    A = _dense_rand(p, (m, k, la), 11)
    B = _dense_rand(p, (k, n, lb), 12)
    dt = np.uint32 if eb == 4 else np.uint64
    Ah, Bh = A.astype(dt), B.astype(dt)
    Ch = np.zeros((m, n, la + lb - 1), dtype=dt)
    h = _lib.context()
    _lib.check(_lib.lib().fpm_polmat_mul_host(
        h, p, eb, Ah.ctypes.data, m, k, la, Bh.ctypes.data, n, lb, Ch.ctypes.data), "host")
    ref = dense.to_numpy(dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p), p)
    assert np.array_equal(Ch, ref)
    # sampled entries against the oracle as well
    for (i, j) in [(0, 0), (m - 1, n - 1), (m // 2, n // 3)]:
        exp = O.pm_mul(p, A[i:i + 1], B[:, j:j + 1])
        assert np.array_equal(Ch[i, j].astype(np.uint64), exp[0, 0])


def _sha_of_mul(seed, p, m, k, n, deg):
    rng = random.Random(seed)
    A = random_polmat_dense(p, m, k, deg, rng)
    B = random_polmat_dense(p, k, n, deg, rng)
    C = dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p)
    return O.sha16(p, dense.to_numpy(C, p))


@pytest.mark.parametrize("key,args", [
    ("mul_s1_p2013265921_4x4x4_d1023", (1, P31, 4, 4, 4, 1023)),
    ("mul_s2_p2013265921_32x32x32_d4095", (2, P31, 32, 32, 32, 4095)),
    ("mul_s3_p1152921504606846883_16x16x16_d2047", (3, P60, 16, 16, 16, 2047)),
    ("mul_s5_p2013265921_64x64x64_d2047", (5, P31, 64, 64, 64, 2047)),
])
def test_full_size_mul_checksums(key, args):
    """cfg1, cfg2, cfg3 and the cfg5 scaled proxy against the checksum of the
    reference's own output (tests/golden/big_goldens.jsonl)."""
    g = big_goldens().get(key)
    if g is None:
        pytest.skip(f"{key} not generated")
    assert _sha_of_mul(*args) == g["sha16"]


@pytest.mark.parametrize("sigma", [64, 128, 256])
def test_pmbasis_checksums(sigma):
    g = big_goldens().get(f"pmb_s3_p2013265921_64x32_o{sigma}")
    if g is None:
        pytest.skip("not generated")
    rng = random.Random(3)
    Fd = random_polmat_dense(P31, 64, 32, sigma - 1, rng)
    P, _ = dense.pmbasis_dense(dense.to_device(Fd, P31), sigma, [0] * 64, P31)
    assert O.sha16(P31, dense.to_numpy(P, P31)) == g["sha16"]


def test_cfg4_full_checksum():
    g = big_goldens().get("pmb_s4_p2013265921_64x32_o4096")
    if g is None:
        pytest.skip("cfg4 reference checksum not generated yet")
    rng = random.Random(4)
    Fd = random_polmat_dense(P31, 64, 32, 4095, rng)
    P, _ = dense.pmbasis_dense(dense.to_device(Fd, P31), 4096, [0] * 64, P31)
    assert O.sha16(P31, dense.to_numpy(P, P31)) == g["sha16"]


def _eval_dense(M, x, p):
    """Horner evaluation of every entry at x (uint64, values < 2^31)."""
    acc = np.zeros(M.shape[:2], dtype=np.uint64)
    for t in range(M.shape[2] - 1, -1, -1):
        acc = (acc * np.uint64(x) + M[:, :, t].astype(np.uint64)) % np.uint64(p)
    return acc


def _matmul_mod(A, B, p):
    lo = (B & np.uint64(0xFFFF)).astype(np.uint64)
    hi = (B >> np.uint64(16)).astype(np.uint64)
    r_lo = (A @ lo) % np.uint64(p)
    r_hi = (A @ hi) % np.uint64(p)
    return (r_lo + (r_hi * np.uint64(1 << 16)) % np.uint64(p)) % np.uint64(p)


def test_cfg5_full_size_properties():
    """cfg5 (256x256 . 256x256, deg < 2048): Schwartz-Zippel at random points
    plus exact oracle products for sampled output entries."""
    import torch

    p = P31
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randint(0, p, (256, 256, 2048), generator=g, device="cuda", dtype=torch.int64)
    B = torch.randint(0, p, (256, 256, 2048), generator=g, device="cuda", dtype=torch.int64)
    A = A.to(torch.int32)
    B = B.to(torch.int32)
    C = dense.pm_mul_dense(A, B, p)
    An = dense.to_numpy(A, p).astype(np.uint64)
    Bn = dense.to_numpy(B, p).astype(np.uint64)
    Cn = dense.to_numpy(C, p).astype(np.uint64)
    for x in (12345, 987654321):
        assert np.array_equal(_eval_dense(Cn, x, p),
                              _matmul_mod(_eval_dense(An, x, p), _eval_dense(Bn, x, p), p))
    rng = np.random.default_rng(7)
    for _ in range(3):
        i, j = (int(v) for v in rng.integers(0, 256, 2))
        ref = O.pm_mul(p, An[i:i + 1], Bn[:, j:j + 1])
        assert np.array_equal(Cn[i:i + 1, j:j + 1], ref)


def test_cfg5_full_size_every_entry():
    """cfg5 at BASELINE's full size, every one of the 256 x 256 x 4095 output
    words against the multi-threaded C port (oracle/fpm_port.c, itself checked
    against the pinned oracle in tests/test_oracle_golden.py)."""
    import torch

    p = P31
    g = torch.Generator(device="cuda").manual_seed(55)
    A = torch.randint(0, p, (256, 256, 2048), generator=g, device="cuda", dtype=torch.int64)
    B = torch.randint(0, p, (256, 256, 2048), generator=g, device="cuda", dtype=torch.int64)
    A[3, 5, :] = p - 1
    B[5, 7, :] = p - 1
    A = A.to(torch.int32)
    B = B.to(torch.int32)
    Cn = dense.to_numpy(dense.pm_mul_dense(A, B, p), p)
    ref = O.port_mul31(p, dense.to_numpy(A, p), dense.to_numpy(B, p))
    assert Cn.shape == ref.shape
    assert np.array_equal(Cn.astype(np.uint32), ref)


@pytest.mark.parametrize("p", [(1 << 62) - 57, P60, (1 << 40) - 87])
def test_pm_mul_multiprime_extremes(p):
    """Multi-prime products at the top of the modulus range: the Garner
    recombination sums the mixed-radix digits as one 128-bit value before a
    single reduction (crt.cu), so all-(p-1) operands are the worst case."""
    rng = np.random.default_rng(p % 1000)
    for (m, k, n, la, lb, full) in [(3, 4, 2, 1500, 1300, False), (2, 5, 3, 700, 900, True)]:
        if full:
            A = np.full((m, k, la), p - 1, dtype=np.uint64)
            B = np.full((k, n, lb), p - 1, dtype=np.uint64)
        else:
            A = rng.integers(0, p, size=(m, k, la), dtype=np.uint64)
            B = rng.integers(0, p, size=(k, n, lb), dtype=np.uint64)
        C = dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p)
        assert np.array_equal(dense.to_numpy(C, p).astype(np.uint64), O.pm_mul(p, A, B)), (p, m, k, n)
