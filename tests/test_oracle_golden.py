"""Pin the CPU oracle (oracle/) against fixtures produced by the reference
itself (tests/golden/make_golden.py, make_golden_big.py).  CPU only."""
import random

import numpy as np
import pytest

from golden_util import big_goldens, dense, random_polmat_dense, rows_from_dense, small
from oracle import oracle as O


def test_field_roots():
    for rec in small()["primes"]:
        assert O.two_adicity(rec["p"]) == rec["two_adicity"]
        if rec["p"] > 2:
            assert O.ntt_root(rec["p"]) == rec["ntt_root"]


def test_ntt_vectors():
    for rec in small()["ntt"]:
        p = rec["p"]
        assert O.ntt(p, rec["v"]).tolist() == rec["fwd"]
        assert O.ntt(p, rec["v"], inverse=True).tolist() == rec["inv"]


def test_pm_mul_golden():
    for rec in small()["mul"]:
        A = dense(rec["A"], rec["m"], rec["k"])
        B = dense(rec["B"], rec["k"], rec["n"])
        if A.shape[2] == 0 or B.shape[2] == 0:
            assert all(not e for r in rec["C"] for e in r)
            continue
        C = O.pm_mul(rec["p"], A, B)
        assert rows_from_dense(C) == rec["C"]


def test_pm_middle_golden():
    for rec in small()["middle"]:
        A = dense(rec["A"], rec["m"], rec["k"])
        B = dense(rec["B"], rec["k"], rec["n"])
        R = O.pm_middle(rec["p"], A, B, rec["c"], rec["d"])
        assert rows_from_dense(R) == rec["R"]


def test_mbasis1_golden():
    for rec in small()["mbasis1"]:
        if "pivots" not in rec:
            continue
        isp, kern = O.mbasis1_struct(rec["p"], np.array(rec["R"], dtype=np.uint64), rec["s"])
        assert sorted(np.flatnonzero(isp).tolist()) == rec["pivots"]
        for i_str, kv in rec["kernel"].items():
            i = int(i_str)
            got = [(j, int(c)) for j, c in enumerate(kern[i].tolist()) if c]
            assert got == [tuple(x) for x in kv]


def test_mbasis_golden():
    for rec in small()["mbasis"]:
        F = dense(rec["F"], rec["m"], rec["n"], rec["sigma"])
        P, _ = O.mbasis(rec["p"], F, rec["sigma"], rec["s"])
        assert rows_from_dense(P) == rec["P"]


@pytest.mark.parametrize("T", [32, 4, 1])
def test_pmbasis_golden(T):
    for rec in small()["pmbasis"]:
        F = dense(rec["F"], rec["m"], rec["n"], rec["sigma"])
        P = O.pmbasis(rec["p"], F, rec["sigma"], rec["s"], T=T)
        assert rows_from_dense(P) == rec["P"]


def test_cfg1_checksum():
    """cfg1 full size against the reference's checksum."""
    g = big_goldens().get("mul_s1_p2013265921_4x4x4_d1023")
    if g is None:
        pytest.skip("big golden not generated yet")
    p = 2013265921
    rng = random.Random(1)
    A = random_polmat_dense(p, 4, 4, 1023, rng)
    B = random_polmat_dense(p, 4, 4, 1023, rng)
    assert O.sha16(p, O.pm_mul(p, A, B)) == g["sha16"]


def test_pmbasis_sigma64_checksum():
    g = big_goldens().get("pmb_s3_p2013265921_64x32_o64")
    if g is None:
        pytest.skip("big golden not generated yet")
    p = 2013265921
    rng = random.Random(3)
    F = random_polmat_dense(p, 64, 32, 63, rng)
    O.set_threads(8)
    assert O.sha16(p, O.pmbasis(p, F, 64, [0] * 64)) == g["sha16"]


@pytest.mark.parametrize("m,k,n,la,lb,threads", [(3, 5, 2, 100, 37, 1), (4, 4, 4, 1024, 1024, 4),
                                                 (17, 9, 6, 1, 300, 3), (2, 33, 2, 2048, 2047, 2)])
def test_port_matches_oracle(m, k, n, la, lb, threads):
    """The multi-threaded C port (oracle/fpm_port.c: the bench's reference arm and
    the checker of the full-size cfg5 GPU test) against the pinned oracle."""
    for p in (2013265921, 469762049):
        rng = np.random.default_rng(m * 1000 + la)
        A = rng.integers(0, p, size=(m, k, la), dtype=np.uint64)
        B = rng.integers(0, p, size=(k, n, lb), dtype=np.uint64)
        A[0, 0, :] = p - 1
        B[0, 0, :] = p - 1
        got = O.port_mul31(p, A.astype(np.uint32), B.astype(np.uint32), threads=threads)
        assert np.array_equal(got.astype(np.uint64), O.pm_mul(p, A, B))
