"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck).

usage: python tools/sanitize_cases.py CASE
Each case runs one product / basis through the package on cuda:0 and checks
it against the oracle, so a sanitizer run also proves the result.  Cases are
sized so racecheck (which serialises shared-memory accesses) finishes in
minutes:
  cfg1     4x4 deg<1024 product (ntt_tma G=1, pointwise_cc)
  cfg2s    32x32x32 deg<1024 product (grouped TMA NTT, tc_pq tensor-core kernel)
  cfg3s    16x16x16 deg<256 over a 60-bit prime (split-reduce, CRT)
  cfg5p    64x64x64 deg<512 product (persistent PM NTT, tc_grouped kernel)
  pmb256   PM-Basis 16x8 order 256 (M-Basis leaves, tree products, middle products)
  big      2x2 deg<40000 product (multi-pass four-step NTT, N = 2^17)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1905_04356_b200 import dense  # noqa: E402

P31 = 2013265921
P60 = 1152921504606846883


def _mul(p, m, k, n, ln, seed):
    rng = np.random.default_rng(seed)
    A = rng.integers(0, p, size=(m, k, ln), dtype=np.uint64)
    B = rng.integers(0, p, size=(k, n, ln), dtype=np.uint64)
    C = dense.pm_mul_dense(dense.to_device(A, p), dense.to_device(B, p), p)
    got = dense.to_numpy(C, p).astype(np.uint64)
    if m * k * n * ln <= 32 * 32 * 32 * 1024:
        ref = O.pm_mul(p, A, B)
        assert np.array_equal(got, ref), "product differs from the oracle"
    else:
        # sampled entries against the oracle
        for (i, j) in [(0, 0), (m - 1, n - 1)]:
            ref = O.pm_mul(p, A[i:i + 1], B[:, j:j + 1])
            assert np.array_equal(got[i:i + 1, j:j + 1], ref), "sampled entry differs"


def main():
    case = sys.argv[1]
    if case == "cfg1":
        _mul(P31, 4, 4, 4, 1024, 1)
    elif case == "cfg2s":
        _mul(P31, 32, 32, 32, 1024, 2)
    elif case == "cfg3s":
        _mul(P60, 16, 16, 16, 256, 3)
    elif case == "cfg5p":
        _mul(P31, 64, 64, 64, 512, 5)
    elif case == "big":
        _mul(P31, 2, 2, 2, 40000, 7)
    elif case == "pmb256":
        rng = np.random.default_rng(4)
        F = rng.integers(0, P31, size=(16, 8, 256), dtype=np.uint64)
        P, _ = dense.pmbasis_dense(dense.to_device(F, P31), 256, [0] * 16, P31)
        got = dense.to_numpy(P, P31).astype(np.uint64)
        ref = O.pmbasis(P31, F, 256, [0] * 16)
        assert got.shape == ref.shape and np.array_equal(got, ref), "pmbasis differs"
    else:
        raise SystemExit("unknown case " + case)
    print("ok", case)


if __name__ == "__main__":
    main()
