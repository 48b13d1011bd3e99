"""Round-2 goldens from the unmodified reference (tests/golden/make_golden_r2.py):
PM-Basis over a 60-bit prime of two-adicity 1 (entrywise middle products
on strided bases) and interpolant bases whose points repeat a residue."""
import json
import os
import random

import numpy as np
import pytest

import paper_1905_04356_b200 as F
from paper_1905_04356_b200 import dense

pytestmark = pytest.mark.gpu

with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "r2.json")) as f:
    R2 = json.load(f)


def _draw_pmb(rec):
    rng = random.Random(rec["seed"])
    p, m, n, order = rec["p"], rec["m"], rec["n"], rec["order"]
    return np.array([[[rng.randrange(p) for _ in range(order)] for _ in range(n)]
                     for _ in range(m)], dtype=np.uint64)


def _draw_ib(rec):
    rng = random.Random(rec["seed"])
    p, m, n, order = rec["p"], rec["m"], rec["n"], rec["order"]
    E = [[[rng.randrange(p) for _ in range(n)] for _ in range(m)] for _ in range(order)]
    alpha = [1, 1 + p] + rng.sample(range(1, p), order - 2)
    return E, alpha


@pytest.mark.parametrize("idx", range(len(R2["pmbasis"])))
def test_pmbasis_p60_two_adicity_1(idx):
    rec = R2["pmbasis"][idx]
    p = rec["p"]
    Fm = _draw_pmb(rec)
    P, _ = dense.pmbasis_dense(dense.to_device(Fm, p), rec["order"], rec["s"], p, T=rec["T"])
    got = F.polmat.from_dense(F.field_new(p), dense.to_numpy(P, p).astype(object),
                              ncols=rec["m"])
    assert got.rows == rec["P"]


@pytest.mark.parametrize("idx", range(len(R2["intbasis"])))
def test_intbasis_repeated_residue(idx):
    rec = R2["intbasis"][idx]
    E, alpha = _draw_ib(rec)
    assert alpha[0] % rec["p"] == alpha[1] % rec["p"]
    ctx = F.field_new(rec["p"])
    fn = getattr(F, rec["fn"])
    P = fn(E, alpha, [0] * rec["m"], ctx)
    assert P.rows == rec["P"]


def _one_rank_nccl():
    import socket

    import torch.distributed as dist

    if dist.is_initialized():
        return
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1)


def test_prime_split_pieces_match_the_product():
    """cfg3's shape through the split pieces on one GPU: residues per word
    prime, one direct product per prime, Garner -- equal to pm_mul_dense
    (which fuses the same steps), and through pm_mul_prime_split on a
    one-rank NCCL group."""
    from paper_1905_04356_b200 import parallel

    p = (1 << 60) - 93
    rng = np.random.default_rng(3)
    A = rng.integers(0, p, size=(16, 16, 2048), dtype=np.uint64)
    B = rng.integers(0, p, size=(16, 16, 2048), dtype=np.uint64)
    A[0, 0] = p - 1
    Ad, Bd = dense.to_device(A, p), dense.to_device(B, p)
    want = dense.to_numpy(dense.pm_mul_dense(Ad, Bd, p), p)
    primes = dense.product_primes(p, 16, 2048, 2048)
    assert len(primes) == 5
    Ar, Br = dense.split_residues(Ad, p, primes), dense.split_residues(Bd, p, primes)
    import torch

    R = torch.stack([dense.pm_mul_dense(Ar[z].contiguous(), Br[z].contiguous(), q)
                     for z, q in enumerate(primes)])
    got = dense.to_numpy(dense.crt_combine(R, p, primes), p)
    assert np.array_equal(got, want)
    _one_rank_nccl()
    C = parallel.pm_mul_prime_split(Ad, Bd, p, dst=0)
    assert np.array_equal(dense.to_numpy(C, p), want)


def test_2d_blocks_on_nccl():
    from paper_1905_04356_b200 import parallel

    p = 2013265921
    rng = np.random.default_rng(4)
    A = rng.integers(0, p, size=(40, 8, 300), dtype=np.uint64)
    B = rng.integers(0, p, size=(8, 24, 200), dtype=np.uint64)
    Ad, Bd = dense.to_device(A, p), dense.to_device(B, p)
    want = dense.to_numpy(dense.pm_mul_dense(Ad, Bd, p), p)
    _one_rank_nccl()
    C = parallel.pm_mul_sharded(Ad, Bd, p)
    assert np.array_equal(dense.to_numpy(C, p), want)
    # every block of a 2 x 4 grid, computed here one after another
    for r in range(8):
        Cb = parallel.pm_mul_2d(Ad, Bd, p, r, 8)
        (a, b), (c, d) = parallel.block_of(r, 8, 40, 24)
        assert np.array_equal(dense.to_numpy(Cb, p), want[a:b, c:d])


def _degenerate_64x32(kind, order, seed):
    """64 x 32 inputs whose residuals have zero leading minors: the pair solve
    of the leaf (csrc/mbasis_fast.cu:solve_pairs) must hand over to the general
    elimination, as appint._mbasis1_struct (appint.py:24-60) picks other pivots"""
    p = 2013265921
    rng = np.random.default_rng(seed)
    Fm = rng.integers(0, p, size=(64, 32, order), dtype=np.uint64)
    if kind == "equal_rows":
        Fm[1] = Fm[0]
        Fm[40] = Fm[7]
    elif kind == "zero_column":
        Fm[:, 5, :] = 0
    elif kind == "zero_constant":
        Fm[:, :, 0] = 0          # first residual is zero: a step without pivots
    elif kind == "zero_rows":
        Fm[0:3] = 0
    elif kind == "rank_drop":
        Fm[:, 16:, :] = Fm[:, :16, :]   # column j + 16 repeats column j
    return p, Fm


@pytest.mark.parametrize("kind", ["equal_rows", "zero_column", "zero_constant", "zero_rows",
                                  "rank_drop"])
@pytest.mark.parametrize("order,shift", [(8, "uniform"), (16, "mixed")])
def test_leaf_pair_solve_degenerate_residuals(kind, order, shift):
    from oracle import oracle as O

    p, Fm = _degenerate_64x32(kind, order, 5)
    s = [0] * 64 if shift == "uniform" else [(3 * i) % 5 - 2 for i in range(64)]
    P, _ = dense.pmbasis_dense(dense.to_device(Fm, p), order, s, p)
    got = dense.to_numpy(P, p).astype(np.uint64)
    ref = O.pmbasis(p, Fm, order, s)
    assert got.shape == ref.shape and np.array_equal(got, ref)
