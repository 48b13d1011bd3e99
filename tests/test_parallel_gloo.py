"""world_size 2 and 4 gloo tests of the multi-rank product splits (CPU only):
2-D (A-row x B-column) blocking with all_gather / gather to one rank, and the
multi-prime product split one word prime per rank with the residues
gathered to the CRT rank.  The per-rank compute is injected (the CPU
oracle), so these check the host logic: block and prime assignment,
padding, collectives, reassembly and recombination."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1905_04356_b200.parallel import (block_of, grid_shape, max_over_ranks, primes_of,
                                            row_block)

P31 = 2013265921
P60 = (1 << 60) - 93


def _oracle_mul(A, B, p):
    from oracle import oracle as O

    if A.dtype == torch.int32:
        a = A.numpy().view(np.uint32).astype(np.uint64)
        b = B.numpy().view(np.uint32).astype(np.uint64)
        return torch.from_numpy(O.pm_mul(p, a, b).astype(np.uint32).view(np.int32))
    c = O.pm_mul(p, A.numpy().view(np.uint64), B.numpy().view(np.uint64))
    return torch.from_numpy(c.view(np.int64))


def _cpu_residues(X, p, qs):
    x = X.numpy().view(np.uint64) if X.dtype == torch.int64 else X.numpy().view(np.uint32)
    out = np.stack([(x.astype(np.uint64) % np.uint64(q)).astype(np.uint32) for q in qs])
    return torch.from_numpy(out.view(np.int32))


def _cpu_crt(R, p, qs):
    """Garner-free CRT with Python integers (test stand-in for fpm_crt_combine)."""
    r = R.numpy().view(np.uint32).astype(object)
    M = 1
    for q in qs:
        M *= q
    acc = np.zeros(r.shape[1:], dtype=object)
    for z, q in enumerate(qs):
        Mi = M // q
        acc = acc + r[z] * (Mi * pow(Mi, -1, q))
    out = (acc % M) % p
    return torch.from_numpy(out.astype(np.uint64).view(np.int64))


def _worker(rank, world, port, q, kind):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1905_04356_b200 import parallel

        rng = np.random.default_rng(42)  # same inputs on every rank
        res = {}
        if kind == "2d":
            A = rng.integers(0, P31, size=(7, 3, 20), dtype=np.uint64).astype(np.uint32)
            B = rng.integers(0, P31, size=(3, 5, 15), dtype=np.uint64).astype(np.uint32)
            At = torch.from_numpy(A.view(np.int32))
            Bt = torch.from_numpy(B.view(np.int32))
            full = _oracle_mul(At, Bt, P31)
            C = parallel.pm_mul_sharded(At, Bt, P31, mul=_oracle_mul)
            res["all"] = torch.equal(C, full)
            Cb = parallel.pm_mul_2d(At, Bt, P31, rank, world, mul=_oracle_mul)
            (a, b), (c, d) = block_of(rank, world, 7, 5)
            res["block"] = torch.equal(Cb, full[a:b, c:d])
            C1 = parallel.gather_blocks(Cb, 7, 5, dst=world - 1)
            res["dst"] = (C1 is None) if rank != world - 1 else torch.equal(C1, full)
        else:
            from paper_1905_04356_b200 import dense

            A = rng.integers(0, P60, size=(3, 4, 25), dtype=np.uint64)
            B = rng.integers(0, P60, size=(4, 2, 18), dtype=np.uint64)
            A[0, 0, :] = P60 - 1
            B[0, 0, :] = P60 - 1
            At = torch.from_numpy(A.view(np.int64))
            Bt = torch.from_numpy(B.view(np.int64))
            primes = dense.product_primes(P60, 4, 25, 18)
            res["nprimes"] = len(primes)
            C = parallel.pm_mul_prime_split(At, Bt, P60, dst=0, primes=primes, mul=_oracle_mul,
                                             residues=_cpu_residues, crt=_cpu_crt)
            if rank == 0:
                res["all"] = torch.equal(C, _oracle_mul(At, Bt, P60))
            else:
                res["all"] = C is None
        res["max"] = max_over_ranks(1.0 + rank)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _spawn(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + 7 * world + (0 if kind == "2d" else 3)
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, kind)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    return res


def test_partitions():
    for m in (1, 5, 64, 257):
        for w in (1, 2, 3, 8):
            blocks = [row_block(m, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
    assert [grid_shape(w) for w in (1, 2, 4, 8, 6)] == [(1, 1), (1, 2), (2, 2), (2, 4), (2, 3)]
    for w in (1, 2, 4, 8):
        cover = np.zeros((256, 256), dtype=int)
        for r in range(w):
            (a, b), (c, d) = block_of(r, w, 256, 256)
            cover[a:b, c:d] += 1
        assert (cover == 1).all()
    qs = [1, 2, 3, 4, 5]
    assert sorted(sum((primes_of(r, 2, qs) for r in range(2)), [])) == qs


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 4])
def test_2d_blocked_product_gloo(world):
    res = _spawn(world, "2d")
    assert all(r["all"] and r["block"] and r["dst"] for _, r in res), res
    assert all(r["max"] == float(world) for _, r in res)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 4])
def test_prime_split_product_gloo(world):
    res = _spawn(world, "prime")
    assert all(r["all"] for _, r in res), res
    assert res[0][1]["nprimes"] == 5  # cfg3's prime count for a 60-bit modulus
