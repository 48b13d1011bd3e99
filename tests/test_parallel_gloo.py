"""world_size-2 gloo tests of the multi-rank product path (CPU only)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1905_04356_b200.parallel import max_over_ranks, pm_mul_rowsharded, row_block

P = 2013265921


def _oracle_mul(A, B, p):
    from oracle import oracle as O

    a = A.numpy().view(np.uint32).astype(np.uint64)
    b = B.numpy().view(np.uint32).astype(np.uint64)
    c = O.pm_mul(p, a, b).astype(np.uint32)
    return torch.from_numpy(c.view(np.int32))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(42)  # same inputs on every rank
        A = rng.integers(0, P, size=(7, 3, 20), dtype=np.uint64).astype(np.uint32)
        B = rng.integers(0, P, size=(3, 2, 15), dtype=np.uint64).astype(np.uint32)
        At = torch.from_numpy(A.view(np.int32))
        Bt = torch.from_numpy(B.view(np.int32))
        C = pm_mul_rowsharded(At, Bt, P, mul=_oracle_mul)
        full = _oracle_mul(At, Bt, P)
        ok = torch.equal(C, full)
        t = max_over_ranks(1.0 + rank)
        q.put((rank, ok, t))
    finally:
        dist.destroy_process_group()


def test_row_block_partition():
    for m in (1, 5, 64, 257):
        for w in (1, 2, 3, 8):
            blocks = [row_block(m, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))


@pytest.mark.timeout(300)
def test_rowsharded_product_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    assert all(t == 2.0 for _, _, t in res)  # max over ranks
