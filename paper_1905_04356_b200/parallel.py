"""Multi-GPU sharding of the product path.

One process per GPU with torch.distributed (NCCL over NVLink on B200 boxes,
gloo in the CPU tests).  The reference is single-process; these helpers are
the only place a collective appears:

* ``pm_mul`` shards by ROW BLOCKS of A: every rank multiplies its row block
  by the full B (no data-path exchange during the product) and one
  all-gather assembles C.  Independent products (the bench's units) need no
  collective at all (weak scaling, replicas).
* multi-prime products could shard by prime (one residue product per rank,
  gather to the CRT rank); PM-Basis is replicas only -- its order-1 chain is
  sequential (appint.py:153-179, :188-196).
"""


def row_block(m, world, rank):
    """[lo, hi) rows owned by `rank` when m rows are split over `world` ranks."""
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def pm_mul_rowsharded(A, B, p, group=None, mul=None):
    """C = A * B with A's rows split across the ranks of `group`.

    A: (m, k, la) tensor (full, or at least this rank's row block at its
    global offset); B: (k, n, lb) replicated.  Returns the full C on every
    rank.  `mul(A_block, B, p)` defaults to the GPU product
    (dense.pm_mul_dense); tests inject a CPU oracle."""
    import torch
    import torch.distributed as dist

    if mul is None:
        from .dense import pm_mul_dense as mul
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m = A.shape[0]
    lo, hi = row_block(m, world, rank)
    Cb = mul(A[lo:hi].contiguous(), B, p)
    rows_max = row_block(m, world, 0)[1] - row_block(m, world, 0)[0]
    n, lc = Cb.shape[1], Cb.shape[2]
    pad = torch.zeros((rows_max, n, lc), dtype=Cb.dtype, device=Cb.device)
    pad[: hi - lo] = Cb
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = []
    for r in range(world):
        rlo, rhi = row_block(m, world, r)
        out.append(parts[r][: rhi - rlo])
    return torch.cat(out, dim=0)


def max_over_ranks(value, group=None):
    """Bench timing rule: the job time is the slowest rank's time."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
