"""Multi-GPU splits of the product path.

One process per GPU with torch.distributed (NCCL over NVLink on B200 boxes,
gloo in the CPU tests).  The reference is single-process; these helpers are
the only place a collective appears.

* ``pm_mul_2d``: C = A * B over a gr x gc grid of ranks (2-D blocking).
  Rank (i, j) owns A's row block i and B's column block j -- the same
  (A-row x B-column) blocks the host pipeline of fpm_polmat_mul_host
  multiplies, each transformed once -- and computes C_ij with no exchange.
  Per rank: forward transforms of (m/gr) k + k (n/gc) entries (not the
  whole of B as a row split would), pointwise and inverse 1/G of the total.
  ``gather_blocks`` is the optional exchange when one consumer needs all of
  C: every rank contributes its (m/gr)(n/gc)(la+lb-1) words.
* ``pm_mul_prime_split``: a multi-prime product (p >= 2^31, cfg3's 60-bit
  prime) split one word prime per rank: rank r multiplies the residues of A
  and B mod q_r, r + G, ... on its GPU, the residue blocks are gathered to
  the CRT rank (dst) and combined there (Garner, fpm_crt_combine).
  Comm: each rank sends its primes' m n (la+lb-1) words; dst receives r of
  them.  The reference computes the same unique product by geometric
  evaluation (polmat.py:311-346); SPEC.md:254 allows splitting the points.
* PM-Basis is replicas only: its order-1 chain is sequential
  (appint.py:153-179, :188-196).

The compute callables (``mul``, ``residues``, ``crt``) default to the GPU
library; the gloo tests inject CPU stand-ins to check the host logic.
"""


def row_block(m, world, rank):
    """[lo, hi) rows owned by `rank` when m rows are split over `world` ranks."""
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def grid_shape(world):
    """(gr, gc) with gr * gc = world, as square as possible, gr <= gc."""
    gr = int(world ** 0.5)
    while world % gr:
        gr -= 1
    return gr, world // gr


def block_of(rank, world, m, n):
    """((row lo, hi), (col lo, hi)) of C owned by `rank` on the 2-D grid."""
    gr, gc = grid_shape(world)
    i, j = divmod(rank, gc)
    return row_block(m, gr, i), row_block(n, gc, j)


def pm_mul_2d(A, B, p, rank, world, mul=None):
    """This rank's block C_ij = A_i * B_j.  A, B: full operands or any
    tensors that hold this rank's rows / columns at their global offsets
    (only those are read).  No collective."""
    if mul is None:
        from .dense import pm_mul_dense as mul
    (r0, r1), (c0, c1) = block_of(rank, world, A.shape[0], B.shape[1])
    return mul(A[r0:r1].contiguous(), B[:, c0:c1].contiguous(), p)


def gather_blocks(Cb, m, n, group=None, dst=None):
    """Assemble C from the ranks' blocks (all_gather, or gather to dst: the
    other ranks return None).  Blocks are padded to the largest block."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lc = Cb.shape[2]
    (R0, R1), (C0, C1) = block_of(0, world, m, n)
    pad = torch.zeros((R1 - R0, C1 - C0, lc), dtype=Cb.dtype, device=Cb.device)
    pad[: Cb.shape[0], : Cb.shape[1]] = Cb
    if dst is None:
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
    else:
        parts = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
        dist.gather(pad, parts, dst=dst, group=group)
        if rank != dst:
            return None
    C = torch.empty((m, n, lc), dtype=Cb.dtype, device=Cb.device)
    for r in range(world):
        (a, b), (c, d) = block_of(r, world, m, n)
        C[a:b, c:d] = parts[r][: b - a, : d - c]
    return C


def pm_mul_sharded(A, B, p, group=None, mul=None, gather=True):
    """C = A * B on the 2-D rank grid of `group`; the full C on every rank
    (gather=True) or this rank's block (gather=False)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    Cb = pm_mul_2d(A, B, p, rank, world, mul=mul)
    return gather_blocks(Cb, A.shape[0], B.shape[1], group) if gather else Cb


def primes_of(rank, world, primes):
    """The word primes rank `rank` multiplies: primes[rank::world]."""
    return primes[rank::world]


def pm_mul_prime_split(A, B, p, group=None, dst=0, primes=None, mul=None, residues=None,
                       crt=None):
    """Multi-prime product split by word prime over the ranks of `group`,
    residues gathered to `dst` and recombined there.  Returns C (mod p) on
    dst, None elsewhere.  A (m, k, la), B (k, n, lb) replicated (values mod p).

    mul(Aq, Bq, q) multiplies residue operands mod the word prime q (default:
    the GPU product, a direct NTT prime); residues(X, p, qs) -> X mod q for q
    in qs; crt(R, p, qs) -> the Garner combination (defaults: the library)."""
    import torch
    import torch.distributed as dist

    from . import dense

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m, k, la = A.shape
    n, lb = B.shape[1], B.shape[2]
    if primes is None:
        primes = dense.product_primes(p, k, la, lb)
    mul = mul or dense.pm_mul_dense
    residues = residues or dense.split_residues
    crt = crt or dense.crt_combine
    mine = primes_of(rank, world, primes)
    lc = la + lb - 1
    per = -(-len(primes) // world)  # residue slots per rank (padded)
    buf = torch.zeros((per, m, n, lc), dtype=torch.int32, device=A.device)
    if mine:
        Ar = residues(A, p, mine)
        Br = residues(B, p, mine)
        for s, q in enumerate(mine):
            buf[s] = mul(Ar[s].contiguous(), Br[s].contiguous(), q)
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, parts, dst=dst, group=group)
    if rank != dst:
        return None
    R = torch.empty((len(primes), m, n, lc), dtype=torch.int32, device=A.device)
    for r in range(world):
        for s, q in enumerate(primes_of(r, world, primes)):
            R[primes.index(q)] = parts[r][s]
    return crt(R, p, primes)


def max_over_ranks(value, group=None):
    """Bench timing rule: the job time is the slowest rank's time."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
