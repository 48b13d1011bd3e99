# exercise the N > 1 step construction of bench.py for every rank of a world of 8 on ONE GPU
# (no process group: the split has no data-path collective)
import sys
sys.path.insert(0, '/root/repo')
import torch, bench
from paper_1905_04356_b200 import dense
from paper_1905_04356_b200.parallel import block_of
cfg = bench.CONFIGS["cfg5"]
A, B = bench.make_inputs(cfg, "cuda", 1000)
full = dense.pm_mul_dense(A, B, cfg["p"])
for world in (2, 4, 8):
    for rank in range(world):
        (r0, r1), (c0, c1) = block_of(rank, world, A.shape[0], B.shape[1])
        Ai, Bj = A[r0:r1].contiguous(), B[:, c0:c1].contiguous()
        out = torch.empty((r1 - r0, c1 - c0, A.shape[2] + B.shape[2] - 1), dtype=A.dtype, device="cuda")
        dense.pm_mul_dense(Ai, Bj, cfg["p"], out=out)
        assert torch.equal(out, full[r0:r1, c0:c1]), (world, rank)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10): dense.pm_mul_dense(Ai, Bj, cfg["p"], out=out)
    e1.record(); e1.synchronize()
    print(f"world {world}: every block equals the slice of the full product; last rank's block {e0.elapsed_time(e1)/10:.3f} ms per step")
