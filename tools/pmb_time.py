"""Best-of-N time of one cfg4-shaped PM-Basis (64 x 32) at order SIGMA.

usage: python tools/pmb_time.py [SIGMA] [N]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1905_04356_b200 import dense  # noqa: E402


def main():
    sigma = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    cfg = dict(bench.CONFIGS["cfg4"], sigma=sigma)
    F = bench.make_inputs(cfg, "cuda", 4)[0]
    ts = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dense.pmbasis_dense(F, sigma, [0] * cfg["m"], cfg["p"])
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    ts = sorted(ts[1:])
    print(f"pmbasis 64x32 order {sigma}: best {ts[0]:.2f} ms, median {ts[len(ts) // 2]:.2f} ms")


if __name__ == "__main__":
    main()
