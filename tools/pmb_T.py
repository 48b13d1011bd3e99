"""PM-Basis (cfg4 shape) time vs. leaf order T (output is T-independent).

usage: python tools/pmb_T.py [SIGMA]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1905_04356_b200 import _lib, dense  # noqa: E402


def main():
    sigma = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    cfg = dict(bench.CONFIGS["cfg4"], sigma=sigma)
    F = bench.make_inputs(cfg, "cuda", 4)[0]
    ref = None
    for T in [int(x) for x in os.environ.get('PMB_TS', '16,8,4,2').split(',')]:
        _lib.set_option("pmbasis_leaf", T)  # the cap of the device leaf order
        dense.pmbasis_dense(F, sigma, [0] * cfg["m"], cfg["p"], T=T)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P, rd = dense.pmbasis_dense(F, sigma, [0] * cfg["m"], cfg["p"], T=T)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        same = ref is None or torch.equal(P, ref)
        ref = P if ref is None else ref
        print(f"T={T:3d} {dt * 1e3:9.2f} ms  same={same}", flush=True)


if __name__ == "__main__":
    main()
