"""PM-Basis (cfg4 shape) cost per tree level: t(2s) - 2 t(s) is the cost of
one node of order 2s (its middle product, product and shift bookkeeping).
Also prints the per-stage profile records of one full run, summed by name.

usage: python tools/pmb_levels.py [SIGMA_MAX]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1905_04356_b200 import _lib, dense  # noqa: E402


def timed(F, sigma, cfg, reps=3):
    best = 1e9
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dense.pmbasis_dense(F, sigma, [0] * cfg["m"], cfg["p"])
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def main():
    smax = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    cfg = dict(bench.CONFIGS["cfg4"], sigma=smax)
    F = bench.make_inputs(cfg, "cuda", 4)[0]
    prev = None
    s = 8
    total_nodes = 0.0
    while s <= smax:
        t = timed(F, s, cfg)
        if prev is not None:
            node = t - 2 * prev
            count = smax // s
            total_nodes += node * count
            print(f"order {s:5d}: {t:9.3f} ms   node {node * 1e3:9.1f} us x {count:4d} = "
                  f"{node * count:7.3f} ms", flush=True)
        else:
            print(f"order {s:5d}: {t:9.3f} ms   (leaf) x {smax // s} = {t * smax / s:7.3f} ms",
                  flush=True)
        prev = t
        s *= 2
    print(f"sum of node costs: {total_nodes:.3f} ms")
    h = _lib.context()
    _lib.profile(h, True)
    dense.pmbasis_dense(F, smax, [0] * cfg["m"], cfg["p"])
    torch.cuda.synchronize()
    recs = _lib.profile_records(h)
    _lib.profile(h, False)
    agg = {}
    for nm, ms in recs:
        c, t = agg.get(nm, (0, 0.0))
        agg[nm] = (c + 1, t + ms)
    for nm, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{nm:28s} {c:6d} launches {t:9.3f} ms  ({t / c * 1e3:8.1f} us each)")


if __name__ == "__main__":
    main()
