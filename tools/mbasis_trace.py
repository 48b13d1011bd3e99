"""Per-step phase clocks of an M-Basis leaf (FPM_MBASIS_TRACE=1).

usage: FPM_MBASIS_TRACE=1 python tools/mbasis_trace.py
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1905_04356_b200 import _lib, dense  # noqa: E402


def main():
    cfg = dict(bench.CONFIGS["cfg4"], sigma=256)
    F = bench.make_inputs(cfg, "cuda", 4)[0]
    dense.pmbasis_dense(F, cfg["sigma"], [0] * cfg["m"], cfg["p"], T=int(os.environ.get("LEAF_T", "16")))
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 512)()
    assert _lib.lib().fpm_debug_mbasis_trace(buf) == 0
    names = ["solve", "inv", "C", "Ct", "residual", "shift", "next_start"]
    print("pair path: solve = [start, first block] [pair loop] [inverses]")
    print("step " + " ".join(f"{n:>10s}" for n in names))
    for k in range(16):
        r = [buf[k * 8 + e] for e in range(8)]
        nxt = buf[(k + 1) * 8] if k < 15 else r[4]
        if r[7] and r[6] and r[5]:
            d = [r[7] - r[0], r[6] - r[7], r[5] - r[6]]
        elif r[5] and r[6]:
            d = [r[5] - r[0], r[6] - r[5], r[1] - r[6]]
        else:
            d = [r[1] - r[0], 0, 0]
        d += [r[2] - r[1], r[3] - r[2], r[4] - r[3], nxt - r[4]]
        print(f"{k:4d} " + " ".join(f"{x:10d}" for x in d) + f"   (solve end -> record start {r[1] - r[5]})")
    t0, t1 = buf[63 * 8], buf[63 * 8 + 1]
    T = int(os.environ.get("LEAF_T", "16"))
    if t0 and t1:
        print(f"kernel {t1 - t0} cycles: start -> step 0 ranked {buf[0] - t0}, "
              f"last step end -> kernel end {t1 - buf[(T - 1) * 8 + 4]}")


if __name__ == "__main__":
    main()
