"""Run one configuration a few times (for ncu / launch-list captures).

usage: python tools/run_one.py CFG [REPS]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg = bench.CONFIGS[name]
    inputs = bench.make_inputs(cfg, "cuda", 11)
    out = None
    for _ in range(reps):
        out = bench.run_step(cfg, inputs, out if cfg["kind"] == "mul" else None)
    torch.cuda.synchronize()
    print("ok", name, reps)


if __name__ == "__main__":
    main()
