"""A/B of library options on one bench configuration (one process): per
variant the mean step time (CUDA events, L2 flushed between steps) and the
per-stage event times.

usage: python tools/opt_ab.py CFG "opt=v,opt=v" ["..." ...]   ("-" = defaults)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1905_04356_b200 import _lib  # noqa: E402


def main():
    name = sys.argv[1]
    cfg = bench.CONFIGS[name]
    inputs = bench.make_inputs(cfg, "cuda", 11)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    h = _lib.context(0)
    for spec in sys.argv[2:]:
        _lib.set_option(None, 0)
        opts = [] if spec == "-" else [kv.split("=") for kv in spec.split(",")]
        for k, v in opts:
            _lib.set_option(k, int(v))
        times, stages, _ = bench.time_steps(cfg, inputs, 10, 3, flush, profile_h=h)
        st = {k: round(sum(v) / len(v), 4) for k, v in stages.items()}
        print(f"{name} [{spec}] ms/step {sum(times) / len(times):.4f} stages {st}", flush=True)
    _lib.set_option(None, 0)


if __name__ == "__main__":
    main()
