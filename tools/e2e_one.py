"""Median end-to-end (host buffers, C ABI) time of one BASELINE config.
usage: [FPM_HOST_BLOCKS=R] python tools/e2e_one.py CFG [STEPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1]]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 9
med, bi, bo = bench.e2e_mul(cfg, steps, 3, 7)
print(sys.argv[1], os.environ.get("FPM_HOST_BLOCKS", "auto"), f"{med * 1e3:.4f} ms", bi, bo)
