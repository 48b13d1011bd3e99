"""Median end-to-end (host buffers, C ABI) time of one BASELINE config.
usage: python tools/e2e_one.py CFG [STEPS] [HOST_BLOCKS ...]
With block counts given, each is forced through fpm_set_option("host_blocks")."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1905_04356_b200 import _lib  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1]]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 9
for r in (sys.argv[3:] or ["0"]):
    _lib.set_option("host_blocks", int(r))
    med, bi, bo = bench.e2e_mul(cfg, steps, 3, 7)
    print(sys.argv[1], "blocks", r if r != "0" else "auto", f"{med * 1e3:.4f} ms", bi, bo, flush=True)
_lib.set_option("host_blocks", 0)
