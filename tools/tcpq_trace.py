"""Per-item timeline of CTA 0 of the point-quad TC kernel (FPM_TCPQ_DBG=32).

usage: FPM_TCPQ_DBG=32 python tools/tcpq_trace.py [CFG]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1905_04356_b200 import _lib  # noqa: E402


def main():
    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
    inputs = bench.make_inputs(cfg, "cuda", 11)
    out = None
    for _ in range(3):
        out = bench.run_step(cfg, inputs, out)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 512)()
    L = _lib.lib()
    fn = L.fpm_debug_tcpq2_trace if os.environ.get("FPM_TCPQ2_TRACE") else L.fpm_debug_tcpq_trace
    assert fn(buf) == 0
    t0 = buf[0]
    names = (["tma", "A_full", "A_done", "B_done", "mma", "epi_t", "epi_stg", "epi_done"] if os.environ.get("FPM_TCPQ2_TRACE") else ["tma", "A_full", "A_done", "B_full", "B_done", "mma", "epi_t", "epi_done"])
    print("item " + " ".join(f"{n:>9s}" for n in names))
    for i in range(20):
        row = [buf[i * 8 + e] for e in range(8)]
        print(f"{i:4d} " + " ".join(f"{(v - t0) / 1000:9.2f}" if v else "        -" for v in row))


if __name__ == "__main__":
    main()
