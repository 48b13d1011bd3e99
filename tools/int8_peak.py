"""Measure the int8 tensor-core GEMM peak on this GPU (torch._int_mm, the
cuBLASLt int8 path) so the pointwise roofline has a measured denominator.

usage: python tools/int8_peak.py OUT.json
"""
import json
import sys
import time

import torch


def main():
    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    # sustained: back to back for ~3 s
    t0 = time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    it = 0
    while time.time() - t0 < 3.0:
        torch._int_mm(a, b)
        it += 1
        if it % 20 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / it
    ops = 2 * n ** 3
    out = {"int8_tops": round(ops / (best * 1e-3) / 1e12, 1),
           "int8_tops_sustained": round(ops / (sus * 1e-3) / 1e12, 1),
           "how": "torch._int_mm int8 8192^3 (2*N^3 ops), best of 10 (burst) and back to back 3 s",
           "gpu": torch.cuda.get_device_name()}
    print(json.dumps(out))
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
