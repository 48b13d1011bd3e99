"""A/B of the inverse-transform kernels on a 256^3 product whose output rows
are 32-byte aligned (lc = 4096) and one whose rows are not (lc = 4095).
usage: python tools/ab_inv.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1905_04356_b200 import _lib, dense  # noqa: E402

p = 2013265921


def run(la, lb, opt):
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randint(0, p, (256, 256, la), dtype=torch.int64, device="cuda", generator=g).to(torch.int32)
    B = torch.randint(0, p, (256, 256, lb), dtype=torch.int64, device="cuda", generator=g).to(torch.int32)
    _lib.set_option("ntt_mma_inv", 1 - opt)
    for _ in range(3):
        C = dense.pm_mul_dense(A, B, p)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        C = dense.pm_mul_dense(A, B, p)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 5, C


for la, lb in [(2049, 2048), (2048, 2048)]:
    t_mma, C1 = run(la, lb, 0)
    t_old, C2 = run(la, lb, 1)
    print(f"lc={la + lb - 1}: product ms  mma-inverse {t_mma:.3f}  shoup-inverse {t_old:.3f}  "
          f"equal={bool(torch.equal(C1, C2))}")
