"""PCIe copy rates with pinned host memory: H2D alone, D2H alone, both at once."""
import time

import torch


def main():
    n = 32 << 20  # bytes
    h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        d1.copy_(h1, non_blocking=True)
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()

    def timeit(fn, reps=10):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return sorted(ts)[len(ts) // 2]

    def h2d():
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    def both():
        h2d()
        d2h()

    for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both)]:
        t = timeit(fn)
        print(f"{name}: {t * 1e3:.3f} ms  {n / t / 1e9:.1f} GB/s per direction")


if __name__ == "__main__":
    main()
