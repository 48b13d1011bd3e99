"""Kernel-time census of one configuration under torch.profiler (CUPTI):
sum of device kernel durations by name vs the wall time of the same step.

usage: python tools/kprof.py CFG [sigma]
"""
import collections
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    name = sys.argv[1]
    cfg = dict(bench.CONFIGS[name])
    if len(sys.argv) > 2:
        cfg["sigma"] = int(sys.argv[2])
    inputs = bench.make_inputs(cfg, "cuda", 11)
    for _ in range(2):
        bench.run_step(cfg, inputs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bench.run_step(cfg, inputs)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        bench.run_step(cfg, inputs)
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    first, last = None, None
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            k = ev.name.replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "")[:60]
            agg[k][0] += 1
            agg[k][1] += ev.device_time_total / 1e3
    tot = sum(v[1] for v in agg.values())
    n = sum(v[0] for v in agg.values())
    print(f"{name}: wall {wall:.2f} ms, kernels {n}, kernel time sum {tot:.2f} ms "
          f"({100 * tot / wall:.0f}% of wall)")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
        print(f"  {t:9.3f} ms {c:6d} x {1e3 * t / c:8.1f} us  {k}")


if __name__ == "__main__":
    main()
