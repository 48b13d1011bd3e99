"""DRAM traffic per stage of ONE product, for bench.py's roofline.traffic.

On the GPU box, under ncu (one warm-up product, then the measured one):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/traffic_CFG.csv \
      python tools/ncu_traffic.py run CFG
Here, on the CSV it brought back:
  python tools/ncu_traffic.py parse gpurun_out/traffic_CFG.csv CFG
which merges {stage: bytes} of the second product's launches into
profiles/r02_traffic.json (stage names as the library's profiler reports
them: ntt_fwd_AB / ntt_fwd_A / ntt_fwd_B, pointwise_tc / pointwise, ntt_inv,
crt, widen, split_reduce).
"""
import collections
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "r02_traffic.json")


def run(name):
    sys.path.insert(0, ROOT)
    import torch

    import bench

    cfg = bench.CONFIGS[name]
    inputs = bench.make_inputs(cfg, "cuda", 11)
    torch.cuda.synchronize()
    from paper_1905_04356_b200 import _lib

    marks = []
    for _ in range(2):
        n0 = _lib.launch_count()
        bench.run_step(cfg, inputs)
        torch.cuda.synchronize()
        marks.append(_lib.launch_count() - n0)
    print("launches per product:", marks)


def stage_of(kernel, fwd_seen):
    k = kernel
    if "ntt_fwd" in k or "ntt_mma_kernel<0>" in k or "ntt_mma_fwd" in k or "ntt_mma64" in k:
        return "ntt_fwd"
    if "ntt_mma_kernel<1>" in k:
        return "ntt_inv"
    if "ntt_inv" in k:
        return "ntt_inv"
    if "tc_pq" in k or "tc_grouped" in k or "tc_pointwise" in k or "tc_pair" in k:
        return "pointwise_tc"
    if "pointwise_cc" in k:
        return "pointwise"
    if "crt_kernel" in k:
        return "crt"
    if "widen" in k:
        return "widen"
    if "split_reduce" in k:
        return "split_reduce"
    if "zero_tail" in k:
        return "zero_tail"
    return k.split("(")[0][:40]


def parse(path, name):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    per = collections.OrderedDict()
    for r in rows:
        kid = int(r["ID"])
        d = per.setdefault(kid, {"kernel": r["Kernel Name"]})
        val = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        if r["Metric Name"].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d["bytes"] = d.get("bytes", 0) + val * scale
        elif r["Metric Name"] == "gpu__time_duration.sum":
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3,
                     "ms": 1e3}.get(unit, 1e-3)
            d["us"] = val * scale
    # own kernels only (input generation runs torch kernels); two identical
    # products were captured: keep the second half of the launches
    ids = [i for i in per if "fpm::" in per[i]["kernel"]]
    half = ids[len(ids) // 2:]
    launches = [per[i] for i in half]
    stages = collections.OrderedDict()
    fwd = [x for x in launches if stage_of(x["kernel"], 0) == "ntt_fwd"]
    for x in launches:
        st = stage_of(x["kernel"], 0)
        if st == "ntt_fwd":
            st = "ntt_fwd_AB" if len(fwd) == 1 else ("ntt_fwd_A" if x is fwd[0] else "ntt_fwd_B")
        stages[st] = stages.get(st, 0) + int(round(x.get("bytes", 0)))
    db = json.load(open(OUT)) if os.path.exists(OUT) else {"per_step": {}, "launches": {}}
    db["per_step"][name] = stages
    db["launches"][name] = [{"kernel": x["kernel"].split("(")[0][:80],
                             "us": round(x.get("us", 0), 2),
                             "dram_bytes": int(round(x.get("bytes", 0)))} for x in launches]
    db["how"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                 "gpu__time_duration.sum --clock-control none of two identical products "
                 "(tools/ncu_traffic.py run CFG); the second product's launches")
    with open(OUT, "w") as f:
        json.dump(db, f, indent=1)
    print(name, dict(stages))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        parse(sys.argv[2], sys.argv[3])
