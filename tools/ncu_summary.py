"""Summarise ncu output for profiles/ (run here, on the files gpurun brought back).

  python tools/ncu_summary.py launches FILE.csv            -> per-kernel share table
  python tools/ncu_summary.py full FILE.ncu-rep [KEY]      -> key metrics per launch (JSON)

`full` also merges dram bytes per kernel into profiles/ncu_traffic.json under KEY
(the bench workload name), which bench.py reports as roofline.traffic.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum",  # reported in us
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    # the integer multiply path: IMAD.HI / IMAD.WIDE issue at a quarter of the
    # IMAD rate on the heavy FMA pipe (tools/micro/tput.cu)
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_selected",
    "smsp__pcsamp_warps_issue_stalled_not_selected",
    "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
]

STAGE_OF = {"ntt_fwd": "ntt_fwd", "ntt_mma_kernel<0>": "ntt_fwd", "ntt_mma64_kernel": "ntt_fwd", "ntt_mma_kernel<1>": "ntt_inv",
            "ntt_inv": "ntt_inv", "pointwise_cc": "pointwise", "tc_pair": "pointwise_tc",
            "tc_pointwise": "pointwise_tc", "tc_grouped": "pointwise_tc", "tc_pq": "pointwise_tc",
            "crt_kernel": "crt"}


def short(name):
    base = name.split("(")[0]
    return base.replace("void ", "").replace("fpm::<unnamed>::", "")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d.get("Metric Unit"), 1.0)
        k = short(d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", "")) * scale
        agg.setdefault(k, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    own = sum(sum(v) for k, v in agg.items() if not k.startswith("at::"))
    lines = ["| kernel | launches | mean us | share of own-kernel time |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = "" if k.startswith("at::") else f"{100 * sum(v) / own:.1f}%"
        lines.append(f"| `{k[:70]}` | {len(v)} | {sum(v) / len(v):.1f} | {share} |")
    print("\n".join(lines))
    print(f"\nown kernels total {own:.1f} us over the capture (all {tot:.1f} us)")


def full(path, key=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          ",".join(METRICS)], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": short(d["Kernel Name"])}
        for m in METRICS:
            if m in d and d[m] != "":
                u = units[hdr.index(m)]
                v = float(d[m].replace(",", ""))
                if u == "Kbyte":
                    v *= 1e3
                elif u == "Mbyte":
                    v *= 1e6
                elif u == "Gbyte":
                    v *= 1e9
                elif u in ("nsecond", "ns"):
                    v *= 1e-3
                elif u in ("msecond", "ms"):
                    v *= 1e3
                rec[m] = v
        res.append(rec)
    print(json.dumps(res, indent=1))
    if key:
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        cur = json.load(open(tp)) if os.path.exists(tp) else {}
        ent = cur[key] = {}  # replaced by this capture
        for rec in res:
            stage = next((v for k, v in STAGE_OF.items() if k in rec["kernel"]), None)
            if stage and "dram__bytes_read.sum" in rec:
                b = rec["dram__bytes_read.sum"] + rec.get("dram__bytes_write.sum", 0.0)
                ent.setdefault(stage, []).append(b)
        json.dump(cur, open(tp, "w"), indent=1)
        pp = os.path.join(ROOT, "profiles", "ncu_pipes.json")
        cur = json.load(open(pp)) if os.path.exists(pp) else {}
        ent = cur[key] = {}
        for rec in res:
            stage = next((v for k, v in STAGE_OF.items() if k in rec["kernel"]), None)
            if not stage:
                continue
            ent.setdefault(stage, []).append({
                "kernel": rec["kernel"],
                "us": rec.get("gpu__time_duration.sum"),
                "fmaheavy_pct_elapsed": rec.get(
                    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                "alu_pct_elapsed": rec.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                "issue_pct_elapsed": rec.get("smsp__issue_active.avg.pct_of_peak_sustained_elapsed"),
                "issue_pct_active": rec.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            })
        json.dump(cur, open(pp, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
