#!/usr/bin/env python
"""Benchmark of the B200 F_p polynomial-matrix product path (driver contract).

Default workload: BASELINE.json configs[4] (cfg5), the largest single-GPU
config: A, B 256x256 over p = 2013265921, entries of degree < 2048, 4096
evaluation points, the 256^3 pointwise products on the int8 tensor cores.  A
step is one exact product C = A*B on device-resident inputs.  value =
algorithmic modular multiplications per second (SURVEY.md 8(d) convention)
for the whole job over all ranks; every rank runs its own product
(independent units, no data-path collective: weak scaling).

--impl reference times the multi-threaded CPU port of the reference path
(oracle/fpm_port.c, "port": the reference itself is pure Python, ~1.3 h per
cfg5 product on one core) on the host cores, on the same config and inputs
recipe, and prints the same config object.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P31 = 2013265921
P60 = (1 << 60) - 93
METRIC = "F_p polmat-mul ms & Gmodmul/s, % roofline (NTT HBM, pointwise MMA); PM-Basis ms"

CONFIGS = {
    "cfg1": dict(kind="mul", p=P31, m=4, k=4, n=4, deg=1023),
    "cfg2": dict(kind="mul", p=P31, m=32, k=32, n=32, deg=4095),
    "cfg3": dict(kind="mul", p=P60, m=16, k=16, n=16, deg=2047),
    "cfg4": dict(kind="pmbasis", p=P31, m=64, n=32, sigma=4096),
    "cfg5": dict(kind="mul", p=P31, m=256, k=256, n=256, deg=2047),
    # not a BASELINE config: the interpolant-basis row of SURVEY 8(f), cfg4's shape
    "ib4": dict(kind="intbasis", p=P31, m=64, n=32, sigma=4096),
}
CRT_PRIMES = [2130706433, 2113929217, 2013265921, 1811939329, 1711276033, 1224736769,
              1107296257]


def two_adicity(p):
    k, m = 0, p - 1
    while m % 2 == 0:
        m //= 2
        k += 1
    return k


def mul_plan(cfg):
    """N, number of word primes r (1 = direct) for a product config."""
    la = lb = cfg["deg"] + 1
    need = la + lb - 1
    logn = max(5, (need - 1).bit_length())
    p = cfg["p"]
    if p < (1 << 31) and two_adicity(p) >= logn:
        return 1 << logn, 1
    lg = (math.log2(cfg["k"]) + math.log2(min(la, lb)) + 2 * math.log2(p - 1) + 2)
    have, r = 0.0, 0
    for q in CRT_PRIMES:
        if have > lg:
            break
        have += math.log2(q)
        r += 1
    return 1 << logn, r


def mul_work(cfg):
    """Algorithmic modmuls and per-stage algorithmic bytes."""
    m, k, n = cfg["m"], cfg["k"], cfg["n"]
    la = lb = cfg["deg"] + 1
    lc = la + lb - 1
    N, r = mul_plan(cfg)
    logn = N.bit_length() - 1
    ntt = (N // 2) * logn
    modmul = r * ((m * k + k * n + m * n) * ntt + m * n * N + N * m * k * n)
    eb = 4 if cfg["p"] < (1 << 31) else 8
    bytes_ = {
        "ntt_fwd_A": r * m * k * (eb * la + 4 * N),
        "ntt_fwd_B": r * k * n * (eb * lb + 4 * N),
        "pointwise": r * 4 * N * (m * k + k * n + m * n),
        "ntt_inv": r * m * n * 4 * (N + lc),
    }
    bytes_["ntt_fwd_AB"] = bytes_["ntt_fwd_A"] + bytes_["ntt_fwd_B"]  # one launch for both
    if r > 1:
        bytes_["crt"] = m * n * lc * (4 * r + 8)
    return modmul, bytes_, N, r


def pmbasis_work(cfg):
    """Algorithmic modmul estimate of PM-Basis (tree ~13.9 G
    + base ~7.1 G at cfg4), scaled by sigma * m^2 * n / (4096 * 64^2 * 32)."""
    s = cfg["sigma"] / 4096.0 * (cfg["m"] / 64.0) ** 2 * (cfg["n"] / 32.0)
    return int(21.0e9 * s)


# ---------------------------------------------------------------------------
class Clocks:
    """SM clock / throttle-reason sampling during the timed region through NVML
    (nvidia_ml_py; the same counters `nvidia-smi --query-gpu=clocks.sm,
    clocks_event_reasons.*` reads), 2 ms period in a background thread."""

    BITS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
            "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
            "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
            "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index, period_ms=2.0):
        self.index = index
        self.period = period_ms * 1e-3
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self.ok = False
        self._stop = threading.Event()

    def start(self):
        try:
            import pynvml as N

            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception as exc:  # pragma: no cover
            self.err = f"{type(exc).__name__}: {exc}"
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                bits = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, attr in self.BITS.items():
                    if bits & getattr(N, attr):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": [getattr(self, "err", "nvml unavailable")]}
        self._stop.set()
        self.t.join(timeout=2)
        sm = sorted(self.samples)
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(sm), "source": f"NVML (nvidia_ml_py), {self.period * 1e3:g} ms period"}


def read_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


TRAFFIC_FILE = os.path.join("profiles", "r02_traffic.json")


def read_traffic():
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per stage of ONE
    product (tools/ncu_traffic.py: the launches of the last of two products
    under ncu), {config: {stage: bytes}}."""
    path = os.path.join(ROOT, TRAFFIC_FILE)
    try:
        with open(path) as f:
            return json.load(f).get("per_step", {})
    except Exception:
        return {}


def read_pipes():
    path = os.path.join(ROOT, "profiles", "ncu_pipes.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


# measured issue cost of the integer multiply forms on this B200
# (tools/micro/tput.cu: cycles per warp-instruction per SM sub-partition)
INT_RATES = {"imad": 2.0, "imad_hi": 4.45, "imad_wide": 4.0, "iadd": 1.0, "viaddmnmx": 2.0}


# ---------------------------------------------------------------------------
def read_int8_peak():
    """Measured int8 tensor-core peak (tools/int8_peak.py on this pool's B200:
    torch._int_mm 8192^3), TOPS.  The burst figure: the pointwise kernel runs
    ~1.7 ms inside a ~4.4 ms step, not back to back for seconds."""
    path = os.path.join(ROOT, "profiles", "int8_peak.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["int8_tops"]), "measured burst (profiles/int8_peak.json int8_tops)"
    except Exception:
        return 4500.0, "nominal dense int8 4.5 POPS"


def tc_ops(cfg):
    """(useful, issued) int8 ops of the tensor-core pointwise stage, mirroring
    the kernel choice in ops.cu cyclic_product; None when it runs on CUDA cores."""
    m, k, n = cfg["m"], cfg["k"], cfg["n"]
    N, r = mul_plan(cfg)
    pts = N * r
    useful = 2 * 16 * m * k * n * pts
    if m * k * n < 4096 or N > 8192:
        return None
    nch = -(-k // 32)

    def pow2(x, lo, hi):
        v = lo
        while v < x and v < hi:
            v *= 2
        return v

    if 16 < m <= 32:                       # tc_pq.cu
        nb = pow2(n, 8, 32)
        per = 2 * 128 * 4 * nb * 128 * nch * -(-n // nb)
    elif m > 32 and k % 4 == 0 and n % 4 == 0:   # tc_grouped.cu (M-tiled above 128)
        mp = pow2(m, 16, 128)
        nb = pow2(n, 8, min(mp, 64))
        per = 2 * 128 * 4 * nb * 128 * nch * -(-n // nb) * -(-m // 128)
    elif m >= 64 and k % 4 == 0 and 64 <= k <= 8192 and n >= 32:  # tc_pointwise.cu
        per = 2 * 256 * -(-m // 256) * 256 * -(-n // 64) * 128 * nch
    else:
        return None
    return useful, per * pts


def roofline_report(cfg, cfgname, avg, sbytes):
    """Roofline of the dominant kernel class (NTT = the forward and inverse
    transform launches, pointwise, CRT) plus a per-stage table.  Bytes are
    SURVEY.md 8(d)'s algorithmic per-stage bytes; `traffic` is ncu
    dram__bytes_read.sum + dram__bytes_write.sum of the same launches
    (profiles/ncu_traffic.json)."""
    hbm, hsrc = read_peaks()
    i8, i8src = read_int8_peak()
    traffic = read_traffic().get(cfgname, {})

    def tr(stage):
        v = traffic.get(stage)
        return None if v is None else int(v)

    table = {}
    for st, ms in avg.items():
        b = sbytes.get("pointwise" if st.startswith("pointwise") else st)
        if b is None:
            continue
        ach = b / (ms * 1e-3) / 1e9
        ent = {"ms": round(ms, 5), "bound": "hbm", "achieved": round(ach, 1), "peak": hbm,
               "unit": "GB/s", "frac": round(ach / hbm, 4), "algorithmic_bytes": b,
               "traffic": tr(st)}
        if st == "pointwise_tc":
            ops = tc_ops(cfg)
            if ops:
                ent["tensor"] = {"useful_tops": round(ops[0] / (ms * 1e-3) / 1e12, 1),
                                 "issued_tops": round(ops[1] / (ms * 1e-3) / 1e12, 1),
                                 "peak_tops": i8, "frac_issued": round(ops[1] / (ms * 1e-3) / 1e12 / i8, 4),
                                 "peak_source": i8src}
        table[st] = ent
    classes = {"ntt": [s for s in table if s.startswith("ntt")],
               "pointwise": [s for s in table if s.startswith("pointwise")],
               "crt": [s for s in table if s == "crt"]}
    dom = max(classes, key=lambda c: sum(avg[s] for s in classes[c]))
    members = classes[dom]
    ms = sum(avg[s] for s in members)
    b = sum(table[s]["algorithmic_bytes"] for s in members)
    trs = [table[s]["traffic"] for s in members]
    ach = b / (ms * 1e-3) / 1e9
    roof = {"kernel": dom, "launches": members, "bound": "hbm", "achieved": round(ach, 1),
            "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
            "traffic": sum(trs) if all(t is not None for t in trs) else None,
            "algorithmic_bytes": b, "ms": round(ms, 5), "peak_source": hsrc}
    if dom == "ntt":
        roof["note"] = ("HBM fraction per SURVEY 8(d).  The NTT kernels are bound by their "
                        "CUDA-core instruction stream, not HBM: the 4096-point forward runs as "
                        "two radix-64 passes on the int8 tensor cores (ntt_mma64.cu) and is "
                        "limited by the limb fold + twiddle epilogue and the TMA store of the "
                        "32-byte point rows; the inverse (Shoup butterflies) by the heavy FMA "
                        "pipe; `compute` gives ncu pipe/issue utilisation, DESIGN.md 4")
        pipes = read_pipes().get(cfgname, {})
        comp = {}
        for st in ("ntt_fwd", "ntt_inv"):
            ent = pipes.get(st)
            if ent:
                e = ent[0]
                comp[st] = {"kernel": e["kernel"], "fmaheavy_util_elapsed": e["fmaheavy_pct_elapsed"],
                            "alu_util_elapsed": e["alu_pct_elapsed"],
                            "issue_util_active": e["issue_pct_active"]}
        if comp:
            roof["compute"] = {"pipe": "fmaheavy (IMAD.HI / IMAD: Shoup twiddles, limb folds)",
                               "per_kernel": comp,
                               "int_rates_cycles_per_warp_op": INT_RATES,
                               "source": "profiles/ncu_pipes.json (ncu --set full), "
                                         "tools/micro/tput.cu"}
    if dom == "pointwise" and "pointwise_tc" in table and "tensor" in table["pointwise_tc"]:
        t = table["pointwise_tc"]["tensor"]
        roof.update({"bound": "tensor", "achieved": t["issued_tops"], "peak": i8,
                     "unit": "TFLOP/s", "frac": t["frac_issued"], "peak_source": i8src,
                     "note": "int8 ops issued (incl. grouping padding) / measured int8 peak"})
    return roof, table


def make_inputs(cfg, device, seed):
    import torch

    from paper_1905_04356_b200 import dense

    g = torch.Generator(device=device).manual_seed(seed)
    p = cfg["p"]
    dt = dense.torch_dtype(p)

    def rnd(shape):
        if p < (1 << 31):
            return torch.randint(0, p, shape, generator=g, device=device, dtype=torch.int64).to(dt)
        hi = torch.randint(0, 1 << 30, shape, generator=g, device=device, dtype=torch.int64)
        lo = torch.randint(0, 1 << 30, shape, generator=g, device=device, dtype=torch.int64)
        return ((hi << 30) | lo) % p

    if cfg["kind"] == "mul":
        L = cfg["deg"] + 1
        return rnd((cfg["m"], cfg["k"], L)), rnd((cfg["k"], cfg["n"], L))
    if cfg["kind"] == "intbasis":
        # sigma constant m x n matrices at a geometric progression of points
        import random as _r

        rr = _r.Random(seed)
        a0, ratio = rr.randrange(1, p), rr.randrange(2, p)
        pts, cur = [], a0
        for _ in range(cfg["sigma"]):
            pts.append(cur)
            cur = cur * ratio % p
        return rnd((cfg["sigma"], cfg["m"], cfg["n"])), pts
    return (rnd((cfg["m"], cfg["n"], cfg["sigma"])),)


def run_step(cfg, inputs, out=None):
    from paper_1905_04356_b200 import dense

    if cfg["kind"] == "mul":
        return dense.pm_mul_dense(inputs[0], inputs[1], cfg["p"], out=out)
    if cfg["kind"] == "intbasis":
        return dense.intbasis_dense(inputs[0], inputs[1], [0] * cfg["m"], cfg["p"])[0]
    return dense.pmbasis_dense(inputs[0], cfg["sigma"], [0] * cfg["m"], cfg["p"])[0]


def time_steps(cfg, inputs, steps, warmup, flush, profile_h=None, step=None):
    """Per-step CUDA-event time (ms list) with an L2 flush between steps.
    step(cfg, inputs, out) defaults to one whole product / basis."""
    import torch

    from paper_1905_04356_b200 import _lib

    run_step_ = step or run_step
    out = None
    if cfg["kind"] == "mul" and step is None:
        out = run_step(cfg, inputs)
    for _ in range(warmup):
        run_step_(cfg, inputs, out)
    torch.cuda.synchronize()
    times = []
    stages = {}
    n0 = _lib.launch_count()
    for _ in range(steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        run_step_(cfg, inputs, out)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    launches = (_lib.launch_count() - n0) // max(steps, 1) * steps
    if profile_h is not None:
        # per-stage CUDA events on separate, untimed steps (the events would
        # otherwise add to the timed region)
        for _ in range(min(steps, 3)):
            flush.zero_()
            _lib.profile(profile_h, True)
            run_step_(cfg, inputs, out)
            torch.cuda.synchronize()
            for name, ms in _lib.profile_records(profile_h):
                stages.setdefault(name, []).append(ms)
        _lib.profile(profile_h, False)
    return times, stages, launches


def e2e_mul(cfg, steps, warmup, seed, rank=0, world=1):
    """Same metric through the C ABI host entry (pinned host buffers): every
    call uploads A and B and downloads C inside the timed region.  On N > 1
    ranks each rank runs its 2-D block (A row block x B column block)."""
    import torch

    from paper_1905_04356_b200 import _lib, dense
    from paper_1905_04356_b200.parallel import block_of

    p = cfg["p"]
    A, B = make_inputs(cfg, "cuda", seed)
    (r0, r1), (c0, c1) = block_of(rank, world, A.shape[0], B.shape[1])
    Ah = A[r0:r1].contiguous().cpu().pin_memory()
    Bh = B[:, c0:c1].contiguous().cpu().pin_memory()
    del A, B
    m, k, la = Ah.shape
    _, n, lb = Bh.shape
    lc = la + lb - 1
    Ch = torch.empty((m, n, lc), dtype=Ah.dtype).pin_memory()
    h = _lib.context()
    L = _lib.lib()
    eb = dense.elem_bytes_for(p)

    def call():
        _lib.check(L.fpm_polmat_mul_host(h, p, eb, Ah.data_ptr(), m, k, la, Bh.data_ptr(), n,
                                         lb, Ch.data_ptr()), "fpm_polmat_mul_host")

    for _ in range(warmup):
        call()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2], Ah.numel() * eb + Bh.numel() * eb, Ch.numel() * eb


def e2e_pmbasis(cfg, steps, seed):
    """cfg4 through fpm_pmbasis_host (the entry INTEGRATION.md binds for
    appint.pmbasis): F uploaded and P downloaded inside the timed region."""
    import ctypes

    import torch

    from paper_1905_04356_b200 import _lib, dense

    p, m, n, sigma = cfg["p"], cfg["m"], cfg["n"], cfg["sigma"]
    (F,) = make_inputs(cfg, "cuda", seed)
    Fh = F.cpu().pin_memory()
    del F
    Ph = torch.empty((m, m, sigma + 1), dtype=Fh.dtype).pin_memory()
    s_arr = (ctypes.c_int64 * m)(*([0] * m))
    lp = ctypes.c_int(0)
    rd = (ctypes.c_int64 * m)()
    h = _lib.context()
    L = _lib.lib()
    eb = dense.elem_bytes_for(p)

    def call():
        _lib.check(L.fpm_pmbasis_host(h, p, eb, Fh.data_ptr(), m, n, sigma, sigma, s_arr,
                                      Ph.data_ptr(), ctypes.byref(lp), rd), "fpm_pmbasis_host")

    call()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2], Fh.numel() * eb, Ph.numel() * eb


def cpu_info():
    """Host CPU model and the threads the CPU legs use (lscpu's model name)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    if model is None:
        try:
            with open("/proc/cpuinfo") as f:
                for line in f:
                    if line.startswith("model name"):
                        model = line.split(":", 1)[1].strip()
                        break
        except Exception:
            model = "unknown"
    return {"model": model, "threads": os.cpu_count() or 1}


def port_inputs(cfg, seed):
    import numpy as np

    p = cfg["p"]
    L = cfg["deg"] + 1
    rng = np.random.default_rng(seed)
    dt = np.uint32 if p < (1 << 32) else np.uint64
    A = rng.integers(0, p, size=(cfg["m"], cfg["k"], L), dtype=np.uint64).astype(dt)
    B = rng.integers(0, p, size=(cfg["k"], cfg["n"], L), dtype=np.uint64).astype(dt)
    return A, B


def port_step(cfg, A, B, threads, out=None):
    """One full product by the CPU port: fpm_port.c for 31-bit NTT primes,
    the restatement fpm_oracle.c (multi-prime-free NTT / schoolbook) else."""
    from oracle import oracle as O

    p = cfg["p"]
    N, r = mul_plan(cfg)
    if r == 1:
        return O.port_mul31(p, A, B, threads=threads, out=out), "oracle/fpm_port.c"
    O.set_threads(threads)
    return O.pm_mul(p, A, B), "oracle/fpm_oracle.c"


def cpu_baseline(cfg, budget_s=20.0, threads=None):
    """The CPU port of the reference path on the host cores, a bounded sample
    of the same workload: full products until ~budget_s of CPU work."""
    threads = threads or os.cpu_count() or 1
    if cfg["kind"] != "mul":
        raise ValueError("cpu baseline only for product configs")
    A, B = port_inputs(cfg, 1)
    work = mul_work(cfg)[0]
    out, src = port_step(cfg, A, B, threads)
    t0 = time.perf_counter()
    reps = 0
    while True:
        port_step(cfg, A, B, threads, out=out if src.endswith("port.c") else None)
        reps += 1
        if time.perf_counter() - t0 > budget_s or reps >= 5:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": work / dt / 1e9, "unit": "Gmodmul/s", "cores": threads, "kind": "port",
            "seconds_per_step": dt, "cpu": cpu_info(),
            "sample": f"{reps} full {cfg['m']}x{cfg['k']}x{cfg['n']} deg<{cfg['deg'] + 1} "
                      f"products ({src}, OpenMP {threads} threads) after one untimed product"}


def bench_config(args, cfg, world):
    """The config object both arms print (identical keys and values)."""
    c = {"workload": args.config, **{k: v for k, v in cfg.items() if k != "kind"}}
    if cfg["kind"] == "mul":
        N, r = mul_plan(cfg)
        c.update({"N": N, "word_primes": r})
    c["l2"] = "flushed: 256 MiB write between timed steps (outside events); inputs > L2"
    c["parallelism"] = parallelism(cfg, world)
    return c


def split_mode(cfg, world):
    """How a product shards over `world` GPUs: 'prime' for a
    multi-prime product (one word prime per rank, residues gathered to rank
    0 for the CRT), '2d' for a direct one (A-row x B-column blocks, C stays
    sharded), None on one GPU or for PM-Basis (replicas only)."""
    if world <= 1 or cfg["kind"] != "mul":
        return None
    return "prime" if mul_plan(cfg)[1] > 1 else "2d"


def parallelism(cfg, world):
    mode = split_mode(cfg, world)
    if mode is None:
        return "single GPU" if world <= 1 else f"replicas x{world} (one instance per rank)"
    if mode == "prime":
        return (f"prime split x{world}: word primes round-robin over ranks, residues gathered "
                "(NCCL) to rank 0 for the CRT; one product per step (strong scaling)")
    from paper_1905_04356_b200.parallel import grid_shape

    gr, gc = grid_shape(world)
    return (f"2-D blocks {gr}x{gc}: rank (i, j) multiplies A row block i by B column block j, "
            "no collective, C stays sharded; one product per step (strong scaling)")


def scaling_of(cfg, world):
    return "strong" if split_mode(cfg, world) else "weak"


def reference_arm(args, cfg, rank, world):
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    if cfg["kind"] != "mul":
        return {"impl": "reference", "unavailable": "the reference arm times products only"}
    A, B = port_inputs(cfg, 1)
    out, src = port_step(cfg, A, B, threads)
    for _ in range(max(0, min(args.warmup, 1) - 1)):
        port_step(cfg, A, B, threads, out=out if src.endswith("port.c") else None)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        port_step(cfg, A, B, threads, out=out if src.endswith("port.c") else None)
        ts.append(time.perf_counter() - t0)
    total = sum(ts)
    work = mul_work(cfg)[0]
    val = work * args.steps / total / 1e9
    line = {
        "metric": METRIC, "value": round(val, 4), "unit": "Gmodmul/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
        "scaling": scaling_of(cfg, world), "vs_baseline": None,
        "dtype": "u32" if cfg["p"] < (1 << 31) else "u64",
        "data": "synthetic (seeded uniform coefficients in [0,p), numpy PCG64)",
        "config": bench_config(args, cfg, world),
        "cpu_baseline": {"value": round(val, 4), "unit": "Gmodmul/s", "cores": threads,
                         "kind": "port", "cpu": cpu_info(),
                         "sample": f"{args.steps} full products per run, one per step, after "
                                   f"one untimed warm-up product ({src}: multi-threaded CPU "
                                   "port of polmat._pm_mul_ntt, polmat.py:290-308; the "
                                   "reference is pure Python)"},
        "e2e": {"value": round(val, 4), "unit": "Gmodmul/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    return line


def pmbasis_split(cfg, device, seed):
    """cfg4 stage split from the library's per-stage CUDA events (untimed
    run): leaf (M-Basis steps + basis build) and tree (products, middle
    products, shifts)."""
    import torch

    from paper_1905_04356_b200 import _lib

    h = _lib.context()
    inputs = make_inputs(cfg, device, seed)
    run_step(cfg, inputs)
    torch.cuda.synchronize()
    _lib.profile(h, True)
    run_step(cfg, inputs)
    torch.cuda.synchronize()
    recs = _lib.profile_records(h)
    _lib.profile(h, False)
    leaf = sum(ms for nm, ms in recs if nm.startswith("mbasis"))
    steps_ms = sum(ms for nm, ms in recs if nm == "mbasis_steps")
    tot = sum(ms for _, ms in recs)
    return {"leaf_ms": round(leaf, 3), "leaf_steps_ms": round(steps_ms, 3),
            "tree_ms": round(tot - leaf, 3), "stage_sum_ms": round(tot, 3),
            "leaf_share": round(leaf / tot, 4) if tot else None,
            "order1_steps": cfg["sigma"],
            "leaf_steps_per_s": round(cfg["sigma"] / (leaf * 1e-3), 1) if leaf else None,
            "note": "per-stage CUDA events around every launch (serialises the PDL overlap, "
                    "so the stage sum exceeds the end-to-end time); leaf = mbasis_steps + "
                    "mbasis_build, tree = every product / middle product / shift stage"}


def per_config_table(device):
    """Short timing of every BASELINE config (ms, Gmodmul/s) for the report."""
    import torch

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    out = {}
    for name, cfg in CONFIGS.items():
        try:
            inputs = make_inputs(cfg, device, 100 + int(name[-1]))
            steps, warm = (3, 1) if cfg["kind"] in ("pmbasis", "intbasis") else (10, 3)
            ts, _, _ = time_steps(cfg, inputs, steps, warm, flush)
            ts.sort()
            ms = ts[len(ts) // 2]
            del inputs
            if cfg["kind"] == "intbasis":
                out[name] = {"ms": round(ms, 4), "note": "PM-IntBasis (SURVEY 8(f) rank 2), "
                             "not a BASELINE config"}
                continue
            work = mul_work(cfg)[0] if cfg["kind"] == "mul" else pmbasis_work(cfg)
            out[name] = {"ms": round(ms, 4), "Gmodmul_s": round(work / ms / 1e6, 2)}
            if cfg["kind"] == "pmbasis":
                out[name]["split"] = pmbasis_split(cfg, device, 104)
                med, bi, bo = e2e_pmbasis(cfg, 3, 104)
                out[name]["e2e"] = {"ms": round(med * 1e3, 3), "h2d_bytes": bi, "d2h_bytes": bo,
                                    "path": "fpm_pmbasis_host (C ABI, pinned host buffers)"}
        except Exception as exc:  # report, never hide
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", choices=sorted(CONFIGS))
    ap.add_argument("--clock-period-ms", type=float, default=2.0,
                    help="NVML clock / throttle-reason sampling period during the timed steps")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip cpu_baseline / e2e / per-config table")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        line = reference_arm(args, cfg, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    import torch

    # one rank per GPU; FPM_BENCH_SMOKE_BACKEND=gloo (functional smoke test of
    # the N > 1 path on a box with fewer GPUs than ranks, never a measurement)
    # lets ranks share a device: the split has no data-path collective
    smoke_backend = os.environ.get("FPM_BENCH_SMOKE_BACKEND")
    if smoke_backend:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if smoke_backend:
            dist.init_process_group(smoke_backend)
        else:
            dist.init_process_group("nccl", device_id=device)

    from paper_1905_04356_b200 import _lib

    h = _lib.context(local)
    mode = split_mode(cfg, world)
    # replicas: every rank its own inputs; a split product: the same inputs
    inputs = make_inputs(cfg, device, 1000 + (0 if mode else rank))
    step = None
    if mode == "2d":
        # each rank holds its own row block of A and column block of B (sliced
        # once, outside the timed steps) and writes its block of C in place
        from paper_1905_04356_b200 import dense
        from paper_1905_04356_b200.parallel import block_of

        (r0, r1), (c0, c1) = block_of(rank, world, inputs[0].shape[0], inputs[1].shape[1])
        inputs = (inputs[0][r0:r1].contiguous(), inputs[1][:, c0:c1].contiguous())
        torch.cuda.empty_cache()
        block_out = torch.empty((r1 - r0, c1 - c0, inputs[0].shape[2] + inputs[1].shape[2] - 1),
                                dtype=inputs[0].dtype, device=device)

        def step(cfg_, inp, out):
            return dense.pm_mul_dense(inp[0], inp[1], cfg_["p"], out=block_out)
    elif mode == "prime":
        from paper_1905_04356_b200.parallel import pm_mul_prime_split

        def step(cfg_, inp, out):
            return pm_mul_prime_split(inp[0], inp[1], cfg_["p"], dst=0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)  # > 126 MB L2
    clocks = Clocks(local, args.clock_period_ms)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    times, stages, launches = time_steps(cfg, inputs, args.steps, args.warmup, flush,
                                         profile_h=h, step=step)
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = sum(times)
    if dist is not None:
        t = torch.tensor([total_ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_step = total_ms / args.steps
    if cfg["kind"] == "mul":
        work, sbytes, N, r = mul_work(cfg)
    else:
        work, sbytes, N, r = pmbasis_work(cfg), {}, None, None
    # replicas: every rank did a whole unit; a split product: one unit per step
    units = 1 if mode else world
    value = units * work * args.steps / (total_ms * 1e-3) / 1e9

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Gmodmul/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": scaling_of(cfg, world), "vs_baseline": None,
        "dtype": "u32" if cfg["p"] < (1 << 31) else "u64",
        "data": "synthetic (seeded uniform coefficients in [0,p), torch.Generator)",
        "config": bench_config(args, cfg, world),
        "gpu_launches": launches,
        "clocks": clk,
    }
    if mode == "2d" and not args.no_extras and not smoke_backend:
        # the optional exchange: one all_gather of the C blocks (NCCL) for a
        # consumer that needs all of C on every rank (not in the timed steps)
        from paper_1905_04356_b200.parallel import gather_blocks

        Cb = step(cfg, inputs, None)
        torch.cuda.synchronize()
        dist.barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record()
        C = gather_blocks(Cb, cfg["m"], cfg["n"])
        g1.record()
        g1.synchronize()
        gms = torch.tensor([g0.elapsed_time(g1)], device=device)
        dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        line["exchange"] = {"kind": "all_gather of the C blocks (NCCL), once after the timed "
                                    "steps", "ms": round(float(gms.item()), 4),
                            "bytes_per_rank_sent": Cb.numel() * Cb.element_size(),
                            "bytes_per_rank_received": C.numel() * C.element_size()}
        del C, Cb
    del inputs
    # roofline of the dominant kernel class, CUDA events inside the timed region
    if stages:
        avg = {k: sum(v) / len(v) for k, v in stages.items()}
        line["stages_ms"] = {k: round(v, 5) for k, v in avg.items()}
        if cfg["kind"] == "mul":
            line["roofline"], line["roofline_stages"] = roofline_report(cfg, args.config, avg,
                                                                        sbytes)
            line["roofline"]["traffic_source"] = TRAFFIC_FILE
    if not args.no_extras and cfg["kind"] == "mul":
        # every rank runs its own host-buffer product (weak scaling, as the
        # device-timed value); the slowest rank's median sets the job time
        err = None
        try:
            med, bi, bo = e2e_mul(cfg, max(3, min(args.steps, 10)), 2, 7 + (0 if mode else rank),
                                  rank if mode else 0, world if mode else 1)
        except Exception as exc:
            med, bi, bo, err = float("inf"), 0, 0, f"{type(exc).__name__}: {exc}"
        if dist is not None:
            t = torch.tensor([med], device=device, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            med = float(t.item())
        if dist is not None:
            tb = torch.tensor([bi, bo], device=device, dtype=torch.float64)
            dist.all_reduce(tb)
            bi, bo = int(tb[0].item()), int(tb[1].item())
        if err is None and math.isfinite(med):
            line["e2e"] = {"value": round(units * work / med / 1e9, 3), "unit": "Gmodmul/s",
                           "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
                           "ms_per_step": round(med * 1e3, 4), "n_gpus": world,
                           "path": "fpm_polmat_mul_host (C ABI, pinned host buffers); "
                                   + ("each rank its 2-D block of one product"
                                      if mode else "one product per rank")
                                   + ", max over ranks"}
        else:
            line["e2e"] = {"error": err or "a rank failed its host-buffer product"}
    if rank == 0 and not args.no_extras and cfg["kind"] == "mul" and world == 1:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg)
        except Exception as exc:
            line["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"}
        line["per_config"] = per_config_table(device)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
