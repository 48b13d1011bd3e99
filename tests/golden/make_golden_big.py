"""Generate full-size golden checksums by running the UNMODIFIED reference
(`fpmat`, /root/reference/pkg/src) in this build container.

Test infrastructure only: the GPU box never runs this (the reference is not
shipped); it consumes the committed JSON written here.

Recipe: rng = random.Random(seed); inputs drawn with
fpmat.polmat.random_polmat (polmat.py:650-659) in the order A then B (or F);
checksum = sha256(polmat_to_text(out)).hexdigest()[:16] (polmat.py:617-623).

usage: python tests/golden/make_golden_big.py KIND ARGS...
  mul  SEED P M K N DEG        -> pm_mul(A, B)
  pmb  SEED P M N SIGMA        -> pmbasis(F, SIGMA, [0]*M)
"""
import hashlib
import json
import os
import random
import sys
import time

sys.dont_write_bytecode = True
sys.path.insert(0, os.environ.get("FPMAT_REF", "/root/reference/pkg/src"))
from fpmat.modring import field_new  # noqa: E402
from fpmat.polmat import pm_mul, polmat_to_text, random_polmat  # noqa: E402
from fpmat.appint import pmbasis  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    kind = sys.argv[1]
    args = [int(a) for a in sys.argv[2:]]
    if kind == "mul":
        seed, p, m, k, n, deg = args
        ctx = field_new(p)
        rng = random.Random(seed)
        A = random_polmat(ctx, m, k, deg, rng)
        B = random_polmat(ctx, k, n, deg, rng)
        t0 = time.perf_counter()
        C = pm_mul(A, B)
        dt = time.perf_counter() - t0
        key = f"mul_s{seed}_p{p}_{m}x{k}x{n}_d{deg}"
        out = C
    elif kind == "pmb":
        seed, p, m, n, sigma = args
        ctx = field_new(p)
        rng = random.Random(seed)
        F = random_polmat(ctx, m, n, sigma - 1, rng)
        t0 = time.perf_counter()
        out = pmbasis(F, sigma, [0] * m)
        dt = time.perf_counter() - t0
        key = f"pmb_s{seed}_p{p}_{m}x{n}_o{sigma}"
    else:
        raise SystemExit(f"unknown kind {kind}")
    txt = polmat_to_text(out)
    rec = {
        "key": key,
        "sha16": hashlib.sha256(txt.encode()).hexdigest()[:16],
        "degree": out.degree,
        "ref_seconds": round(dt, 2),
        "cores": 1,
    }
    # degree profile (per-entry lengths) is cheap and pins structure
    rec["row_lengths_sum"] = sum(len(e) for r in out.rows for e in r)
    path = os.path.join(HERE, "big_goldens.jsonl")
    with open(path, "a") as f:
        f.write(json.dumps(rec) + "\n")
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
