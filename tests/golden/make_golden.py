"""Generate the small golden fixtures (tests/golden/small.json) by running the
UNMODIFIED reference `fpmat` (/root/reference/pkg/src) in the build container.

Test infrastructure only.  The reference does not travel to the GPU box; the
committed JSON does.  Re-run with:  python tests/golden/make_golden.py

Every case stores its inputs and the reference's output as PolMat row lists
(trimmed coefficient lists, low degree first, polmat.py:48-58).
"""
import json
import os
import random
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, os.environ.get("FPMAT_REF", "/root/reference/pkg/src"))

from fpmat import config  # noqa: E402
from fpmat.appint import _mbasis1_struct, mbasis, mbasis1, pmbasis  # noqa: E402
from fpmat.forms import is_owp, rdeg  # noqa: E402
from fpmat.modring import NttPlan, field_new, ntt_forward, ntt_inverse  # noqa: E402
from fpmat.polmat import (  # noqa: E402
    PolMat,
    _pm_middle,
    applicable_strategies,
    pm_middle_product,
    pm_mul,
    random_polmat,
)
from fpmat.upoly import _trim  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
P31 = 2013265921
P60NTT = 1152921493869428737
P60 = (1 << 60) - 93
PRIMES = [97, 65537, 786433, P31, 1811939329, 2113929217, 1711276033, 1107296257,
          P60NTT, P60, 3, 5]


def rand_polmat_ragged(ctx, m, n, maxdeg, rng, pzero=0.15):
    """Entries with independent random lengths, some zero."""
    rows = []
    for _ in range(m):
        row = []
        for _ in range(n):
            if rng.random() < pzero:
                row.append([])
            else:
                L = rng.randint(1, maxdeg + 1)
                row.append(_trim([rng.randrange(ctx.p) for _ in range(L)]))
        rows.append(row)
    return PolMat(ctx, rows, ncols=n)


def rows_of(M):
    return [[list(e) for e in r] for r in M.rows]


def main():
    out = {"primes": [], "ntt": [], "mul": [], "middle": [], "mbasis1": [], "mbasis": [],
           "pmbasis": []}
    rng = random.Random(20260101)

    for p in PRIMES:
        ctx = field_new(p)
        out["primes"].append({"p": p, "two_adicity": ctx.two_adicity, "ntt_root": ctx.ntt_root})

    # NTT vectors (modring.py:272-286); SPEC S:55 example and random ones
    ctx97 = field_new(97)
    plan = NttPlan(ctx97, 2)
    out["ntt"].append({"p": 97, "v": [0, 1, 0, 0], "fwd": ntt_forward(plan, [0, 1, 0, 0]),
                       "inv": ntt_inverse(plan, [0, 1, 0, 0])})
    for p, logs in ((P31, range(1, 14)), (786433, (3, 6, 10)), (P60NTT, (2, 5, 8)),
                    (1811939329, (4, 9)), (1107296257, (7,)), (97, (1, 3, 5))):
        ctx = field_new(p)
        for lg in logs:
            plan = NttPlan(ctx, lg)
            v = [rng.randrange(p) for _ in range(1 << lg)]
            out["ntt"].append({"p": p, "v": v, "fwd": ntt_forward(plan, v),
                               "inv": ntt_inverse(plan, v)})

    # pm_mul: random instances over several primes, all strategies equal
    mul_primes = [97, 786433, P31, P60NTT, P60, 65537, 3]
    for idx in range(90):
        p = mul_primes[idx % len(mul_primes)]
        ctx = field_new(p)
        m, k, n = rng.randint(1, 6), rng.randint(1, 6), rng.randint(1, 6)
        maxdeg = rng.choice([0, 1, 3, 7, 16, 31, 64])
        if idx % 9 == 0:
            A = PolMat.zeros(ctx, m, k)
        else:
            A = rand_polmat_ragged(ctx, m, k, maxdeg, rng)
        B = rand_polmat_ragged(ctx, k, n, rng.choice([0, 2, 9, 33, 64]), rng)
        C = pm_mul(A, B)
        strategies = applicable_strategies(A, B)
        for st in strategies:
            assert pm_mul(A, B, strategy=st) == C, (idx, st)
        out["mul"].append({"p": p, "m": m, "k": k, "n": n, "A": rows_of(A), "B": rows_of(B),
                           "C": rows_of(C), "strategies": strategies})
    # dispatch-relevant shapes: dims > 10 so the reference takes its ntt path
    for (m, k, n, d, p) in ((12, 11, 13, 40, P31), (16, 16, 16, 100, P31), (11, 12, 11, 30, P60)):
        ctx = field_new(p)
        A = random_polmat(ctx, m, k, d, rng)
        B = random_polmat(ctx, k, n, d, rng)
        out["mul"].append({"p": p, "m": m, "k": k, "n": n, "A": rows_of(A), "B": rows_of(B),
                           "C": rows_of(pm_mul(A, B)), "strategies": applicable_strategies(A, B)})

    # middle products: _pm_middle (internal, reference semantics incl. its
    # cyclic fold, polmat.py:484-536) and the checked public wrapper
    mid_cases = [
        # (p, m, k, n, degA, degB, c, d) -- first two alias
        (P31, 2, 2, 2, 3, 259, 200, 60),
        (P31, 2, 2, 2, 23, 80, 41, 40),
        (P31, 2, 2, 2, 63, 127, 64, 64),
        (P31, 2, 2, 2, 32, 127, 64, 64),
        (P31, 3, 4, 2, 20, 39, 20, 20),
        (97, 2, 3, 2, 10, 40, 11, 30),
        (786433, 3, 3, 3, 40, 120, 41, 80),
        (P60, 2, 2, 3, 15, 47, 16, 32),
        (P31, 4, 4, 2, 7, 200, 8, 150),
        (P31, 1, 1, 1, 19, 299, 200, 100),
    ]
    for (p, m, k, n, da, db, c, d) in mid_cases:
        ctx = field_new(p)
        A = random_polmat(ctx, m, k, da, rng)
        B = random_polmat(ctx, k, n, db, rng)
        R = _pm_middle(A, B, c, d)
        full = pm_mul(A, B, strategy="naive").slice_coeffs(c, c + d)
        rec = {"p": p, "m": m, "k": k, "n": n, "c": c, "d": d, "A": rows_of(A),
               "B": rows_of(B), "R": rows_of(R), "is_true_slice": R == full,
               "true_slice": rows_of(full)}
        try:
            rec["public"] = rows_of(pm_middle_product(A, B, c, d))
        except Exception as exc:  # DegreeTooLarge etc.
            rec["public_error"] = type(exc).__name__
        out["middle"].append(rec)
    for idx in range(20):
        p = [P31, 97, 786433][idx % 3]
        ctx = field_new(p)
        m, k, n = rng.randint(1, 4), rng.randint(1, 4), rng.randint(1, 4)
        c = rng.randint(1, 70)
        d = rng.randint(1, 70)
        A = rand_polmat_ragged(ctx, m, k, c - 1, rng)
        B = rand_polmat_ragged(ctx, k, n, c + d - 1, rng)
        R = _pm_middle(A, B, c, d)
        full = pm_mul(A, B, strategy="naive").slice_coeffs(c, c + d)
        out["middle"].append({"p": p, "m": m, "k": k, "n": n, "c": c, "d": d,
                              "A": rows_of(A), "B": rows_of(B), "R": rows_of(R),
                              "is_true_slice": R == full, "true_slice": rows_of(full),
                              "public": rows_of(pm_middle_product(A, B, c, d))})

    # mbasis1 structure (appint.py:24-60), incl. SPEC S:351-354 examples
    out["mbasis1"].append({"p": 97, "R": [[1], [1]], "s": [0, 0],
                           "P": rows_of(mbasis1([[1], [1]], [0, 0], ctx97))})
    for idx in range(40):
        p = [97, P31, 3][idx % 3]
        ctx = field_new(p)
        m = rng.randint(1, 9)
        n = rng.randint(1, 5)
        rank = rng.randint(0, min(m, n))
        # rank-deficient R = X * Y with duplicate rows sometimes
        X = [[rng.randrange(p) for _ in range(rank)] for _ in range(m)]
        Y = [[rng.randrange(p) for _ in range(n)] for _ in range(rank)]
        R = [[sum(X[i][t] * Y[t][j] for t in range(rank)) % p for j in range(n)] for i in range(m)]
        if idx % 5 == 0 and m > 1:
            R[m - 1] = R[0][:]
        s = [rng.randint(-3, 3) for _ in range(m)]
        kernel, pivots = _mbasis1_struct(R, s, p)
        out["mbasis1"].append({"p": p, "R": R, "s": s, "pivots": pivots,
                               "kernel": {str(i): kv for i, kv in kernel.items()},
                               "P": rows_of(mbasis1(R, s, ctx))})

    # mbasis / pmbasis (appint.py:143-196); pmbasis output is T-independent
    def approx_case(p, m, n, sigma, s, kind, F=None):
        ctx = field_new(p)
        if F is None:
            F = random_polmat(ctx, m, n, sigma - 1, rng)
        rec = {"p": p, "m": m, "n": n, "sigma": sigma, "s": s, "F": rows_of(F)}
        if kind == "mbasis":
            P = mbasis(F.truncate(sigma), sigma, s)
        else:
            P = pmbasis(F, sigma, s)
            old = config.PMBASIS_BASE_ORDER
            try:
                config.PMBASIS_BASE_ORDER = 4
                assert pmbasis(F, sigma, s) == P
            finally:
                config.PMBASIS_BASE_ORDER = old
        assert is_owp(P, s)
        rec["P"] = rows_of(P)
        rec["rdeg"] = [int(x) for x in rdeg(P, s)]
        return rec

    for idx in range(25):
        p = [P31, 97, 786433, P60NTT, P60][idx % 5]
        m = rng.randint(1, 8)
        n = rng.randint(1, max(1, m - 1))
        sigma = rng.randint(1, 30)
        s = [0] * m if idx % 2 == 0 else [rng.randint(-5, 10) for _ in range(m)]
        out["mbasis"].append(approx_case(p, m, n, sigma, s, "mbasis"))
    for idx in range(30):
        p = [P31, 97, 786433, P60, 65537][idx % 5]
        m = rng.randint(2, 8)
        n = rng.randint(1, max(1, m // 2 + 1))
        sigma = rng.choice([33, 40, 64, 65, 77, 100, 128])
        s = [0] * m if idx % 3 == 0 else [rng.randint(-5, 20) for _ in range(m)]
        out["pmbasis"].append(approx_case(p, m, n, sigma, s, "pmbasis"))
    # degenerate pmbasis instances: duplicate row, zero row, zero column, zero F
    for kind in ("dup_row", "zero_row", "zero_col", "zero"):
        p = P31
        ctx = field_new(p)
        m, n, sigma = 6, 3, 70
        F = random_polmat(ctx, m, n, sigma - 1, rng)
        rows = [[list(e) for e in r] for r in F.rows]
        if kind == "dup_row":
            rows[4] = [list(e) for e in rows[1]]
        elif kind == "zero_row":
            rows[2] = [[] for _ in range(n)]
        elif kind == "zero_col":
            for r in rows:
                r[1] = []
        else:
            rows = [[[] for _ in range(n)] for _ in range(m)]
        F = PolMat(ctx, rows, ncols=n)
        s = [0, 3, -2, 1, 0, 5]
        rec = approx_case(p, m, n, sigma, s, "pmbasis", F=F)
        rec["kind"] = kind
        out["pmbasis"].append(rec)

    path = os.path.join(HERE, "small.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, os.path.getsize(path), {k: len(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
