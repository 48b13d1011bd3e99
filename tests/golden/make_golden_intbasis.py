"""Golden vectors for the interpolant bases, produced by
the reference itself: appint.m_intbasis / pm_intbasis / eval_polmat_points
(appint.py:208-319).

usage: PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
       python tests/golden/make_golden_intbasis.py
Inputs are regenerated in the tests from `seed` with random.Random in the
draw order of `draw_case` (kept identical in tests/test_gpu_intbasis.py).
"""
import hashlib
import json
import os
import random

from fpmat.appint import eval_polmat_points, m_intbasis, pm_intbasis
from fpmat.modring import field_new
from fpmat.polmat import PolMat, polmat_to_text

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "intbasis.json")


def draw_case(seed, p, m, n, order, geometric=False, zero_every=0):
    rng = random.Random(seed)
    E = []
    for t in range(order):
        if zero_every and t % zero_every == 0:
            E.append([[0] * n for _ in range(m)])
        else:
            E.append([[rng.randrange(p) for _ in range(n)] for _ in range(m)])
    if geometric:
        a0, r = rng.randrange(1, p), rng.randrange(2, p)
        alpha, cur = [], a0
        for _ in range(order):
            alpha.append(cur)
            cur = cur * r % p
    else:
        alpha = rng.sample(range(p), order)
    return E, alpha


def main():
    cases = []
    specs = [
        # (seed, p, m, n, order, shift, geometric, zero_every, flavor)
        (1, 97, 3, 1, 5, [0, 0, 0], False, 0, "m"),
        (2, 97, 4, 2, 20, [0, 1, 2, 3], False, 0, "m"),
        (3, 65537, 5, 2, 33, [0] * 5, False, 0, "pm"),
        (4, 2013265921, 6, 3, 40, [2, 0, 0, 1, 5, 0], False, 0, "pm"),
        (5, 2013265921, 8, 4, 70, [0] * 8, True, 0, "pm"),
        (6, 2013265921, 4, 2, 24, [0] * 4, False, 3, "m"),
        (7, 2013265921, 8, 2, 64, [-3, 0, 7, 1, 1, 0, 2, 9], False, 5, "pm"),
        (8, 2013265921, 16, 8, 256, [0] * 16, True, 0, "pm"),
        (9, 2013265921, 12, 5, 150, [0] * 12, False, 0, "pm"),
        (10, 2013265921, 2, 3, 12, [0, 0], False, 0, "pm"),          # m < n
        (14, 2013265921, 4, 4, 30, [1, 0, 0, 2], False, 4, "pm"),    # m = n
        (15, 3, 3, 2, 3, [0, 0, 0], False, 0, "m"),                  # p = 3, all points
        (16, 2013265921, 40, 32, 64, [0] * 40, False, 7, "pm"),      # the n = 32 block solve
        (17, 2013265921, 64, 32, 100, [0] * 64, True, 0, "pm"),      # cfg4 / ib4 shape
    ]
    for seed, p, m, n, order, shift, geo, ze, flavor in specs:
        ctx = field_new(p)
        E, alpha = draw_case(seed, p, m, n, order, geo, ze)
        fn = m_intbasis if flavor == "m" else pm_intbasis
        P = fn(E, alpha, list(shift), ctx)
        txt = polmat_to_text(P)
        rec = {"seed": seed, "p": p, "m": m, "n": n, "order": order, "shift": shift,
               "geometric": geo, "zero_every": ze, "flavor": flavor,
               "sha256": hashlib.sha256(txt.encode()).hexdigest(), "deg": P.degree}
        if len(txt) < 20000:
            rec["rows"] = P.rows
        cases.append(rec)
        print("case", seed, m, n, order, "deg", P.degree)
    evals = []
    for seed, p, m, n, deg, npts, geo in [(11, 2013265921, 3, 4, 40, 30, True),
                                          (12, 2013265921, 2, 2, 10, 7, False),
                                          (13, 97, 3, 3, 20, 15, True)]:
        rng = random.Random(seed)
        ctx = field_new(p)
        rows = [[[rng.randrange(p) for _ in range(deg + 1)] for _ in range(n)] for _ in range(m)]
        if geo:
            a0, r = rng.randrange(1, p), rng.randrange(2, p)
            pts, cur = [], a0
            for _ in range(npts):
                pts.append(cur)
                cur = cur * r % p
        else:
            pts = [rng.randrange(p) for _ in range(npts)]
        P = PolMat(ctx, rows)
        evals.append({"p": p, "rows": rows, "pts": pts, "vals": eval_polmat_points(P, pts, ctx)})
    with open(OUT, "w") as f:
        json.dump({"cases": cases, "evals": evals}, f)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
