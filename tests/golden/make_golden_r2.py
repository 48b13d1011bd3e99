"""Round-2 golden vectors, produced by running the UNMODIFIED reference
(`fpmat`, /root/reference/pkg/src) in the build container:

* pmbasis over a 60-bit prime of two-adicity 1 (p = 2^60 - 93), 4x3, orders
  128 and 100, T = 32 / 8: the u64 recursion's middle products then take the
  entrywise branch with a basis of stride order+1 and length deg+1 (ADVICE
  round 1: the stride check rejected it);
* pm_intbasis / m_intbasis with points that are distinct integers but equal
  residues (alpha = 1 and 1 + p): appint._check_points compares the
  integers (appint.py:203-205) and the reference proceeds.

usage: PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
       python tests/golden/make_golden_r2.py
Inputs are regenerated in the tests from `seed` (draw order in `draw_*`).
"""
import json
import os
import random

from fpmat import config
from fpmat.appint import m_intbasis, pm_intbasis, pmbasis
from fpmat.modring import field_new
from fpmat.polmat import random_polmat

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "r2.json")
P60 = (1 << 60) - 93


def draw_pmb(seed, p, m, n, order):
    ctx = field_new(p)
    return random_polmat(ctx, m, n, order - 1, random.Random(seed))


def draw_ib(seed, p, m, n, order):
    rng = random.Random(seed)
    E = [[[rng.randrange(p) for _ in range(n)] for _ in range(m)] for _ in range(order)]
    alpha = rng.sample(range(1, p), order - 2)
    alpha = [1, 1 + p] + alpha  # distinct integers, one residue twice
    return E, alpha


def main():
    out = {"pmbasis": [], "intbasis": []}
    for seed, p, m, n, order, T, s in [(1, P60, 4, 3, 128, 32, [0, 0, 0, 0]),
                                       (2, P60, 4, 3, 100, 8, [0, 1, 0, 2]),
                                       (3, P60, 5, 2, 90, 32, [0, 0, 0, 0, 0])]:
        F = draw_pmb(seed, p, m, n, order)
        old = config.PMBASIS_BASE_ORDER
        config.PMBASIS_BASE_ORDER = T
        try:
            P = pmbasis(F, order, s)
        finally:
            config.PMBASIS_BASE_ORDER = old
        out["pmbasis"].append({"seed": seed, "p": p, "m": m, "n": n, "order": order, "T": T,
                               "s": s, "P": [[list(e) for e in r] for r in P.rows]})
    for seed, p, m, n, order, fn in [(4, 2013265921, 3, 2, 12, "pm_intbasis"),
                                     (5, 97, 4, 2, 20, "m_intbasis"),
                                     (6, 2013265921, 6, 3, 40, "pm_intbasis")]:
        E, alpha = draw_ib(seed, p, m, n, order)
        ctx = field_new(p)
        s = [0] * m
        P = (pm_intbasis if fn == "pm_intbasis" else m_intbasis)(E, alpha, s, ctx)
        out["intbasis"].append({"seed": seed, "p": p, "m": m, "n": n, "order": order, "fn": fn,
                                "alpha": alpha, "P": [[list(e) for e in r] for r in P.rows]})
    with open(OUT, "w") as f:
        json.dump(out, f)
    print(len(out["pmbasis"]), "pmbasis,", len(out["intbasis"]), "intbasis cases")


if __name__ == "__main__":
    main()
