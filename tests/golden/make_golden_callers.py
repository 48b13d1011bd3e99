"""Golden fixtures for the callers one step up the hot path (SURVEY 8(f)
rank 4): `fracrec_series` (fraction.py:54-69), `fracrec_points`
(fraction.py:72-97) and `kernel_direct` (kernel.py:42-76, approx and interp
flavors), produced by running the UNMODIFIED
reference in the build container.

Test infrastructure only; the committed JSON travels to the GPU box.
Re-run with:  python tests/golden/make_golden_callers.py
"""
import json
import os
import random
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, os.environ.get("FPMAT_REF", "/root/reference/pkg/src"))

from fpmat.errors import ReconstructionFailed  # noqa: E402
from fpmat.fraction import fracrec_points, fracrec_series  # noqa: E402
from fpmat.kernel import kernel_direct  # noqa: E402
from fpmat.modring import field_new  # noqa: E402
from fpmat.polmat import PolMat, pm_eval, pm_mul, random_polmat  # noqa: E402
from fpmat.solve import newton_inv_trunc  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
P31 = 2013265921


def _inv(A, p):
    """Inverse of a constant matrix mod p (Gauss-Jordan; fixture helper)."""
    n = len(A)
    M = [list(r) + [1 if i == j else 0 for j in range(n)] for i, r in enumerate(A)]
    for c in range(n):
        r = next(i for i in range(c, n) if M[i][c] % p)
        M[c], M[r] = M[r], M[c]
        iv = pow(M[c][c], -1, p)
        M[c] = [x * iv % p for x in M[c]]
        for i in range(n):
            if i != c and M[i][c]:
                f = M[i][c]
                M[i] = [(x - f * y) % p for x, y in zip(M[i], M[c])]
    return [r[n:] for r in M]


def rows(M):
    return [[list(e) for e in r] for r in M.rows]


def main():
    out = {"fracrec": [], "kernel": []}
    rng = random.Random(2024)
    for p, n, D in [(P31, 2, 6), (P31, 3, 10), (97, 2, 5), (65537, 4, 8), (P31, 1, 12)]:
        ctx = field_new(p)
        for trial in range(2):
            Q = random_polmat(ctx, n, n, D, rng)
            R = random_polmat(ctx, n, n, D - 1, rng)
            try:
                S = newton_inv_trunc(Q, 2 * D)
            except Exception:
                continue
            H = pm_mul(S, R).truncate(2 * D)
            rec = {"p": p, "n": n, "D": D, "H": rows(H)}
            try:
                d = fracrec_series(H, D)
                rec.update({"Q": rows(d.Q), "R": rows(d.R)})
            except ReconstructionFailed as exc:
                rec["error"] = type(exc).__name__
            out["fracrec"].append(rec)
    # a non-proper input: the reference reports ReconstructionFailed
    ctx = field_new(P31)
    H = random_polmat(ctx, 2, 2, 7, rng)
    try:
        d = fracrec_series(H, 2)
        out["fracrec"].append({"p": P31, "n": 2, "D": 2, "H": rows(H), "Q": rows(d.Q),
                               "R": rows(d.R)})
    except ReconstructionFailed as exc:
        out["fracrec"].append({"p": P31, "n": 2, "D": 2, "H": rows(H),
                               "error": type(exc).__name__})
    for p, m, n, d, s in [(P31, 4, 2, 4, [0, 0, 0, 0]), (P31, 5, 2, 3, [0, 1, 2, 0, 1]),
                          (97, 3, 1, 5, [0, 0, 0]), (65537, 6, 3, 3, [2, 0, 0, 1, 0, 3]),
                          (P31, 3, 2, 2, [0, 0, 0])]:
        ctx = field_new(p)
        F = random_polmat(ctx, m, n, d, rng)
        kb = kernel_direct(F, s)
        out["kernel"].append({"p": p, "m": m, "n": n, "s": s, "F": rows(F), "K": rows(kb.K)})
    # a rank-deficient F (duplicate column): a larger kernel
    ctx = field_new(P31)
    F = random_polmat(ctx, 4, 2, 3, rng)
    F = PolMat(ctx, [[r[0], r[0]] for r in F.rows])
    kb = kernel_direct(F, [0, 0, 0, 0])
    out["kernel"].append({"p": P31, "m": 4, "n": 2, "s": [0, 0, 0, 0], "F": rows(F),
                          "K": rows(kb.K)})
    # interpolation routes (PM-IntBasis); a separate rng
    # stream so the cases above keep their inputs
    rng2 = random.Random(4048)
    out["fracrec_points"] = []
    for p, n, D in [(P31, 2, 6), (P31, 3, 9), (65537, 2, 5)]:
        ctx = field_new(p)
        Q = random_polmat(ctx, n, n, D, rng2)
        R = random_polmat(ctx, n, n, D - 1, rng2)
        pts = rng2.sample(range(1, p), 2 * D)
        Hvals = []
        for x in pts:
            Qx, Rx = pm_eval(Q, x), pm_eval(R, x)
            from fpmat._dense import mat_mul
            Hvals.append(mat_mul(_inv(Qx, p), Rx, p))  # H(x) = Q(x)^-1 R(x)
        rec = {"p": p, "n": n, "D": D, "pts": pts, "Hvals": Hvals}
        try:
            d = fracrec_points(ctx, Hvals, pts, D)
            rec.update({"Q": rows(d.Q), "R": rows(d.R)})
        except ReconstructionFailed as exc:
            rec["error"] = type(exc).__name__
        out["fracrec_points"].append(rec)
    out["kernel_interp"] = []
    for p, m, n, d, s in [(P31, 4, 2, 4, [0, 0, 0, 0]), (P31, 5, 2, 3, [0, 1, 2, 0, 1]),
                          (65537, 6, 3, 3, [2, 0, 0, 1, 0, 3])]:
        ctx = field_new(p)
        F = random_polmat(ctx, m, n, d, rng2)
        kb = kernel_direct(F, s, flavor="interp")
        out["kernel_interp"].append({"p": p, "m": m, "n": n, "s": s, "F": rows(F),
                                     "K": rows(kb.K)})
    with open(os.path.join(HERE, "callers.json"), "w") as f:
        json.dump(out, f)
    print(len(out["fracrec"]), "fracrec,", len(out["kernel"]), "kernel,",
          len(out["fracrec_points"]), "fracrec_points,", len(out["kernel_interp"]),
          "kernel interp cases")


if __name__ == "__main__":
    main()
