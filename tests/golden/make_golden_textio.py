"""Golden vectors for the interchange formats, produced by the reference itself
(polmat_to_text / polmat_from_text, polmat.py:617-647).

usage: PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
       python tests/golden/make_golden_textio.py
"""
import hashlib
import json
import os
import random

from fpmat.modring import field_new
from fpmat.polmat import PolMat, polmat_from_text, polmat_to_text

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "textio.json")


def rand_rows(rng, p, m, n, maxlen, zero_frac=0.2):
    rows = []
    for _ in range(m):
        row = []
        for _ in range(n):
            if rng.random() < zero_frac:
                row.append([])
                continue
            L = rng.randrange(1, maxlen + 1)
            c = [rng.randrange(p) for _ in range(L)]
            if rng.random() < 0.3:
                c[-1] = 0  # trailing zero, trimmed by PolMat
            row.append(c)
        rows.append(row)
    return rows


def main():
    rng = random.Random(2026)
    to_text = []
    for p, m, n, maxlen in [(97, 3, 4, 6), (2013265921, 5, 3, 40), ((1 << 60) - 93, 4, 4, 25),
                            (3, 2, 2, 5), (65537, 1, 1, 1), (2013265921, 0, 3, 4),
                            (2013265921, 16, 16, 300)]:
        ctx = field_new(p)
        rows = rand_rows(rng, p, m, n, maxlen)
        A = PolMat(ctx, [[list(e) for e in r] for r in rows], ncols=n)
        for r in A.rows:  # PolMat stores trimmed lists (upoly._trim)
            for e in r:
                while e and e[-1] == 0:
                    e.pop()
        txt = polmat_to_text(A)
        rec = {"p": p, "m": m, "n": n, "rows": rows,
               "sha256": hashlib.sha256(txt.encode()).hexdigest()}
        if len(txt) < 4000:
            rec["text"] = txt
        to_text.append(rec)
    from_text = []
    cases = [
        "97 2 2\n1 2\n\n0 0 5 0\n200\n",                # trailing zero, reduction
        "97 2 2\n1 2\n",                                # missing lines
        "  97   2 1 \n -3 4\n  ",                       # spaces, negative
        "97 1 3\r\n1 2 3\r\n4\r\n\r\n",                 # CRLF
        "97 2 1\n1\t2\x0b3\n",                          # tab, vertical tab line break
        "97 1 2\n1_000 5\n7 8 9\nextra line\n",         # underscore, extra lines
        "2013265921 1 1\n123456789012345678901234567890 -1\n",  # bignum, -1
        "1152921504606846883 2 2\n1152921504606846883 1\n\n-5\n1 0 0\n",
        "5 1 1\n0 0 0\n",                               # all-zero entry
        "7 0 0\n",
    ]
    for t in cases:
        A = polmat_from_text(t)
        from_text.append({"text": t, "p": A.ctx.p, "m": A.m, "n": A.n, "rows": A.rows})
    errors = []
    for t in ["", "97 2\n", "97 a 2\n", "97 1 1\n1 x\n"]:
        try:
            polmat_from_text(t)
            errors.append({"text": t, "error": None})
        except Exception as exc:  # noqa: BLE001
            errors.append({"text": t, "error": type(exc).__name__})
    with open(OUT, "w") as f:
        json.dump({"to_text": to_text, "from_text": from_text, "errors": errors}, f)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
