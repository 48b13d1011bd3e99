"""Aggregate ncu per-instruction stall samples by source-line ranges (roles).

usage: python tools/stall_roles.py NCU_SASS.csv FUNC.dis MANGLED_SUBSTR FILE a-b:name [a-b:name ...]
"""
import collections
import csv
import re
import sys


def main():
    src, dis, want, fname = sys.argv[1:5]
    ranges = []
    for spec in sys.argv[5:]:
        ab, name = spec.split(":")
        a, b = ab.split("-")
        ranges.append((int(a), int(b), name))
    rows = list(csv.reader(open(src)))
    hdr = rows[1]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    iex = hdr.index("Instructions Executed")
    data = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break
        data.append(r)
    funcs, cur = {}, None
    for ln in open(dis):
        if ln.startswith(".text."):
            cur = ln.strip()
            funcs[cur] = []
        if cur:
            funcs[cur].append(ln)
    body = next(b for f, b in funcs.items() if want in f)
    lines, loc = [], None
    for ln in body:
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if m and "//##" in ln:
            loc = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", ln):
            lines.append(loc)
    agg = collections.defaultdict(collections.Counter)
    ins = collections.Counter()
    last = "other"
    for k, r in enumerate(data[: len(lines)]):
        f, l = lines[k] if lines[k] else ("", 0)
        role = last  # inlined helpers count for the role whose code surrounds them
        if f == fname:
            role = next((n for a, b, n in ranges if a <= l <= b), "other")
            last = role
        for c in cols:
            try:
                agg[role][hdr[c][6:]] += int(r[c] or 0)
            except ValueError:
                pass
        try:
            ins[role] += int(r[iex] or 0)
        except ValueError:
            pass
    for role, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values())):
        print(f"{role:10s} samples {sum(c.values()):6d} instr {ins[role]:10d}  ",
              [(k, v) for k, v in c.most_common(6)])


if __name__ == "__main__":
    main()
