"""Join an ncu SASS source page (CSV) with nvdisasm -g line info.

usage: python tools/sass_lines.py NCU_SASS.csv FUNC.dis
Prints executed warp-instructions and stall samples aggregated per CUDA line.
"""
import collections
import csv
import re
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = rows[1]
    iex = hdr.index("Instructions Executed")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    ncu = []
    for r in rows[2:]:
        try:
            ncu.append((int(r[iex] or 0), int(r[iss] or 0)))
        except ValueError:
            pass
    lines = []
    cur = None
    for ln in open(sys.argv[2]):
        m = re.search(r'line (\d+)', ln)
        if m and "//##" in ln:
            cur = int(m.group(1))
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", ln):
            lines.append(cur)
    n = min(len(lines), len(ncu))
    agg = collections.defaultdict(lambda: [0, 0])
    for i in range(n):
        agg[lines[i]][0] += ncu[i][0]
        agg[lines[i]][1] += ncu[i][1]
    tex = sum(v[0] for v in agg.values())
    tss = sum(v[1] for v in agg.values())
    print(f"sass={len(lines)} ncu={len(ncu)} instr={tex} samples={tss}")
    for ln, (ex, ss) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
        print(f"line {ln}: instr {ex:9d} ({ex / tex * 100:5.1f}%)  samples {ss:5d} ({ss / max(tss,1) * 100:5.1f}%)")


if __name__ == "__main__":
    main()
