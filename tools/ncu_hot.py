"""Per-instruction stall samples of one kernel from an ncu report: totals by
stall reason, the waits on each mbarrier / the top instructions.

usage: python tools/ncu_hot.py REPORT.ncu-rep [TOPN]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = [r for r in rows[2:] if r and r[0].startswith("0x")]
    ia, isrc, isamp, iex = (hdr.index(k) for k in ("Address", "Source", "# Samples",
                                                   "Instructions Executed"))
    stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    base = int(data[0][ia], 16)
    tot = collections.Counter()
    lines = []
    prev = ""
    for r in data:
        s = int(r[isamp])
        for i in stall:
            tot[hdr[i]] += int(r[i])
        lines.append((s, int(r[ia], 16) - base, r[isrc].strip(), prev, int(r[iex])))
        prev = r[isrc].strip()
    n = sum(x[0] for x in lines)
    print("samples", n, "warp-instructions", sum(x[4] for x in lines))
    print(tot.most_common(8))
    for s, off, src, prv, ex in sorted(lines, reverse=True)[:topn]:
        note = "   <- " + prv[:60] if "BRA" in src else ""
        print(f"{s:7d} {100 * s / n:5.1f}% {off:#7x} x{ex:<9d} {src[:70]}{note}")


if __name__ == "__main__":
    main()
