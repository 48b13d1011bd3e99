"""Dynamic SASS opcode mix and stall samples per kernel from an ncu report.

usage: python tools/ncu_mix.py REPORT.ncu-rep [TOP]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            secs.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r:
            cur["rows"].append(r)
    for sec in secs:
        h = sec["hdr"]
        iex, iss, isrc = (h.index("Instructions Executed"),
                          h.index("Warp Stall Sampling (All Samples)"), h.index("Source"))
        ops, smp, tot, stot = collections.Counter(), collections.Counter(), 0, 0
        for r in sec["rows"]:
            try:
                n, s = int(r[iex] or 0), int(r[iss] or 0)
            except ValueError:
                continue
            m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", r[isrc].strip())
            op = m.group(2) if m else r[isrc].strip()
            ops[op] += n
            smp[op] += s
            tot += n
            stot += s
        print(sec["name"][:80], "warp-instructions", tot, "stall samples", stot)
        for op, n in ops.most_common(top):
            print(f"  {n / tot * 100:6.2f}% {n:12d}  stall {smp[op] / max(stot, 1) * 100:5.1f}%  {op}")


if __name__ == "__main__":
    main()
