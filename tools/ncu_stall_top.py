"""Instructions with the most samples of one stall reason (ncu source page).

usage: python tools/ncu_stall_top.py SRC.csv REASON [KERNEL_INDEX] [N]
  REASON: a column such as stall_long_sb, stall_math, stall_wait
Prints each hot instruction with the previous 3 instructions for context.
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    reason = sys.argv[2]
    ki = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 12
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            secs.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r:
            cur["rows"].append(r)
    sec = secs[ki]
    h = sec["hdr"]
    col, src = h.index(reason), h.index("Source")
    vals = []
    for k, r in enumerate(sec["rows"]):
        try:
            vals.append((int(r[col] or 0), k))
        except ValueError:
            vals.append((0, k))
    tot = sum(v for v, _ in vals)
    print(sec["name"][:70], reason, "total", tot)
    for v, k in sorted(vals, reverse=True)[:n]:
        print(f"--- {v / max(tot, 1) * 100:5.1f}%")
        for kk in range(max(0, k - 3), k + 1):
            print("    ", sec["rows"][kk][src].strip())


if __name__ == "__main__":
    main()
