"""Join an ncu SASS source page (CSV) with nvdisasm -g line info.

usage: python tools/sass_lines.py NCU_SASS.csv FUNC.dis [MANGLED_SUBSTRING]
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
        if r and r[0] == "Kernel Name":
            break  # next kernel's section
        try:
            ncu.append((int(r[iex] or 0), int(r[iss] or 0)))
        except ValueError:
            pass
    # a cubin may hold several kernels: keep the function whose instruction
    # count matches the ncu source page
    funcs, cur_f = {}, None
    for ln in open(sys.argv[2]):
        if ln.startswith("\t.text.") or ln.startswith(".text."):
            cur_f = ln.strip().rstrip(":")
            funcs[cur_f] = []
        if cur_f is not None:
            funcs[cur_f].append(ln)
    chosen = None
    want = sys.argv[3] if len(sys.argv) > 3 else None  # substring of the mangled name
    for f, body in funcs.items():
        cnt = sum(1 for l in body if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", l))
        if cnt == len(ncu) and (want is None or want in f):
            chosen = body
    body = chosen if chosen is not None else open(sys.argv[2]).readlines()
    lines = []
    cur = None
    for ln in body:
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if m and "//##" in ln:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
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
        print(f"{ln}: instr {ex:9d} ({ex / tex * 100:5.1f}%)  samples {ss:5d} ({ss / max(tss,1) * 100:5.1f}%)")


if __name__ == "__main__":
    main()
