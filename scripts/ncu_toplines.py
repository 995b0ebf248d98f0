"""Top CUDA source lines by warp-stall samples from an ncu source page csv
(--page source --csv --print-source cuda,sass).  usage: ncu_toplines.py src.csv [file] [n]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else None
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur = hdr = None
samp = collections.Counter()
inst = collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0].isdigit() and len(r) > 2 and r[2] == "-":
        d = dict(zip(hdr, r))
        if want and cur != want:
            continue
        key = (cur, int(r[0]))
        samp[key] += int(d.get("Warp Stall Sampling (All Samples)") or 0)
        inst[key] += int(d.get("Instructions Executed") or 0)
tot = sum(samp.values())
print("total samples", tot)
for (f, ln), s in samp.most_common(n):
    print(f"{f}:{ln:5d} {s:8d} {100 * s / max(tot, 1):5.1f}%  inst {inst[(f, ln)]}")
