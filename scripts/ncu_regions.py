"""Per-region SASS instruction counts / stall samples from an ncu source page
(csv, --print-source cuda,sass): each SASS row is charged to the CUDA line
printed above it.  usage: python scripts/ncu_regions.py src.csv"""
import collections
import csv
import re
import sys

MLP_REGIONS = [(157, 380, "consumer_mlp"), (380, 470, "clamp/loads"), (470, 650, "producer_feat"),
               (650, 830, "producer_csr"), (830, 905, "consumer_sweep"), (905, 1300, "kernel_loop")]


def region(f, ln):
    if f == "mlp.cu":
        for a, b, n in MLP_REGIONS:
            if a <= ln < b:
                return n
    return f


rows = list(csv.reader(open(sys.argv[1])))
cur = hdr = None
line = None
inst = collections.Counter()
samp = collections.Counter()
ops = collections.defaultdict(collections.Counter)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0].isdigit() and r[2] == "-":
        line = int(r[0])
        d = dict(zip(hdr, r))
        reg = region(cur, line)
        inst[reg] += int(d.get("Instructions Executed") or 0)
        samp[reg] += int(d.get("Warp Stall Sampling (All Samples)") or 0)
        continue
    if r[0] == "" and hdr is not None and line is not None and r[4] != "-":
        d = dict(zip(hdr, r))
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[3])
        if m:
            ops[region(cur, line)][m.group(2)] += int(d.get("Instructions Executed") or 0)
tot = sum(inst.values())
print("total SASS instructions", tot)
for reg, n in inst.most_common():
    top = ", ".join(f"{o}:{c * 100 // max(n, 1)}%" for o, c in ops[reg].most_common(8))
    print(f"{reg:28s} {n:12d} {100 * n / tot:5.1f}%  samples {samp[reg]:6d}  [{top}]")
