"""Warp-stall samples of the tcgen05 pipeline kernel per role and stall reason, from
an ncu source page (--page source --csv --print-source cuda,sass).
usage: ncu_roles.py src.csv [mlp_tc.cuh line ranges: mma=a-b producer=a-b epilogue=a-b]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
rng = {"mma": (395, 490), "producer": (491, 880), "epilogue": (881, 1020)}
for a in sys.argv[2:]:
    k, v = a.split("=")
    lo, hi = v.split("-")
    rng[k] = (int(lo), int(hi))
cur = hdr = None
agg = collections.defaultdict(collections.Counter)
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
        ln = int(r[0])
        role = cur
        if cur == "mlp_tc.cuh":
            role = "tc-helpers"
            for k, (lo, hi) in rng.items():
                if lo <= ln <= hi:
                    role = k
        if cur == "sweep_core.cuh":
            role = "epilogue(sweep)"
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "-"):
                agg[role][k[6:]] += int(v)
        agg[role]["inst"] += int(d.get("Instructions Executed") or 0)
tot = sum(sum(v for k, v in c.items() if k != "inst") for c in agg.values())
for role, c in sorted(agg.items(), key=lambda x: -sum(v for k, v in x[1].items() if k != "inst")):
    s = sum(v for k, v in c.items() if k != "inst")
    top = ", ".join(f"{k} {100 * v / max(s, 1):.0f}%" for k, v in c.most_common(7) if k != "inst")
    print(f"{role:18s} samples {100 * s / tot:5.1f}%  inst {c['inst']:>11d}  [{top}]")
