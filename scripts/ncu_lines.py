"""Aggregate ncu --page source (cuda) warp-stall samples per source line.
usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur = None
hdr = None
agg = []
total = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        cur = r[1].split("/")[-1]
        hdr = None
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    if len(r) < 5 or r[2] != "-":
        continue  # SASS rows; keep the per-CUDA-line aggregate rows
    try:
        s = int(r[4] or 0)
    except ValueError:
        continue
    total += s
    agg.append((s, cur, int(r[0]), r[1][:90]))
agg.sort(reverse=True)
print("total samples", total)
for s, f, l, src in agg[:top]:
    print(f"{100.0*s/max(total,1):5.1f}%  {f}:{l}  {src}")
