"""Summarise an ncu report's SASS page: instruction share and stall-sample
share per 100-instruction region (experiment helper)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
step = int(sys.argv[2]) if len(sys.argv) > 2 else 100
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
rows = r[2:]
tot = sum(int(x[5]) for x in rows)
samp = sum(int(x[2]) for x in rows) or 1
print("total warp-instructions", tot, "samples", samp)
for i in range(0, len(rows), step):
    s = sum(int(x[5]) for x in rows[i:i + step])
    sm = sum(int(x[2]) for x in rows[i:i + step])
    if s / tot > 0.002 or sm / samp > 0.002:
        print(i, "%.3f" % (s / tot), "%.3f" % (sm / samp), rows[i][1].strip()[:50])
