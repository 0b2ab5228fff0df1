"""Aggregate executed warp-instructions per CUDA source line (ncu source page)."""
import csv
import subprocess
import sys
from collections import defaultdict

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
cur = None
agg = defaultdict(lambda: [0, ""])
tot = 0
fname = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        continue
    if r[0] == "Function Name":
        continue
    if r[0]:
        try:
            v = int(r[ie])
        except (ValueError, IndexError, NameError):
            v = 0
        agg[(fname, int(r[0]))][0] += v
        agg[(fname, int(r[0]))][1] = r[1].strip()[:80]
        tot += v
print("total warp instructions", tot)
for (f, ln), (v, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100 * v / tot:5.1f}% {v / 1e6:8.1f}M {f}:{ln} {s}")
