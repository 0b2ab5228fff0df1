"""Warp-stall samples of one kernel aggregated per SASS opcode and per stall reason
(`ncu --page source --print-source sass`)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
by_op = defaultdict(lambda: defaultdict(int))
tot = defaultdict(int)
for r in rows:
    if not r or r[0] in ("Address", "Kernel Name") or len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    tok = src.split()
    op = tok[0] if tok else "?"
    if op.startswith("@"):
        op = tok[1] if len(tok) > 1 else op
    op = op.split(".")[0]
    for rs in reasons:
        try:
            v = int(r[ix[rs]])
        except ValueError:
            continue
        by_op[op][rs] += v
        tot[rs] += v
allv = sum(tot.values())
print("total samples", allv)
print("by reason:", ", ".join(f"{k[6:]} {100*v/allv:.1f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
ops = sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:22]
for op, d in ops:
    s = sum(d.values())
    top = ", ".join(f"{k[6:]} {100*v/s:.0f}%" for k, v in sorted(d.items(), key=lambda kv: -kv[1])[:4] if v)
    print(f"{op:10s} {100*s/allv:5.1f}%  {top}")
