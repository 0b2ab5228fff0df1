"""Aggregate warp-stall samples per CUDA source line from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import subprocess
import sys
from collections import defaultdict


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur_file, cur_line, cur_src = None, None, None
    agg = defaultdict(lambda: [0, 0, ""])
    total = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if r[0]:  # a source line row
            cur_line, cur_src = r[0], r[1]
            try:
                s = int(r[4])
            except (ValueError, IndexError):
                s = 0
            key = (cur_file, int(cur_line))
            agg[key][0] += s
            agg[key][2] = cur_src.strip()[:90]
            total += s
    print(f"total samples {total}")
    for (f, ln), (s, _, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * s / total:5.1f}% {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
