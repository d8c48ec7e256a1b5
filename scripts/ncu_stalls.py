"""Stall-reason totals (warp-state samples) of one ncu capture, optionally per SASS line range.

    python scripts/ncu_stalls.py REP [LINE_LO LINE_HI]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 1 << 30)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
for k, r in enumerate(rows[:5]):
    if "Source" in r:
        h, start = r, k + 1
        break
data = [r for r in rows[start:] if len(r) == len(h)]
idx = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = {}
for ln, r in enumerate(data):
    if not lo <= ln <= hi:
        continue
    for i in idx:
        try:
            tot[h[i]] = tot.get(h[i], 0) + float(r[i])
        except ValueError:
            pass
s = sum(tot.values()) or 1
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
    print(f"{k:28s} {v:8.0f} {100 * v / s:5.1f}%")
