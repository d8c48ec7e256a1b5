"""Per-SASS-line instruction counts and stall samples of one ncu capture.

    python scripts/ncu_src.py REP [N_UNITS]   (N_UNITS: divide counts, e.g. particles)
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isamp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) > ia and r[ia].isdigit()]
ti = sum(int(r[ia]) for r in data)
ts = sum(int(r[isamp]) for r in data) or 1
print(f"# total warp instr {ti} ({ti / units:.2f} per unit), stall samples {ts}")
for idx, r in enumerate(data):
    print(f"{idx:4d} {int(r[ia]) / units:7.3f} {100 * int(r[isamp]) / ts:5.1f}  {r[1].strip()[:80]}")
