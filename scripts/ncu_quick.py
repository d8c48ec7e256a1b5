"""Headline metrics + stall ratios of one ncu capture: python scripts/ncu_quick.py REP"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct"]
for v in rows[2:]:
    for k, x in zip(h, v):
        if k in want or ("stalled" in k and k.endswith("per_issue_active.ratio") and float(x or 0) > 0.3):
            print(f"  {k:70s} {x}")
