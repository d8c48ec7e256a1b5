"""Summarise ncu captures (gpurun_out/) into committed profiles/ files.

    python scripts/ncu_summary.py TAG

Reads gpurun_out/launches_TAG.csv (per-launch gpu__time_duration.sum) and
gpurun_out/full_<kernel>_TAG.ncu-rep (--set full), writes
profiles/TAG_launches.txt, profiles/TAG_ncu.md and profiles/force_dram_bytes.json
(dram bytes per k_force launch, the bench's roofline "traffic").
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("Duration", "gpu__time_duration.sum"),
    ("DRAM read bytes", "dram__bytes_read.sum"),
    ("DRAM write bytes", "dram__bytes_write.sum"),
    ("DRAM throughput %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("SM throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("Issue slots busy %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("Executed IPC", "sm__inst_executed.avg.per_cycle_active"),
    ("Warp instructions", "smsp__inst_executed.sum"),
    ("Achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("Registers/thread", "launch__registers_per_thread"),
    ("L1 hit %", "l1tex__t_sector_hit_rate.pct"),
    ("L2 hit %", "lts__t_sector_hit_rate.pct"),
    ("Avg active threads/warp", "smsp__thread_inst_executed_per_inst_executed.ratio"),
    ("Global ld useful bytes/sector", "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio"),
    ("Global ld L1 sector hit %", "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct"),
]


def raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        d["_units"] = dict(zip(hdr, units))
        out.append(d)
    return out


def launches(tag):
    p = os.path.join(OUT, f"launches_{tag}.csv")
    rows = list(csv.reader(open(p)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                k = d["Kernel Name"].split("(")[0]
                agg[k][0] += 1
                agg[k][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none, "
             f"scripts/prof_run.py 20 (C3 4,194,304 particles: setup + 20 steps, 2 rebuilds)",
             "# cold-cache, serialised per-launch times: compare SHARES, not absolutes",
             "# total_ns   launches  share  kernel"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{t:12.0f} {c:8d} {100 * t / tot:6.1f}%  {k}")
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    return agg


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    agg = launches(tag)
    md = [f"# ncu summary `{tag}` (B200, --set full --clock-control none)", ""]
    force_bytes, force_extra = None, {}
    for f in sorted(os.listdir(OUT)):
        if not (f.startswith("full_") and f.endswith(f"_{tag}.ncu-rep")):
            continue
        for d in raw(os.path.join(OUT, f)):
            name = d.get("Kernel Name", "?").split("(")[0]
            md.append(f"## {name}  ({f})")
            md.append("")
            md.append("| metric | value |")
            md.append("|---|---|")
            for label, m in METRICS:
                if m in d:
                    md.append(f"| {label} | {d[m]} {d['_units'].get(m, '')} |")
            try:
                sec = float(d["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"].replace(",", ""))
                req = float(d["l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"].replace(",", ""))
                md.append(f"| Global ld sectors/request | {sec / max(req, 1):.2f} |")
            except (KeyError, ValueError):
                pass
            try:
                rb = float(d["dram__bytes_read.sum"].replace(",", ""))
                wb = float(d["dram__bytes_write.sum"].replace(",", ""))
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rb *= scale.get(d["_units"].get("dram__bytes_read.sum", "byte"), 1)
                wb *= scale.get(d["_units"].get("dram__bytes_write.sum", "byte"), 1)
                md.append(f"| DRAM bytes per launch | {rb + wb:.4g} |")
                if "k_force" in name and force_bytes is None:
                    force_bytes = rb + wb
                    force_extra = {
                        "kernel_name": name,
                        "issue_slots_busy_pct": float(d.get("sm__inst_issued.avg.pct_of_peak_sustained_active", "nan")),
                        "warp_instructions": float(d.get("smsp__inst_executed.sum", "nan").replace(",", "")),
                        "dram_throughput_pct": float(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "nan")),
                        "l2_hit_pct": float(d.get("lts__t_sector_hit_rate.pct", "nan")),
                    }
            except (KeyError, ValueError):
                pass
            md.append("")
    open(os.path.join(PROF, f"{tag}_ncu.md"), "w").write("\n".join(md) + "\n")
    if force_bytes is not None:
        json.dump({"tag": tag, "kernel": "k_force", "bytes_per_launch": force_bytes, **force_extra,
                   "source": f"profiles/{tag}_ncu.md (dram__bytes_read.sum + dram__bytes_write.sum)"},
                  open(os.path.join(PROF, "force_dram_bytes.json"), "w"), indent=1)
    print(open(os.path.join(PROF, f"{tag}_launches.txt")).read())
    print("\n".join(md[:80]))


if __name__ == "__main__":
    main(sys.argv[1])
