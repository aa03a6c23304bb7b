#!/usr/bin/env python3
"""Summarise ncu captures for profiles/ (run in the build container on
reports brought back in gpurun_out/).

    python scripts/ncu_summary.py gpurun_out/ring_vec.ncu-rep > profiles/r01_ring_vec.txt
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv > profiles/r01_launches.txt
"""
import csv
import io
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__cluster_size",
    "launch__cluster_max_active", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
]
STALL = re.compile(r"^smsp__pcsamp_warps_issue_stalled_([a-z_]+)$")


def summarise_report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        print(f"kernel: {d.get('Kernel Name', '?')[:160]}")
        for m in METRICS:
            if m in d and d[m] not in ("", "n/a"):
                print(f"  {m:60s} {d[m]:>18s} {units[hdr.index(m)]}")
        stalls = {STALL.match(h).group(1): float(d[h]) for h in hdr
                  if STALL.match(h) and not h.endswith("_not_issued") and d[h] not in ("", "n/a")}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        print("  stall samples (top):", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in top))
        print()


def summarise_launches(path):
    agg = {}
    hdr = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                k = d["Kernel Name"]
                k = re.sub(r"\(.*", "", k)[:110]
                agg.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")))
                unit = d.get("Metric Unit", "")
    tot = sum(sum(v) for v in agg.values())
    print(f"{'launches':>8} {'mean':>12} {'total':>12} {'share':>6}  kernel   (unit {unit}, ncu serialised cold-cache times)")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v):12.1f} {sum(v):12.1f} {100 * sum(v) / tot:5.1f}%  {k}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        summarise_launches(sys.argv[2])
    else:
        for p in sys.argv[1:]:
            summarise_report(p)
