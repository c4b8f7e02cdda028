"""Summarise an ncu report (--set full) or an ncu launch-list CSV into profiles/.

  python tools/ncu_summary.py rep  <file.ncu-rep>  [--out profiles/x.txt]
  python tools/ncu_summary.py launches <launches.csv> [--out profiles/x.txt]
"""
import argparse
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
]


def rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        out.append(f"kernel: {name}")
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                out.append(f"  {m:66s} {vals[i]:>22s} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                if v > 0:
                    stalls.append((v, h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(v for v, _ in stalls) or 1
        out.append("  stall samples (share):")
        for v, h in sorted(stalls, reverse=True)[:8]:
            out.append(f"    {h:40s} {100 * v / tot:5.1f}%")
    return "\n".join(out)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[r[ki]][0] += 1
        agg[r[ki]][1] += v
    tot = sum(v[1] for v in agg.values())
    out = ["launches  total_ms  share  avg_ms  kernel"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{c:8d} {v / 1e6:9.3f} {100 * v / tot:5.1f}% {v / c / 1e6:7.3f}  {k[:110]}")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind", choices=["rep", "launches"])
    ap.add_argument("path")
    ap.add_argument("--out")
    a = ap.parse_args()
    text = rep(a.path) if a.kind == "rep" else launches(a.path)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    sys.exit(main())
