#!/usr/bin/env python
"""Key counters of every kernel in an ncu report (one line per launch)."""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
     "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
     "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
SHORT = ["us", "dramR", "dramW", "dram%", "sm%", "warps%", "inst", "fp64%", "L2B", "regs", "occR", "occS", "l1%", "issue%",
         "L2hit%", "dramBW%"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(h, r))
    u = dict(zip(h, units))
    vals = []
    for m, s in zip(M, SHORT):
        v = d.get(m, "")
        un = u.get(m, "")
        try:
            x = float(v.replace(",", ""))
            if un in ("Gbyte",): x *= 1e3; un = "MB"
            if un in ("Mbyte",): un = "MB"
            if un in ("Kbyte",): x /= 1e3; un = "MB"
            if un == "msecond": x *= 1e3
            if un == "nsecond": x /= 1e3
            vals.append(f"{s}={x:.4g}")
        except ValueError:
            vals.append(f"{s}={v}")
    print(d.get("Kernel Name", "")[:34], " ".join(vals))
