#!/usr/bin/env python
"""Summarise ncu outputs into markdown for profiles/.

  python scripts/ncu_summary.py launches <launches.csv>          # per-kernel share of the launch list
  python scripts/ncu_summary.py full <report.ncu-rep> [regex]    # key counters of a --set full capture
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_shared_mem",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__inst_executed.sum"]


def to_ns(v, unit):
    v = float(v.replace(",", ""))
    return v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    H = rows[hdr]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) != len(H):
            continue
        d = dict(zip(H, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"^void ", "", d["Kernel Name"].split("(")[0])
        tot[name] += to_ns(d["Metric Value"], d["Metric Unit"])
        cnt[name] += 1
    T = sum(tot.values())
    out = ["| kernel | launches | mean us/launch | share of listed device time |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| `{k}` | {cnt[k]} | {v / 1e3 / cnt[k]:.1f} | {100 * v / T:.1f}% |")
    return "\n".join(out)


def full(path, regex=None):
    cmd = ["ncu", "-i", path, "--page", "raw", "--csv"]
    txt = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    H = rows[0]
    out = []
    for r in rows[2:]:
        d = dict(zip(H, r))
        name = d.get("Kernel Name", "")
        if regex and not re.search(regex, name):
            continue
        out.append(f"### `{name[:100]}`\n")
        out.append("| metric | value |\n|---|---|")
        for k in KEYS:
            if k in d:
                out.append(f"| {k} | {d[k]} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        print(full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None))
