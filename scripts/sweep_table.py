#!/usr/bin/env python
"""Print the rows of a `bench.py --sweep` JSON line as a markdown table."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"peak {d['peak_gbs']} GB/s, clocks {d['clocks']}")
print("| kernel | n | us | B/unknown | GB/s | frac |")
print("|---|---|---|---|---|---|")
for r in d["sweep"]:
    us = r.get("us_per_launch", r.get("us_per_iteration", 0))
    print(f"| {r['kernel']} | {r['n']} | {us:.1f} | {r['bytes_per_unknown']:.1f} | {r['achieved_gbs']:.0f} | {r['frac']:.3f} |")
