#!/usr/bin/env python
"""Per-kernel warp-stall hotspots (SASS) from an ncu --set full report: python scripts/ncu_hotspots.py rep [top]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 10
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
cur = hdr = None; data = collections.defaultdict(list)
for r in csv.reader(io.StringIO(txt)):
    if not r: continue
    if r[0] == "Kernel Name": cur = r[1]; continue
    if r[0] == "Address": hdr = r; continue
    if hdr and cur: data[cur].append(dict(zip(hdr, r)))
for k, v in data.items():
    tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in v) or 1
    st = collections.Counter()
    for d in v:
        for key in d:
            if key.startswith("stall_") and "Not Issued" not in key:
                try: st[key[6:]] += int(d[key] or 0)
                except ValueError: pass
    print(f"== {k[:90]}  samples={tot}")
    print("   stalls:", ", ".join(f"{a} {100*b/tot:.0f}%" for a, b in st.most_common(6)))
    idx = sorted(range(len(v)), key=lambda i: -int(v[i]["Warp Stall Sampling (All Samples)"] or 0))[:top]
    for i in sorted(idx):
        d = v[i]
        print(f"   {i:5d} {100*int(d['Warp Stall Sampling (All Samples)'] or 0)/tot:5.1f}%  {d['Source'][:76]}")
