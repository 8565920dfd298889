#!/usr/bin/env python
"""Warp-stall samples of an ncu --set full capture aggregated per CUDA source line.

  python scripts/ncu_lines.py <report.ncu-rep> <kernel-name-substring> <mangled-name-substring> [top]

ncu's source page in CSV form carries no line column, so the SASS rows (in address order) are
matched by offset against `nvdisasm -g` of the in-tree library's cubin (built with -lineinfo).
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line_map(func):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2402_05598_b200", "libfcgno.so")],
                   cwd=tmp, capture_output=True)
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        m0 = re.search(r"^\.text\.(\S*" + re.escape(func) + r"\S*):", txt, re.M)
        if not m0:
            continue
        start = m0.start()
        end = txt.find("//--------------------- .text.", start)
        txt = txt[start:end if end > 0 else len(txt)]
        cur, m = None, {}
        for ln in txt.splitlines():
            g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if g:
                cur = f"{os.path.basename(g.group(1))}:{g.group(2)}"
                continue
            g = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if g:
                m[int(g.group(1), 16)] = cur
        return m
    raise SystemExit(f"function {func} not found")


def main():
    rep, kname, func = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    which = int(sys.argv[5]) if len(sys.argv) > 5 else 0   # n-th captured launch whose name matches
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows, cur, hdr, seen = [], None, None, -1
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "Kernel Name":
            cur = r[1]
            if kname in cur:
                seen += 1
            if seen != which:
                cur = None
            continue
        if r[0] == "Address":
            hdr = r
            continue
        if hdr and cur and kname in cur:
            rows.append(dict(zip(hdr, r)))
    if not rows:
        raise SystemExit("kernel not in report")
    base = min(int(d["Address"], 16) for d in rows)
    lm = line_map(func)
    per = collections.Counter()
    ins = collections.Counter()
    stall = collections.defaultdict(collections.Counter)
    tot = tot_ins = 0
    for d in rows:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        tot += s
        src = lm.get(int(d["Address"], 16) - base, "?")
        per[src] += s
        try:
            ni = int((d.get("Instructions Executed") or "0").replace(",", ""))
        except ValueError:
            ni = 0
        ins[src] += ni
        tot_ins += ni
        for k in d:
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    stall[src][k[6:]] += int(d[k] or 0)
                except ValueError:
                    pass
    print(f"samples={tot} warp-instructions={tot_ins}")
    print("stall%  inst%  line")
    for src, s in per.most_common(top):
        top3 = ", ".join(f"{k} {v * 100 // max(s, 1)}%" for k, v in stall[src].most_common(3))
        print(f"{s * 100.0 / tot:5.1f}% {ins[src] * 100.0 / max(tot_ins, 1):5.1f}%  {src:28s} {top3}")
    print("-- by instructions")
    for src, ni in ins.most_common(top):
        print(f"{ni * 100.0 / max(tot_ins, 1):5.1f}%  {src}")


if __name__ == "__main__":
    main()
