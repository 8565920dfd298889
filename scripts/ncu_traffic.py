"""Write profiles/ncu_traffic.json from an ncu --set full capture of the layer kernels:
per-launch dram__bytes_read.sum + dram__bytes_write.sum of k_px_layer (averaged over the captured
launches), keyed by config, with the source hash the capture was taken on (bench.py reports the
number only for matching sources).
  python scripts/ncu_traffic.py <report.ncu-rep> <config> [kernel-substring]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    rep, config = sys.argv[1], int(sys.argv[2])
    kname = sys.argv[3] if len(sys.argv) > 3 else "k_px_layer"
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    ki, ri, wi = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    unit = rows[1][ri]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    per = [(float(r[ri]) + float(r[wi])) * scale for r in rows[2:] if kname in r[ki]]
    if not per:
        raise SystemExit("no launches of " + kname)
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(path))
    except (OSError, ValueError):
        d = {}
    if d.get("src_sha16") != bench.src_hash():
        d = {}
    d["src_sha16"] = bench.src_hash()
    d["source"] = (f"ncu --set full --clock-control none, {len(per)} {kname} launches (layers 1-3 of one NO apply), "
                   "dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged")
    d.setdefault(f"config{config}", {})["k_px_layer"] = sum(per) / len(per)
    d[f"config{config}"]["per_launch_bytes"] = per
    json.dump(d, open(path, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
