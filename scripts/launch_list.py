"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-launch device time of
the last `--tail` launches, and per-kernel totals.  python scripts/launch_list.py <csv> [--tail N]"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    tail = int(sys.argv[sys.argv.index("--tail") + 1]) if "--tail" in sys.argv else 0
    rows, hdr = [], None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"]) * (1e-3 if d.get("Metric Unit") == "nsecond" else 1.0)
                rows.append((d["Kernel Name"].split("(")[0].replace("void ", ""), v))
    sel = rows[-tail:] if tail else rows
    tot = collections.Counter()
    cnt = collections.Counter()
    for name, v in sel:
        if tail:
            print(f"{v:9.1f} us  {name}")
        tot[name] += v
        cnt[name] += 1
    print("-- totals (us)")
    for name, v in tot.most_common():
        print(f"{v:9.1f}  x{cnt[name]:<3d} {name}")
    print(f"{sum(tot.values()):9.1f}  total")


if __name__ == "__main__":
    main()
