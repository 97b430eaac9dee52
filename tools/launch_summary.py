"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): per kernel, launches,
total and mean time, share of the listed time.

    python tools/launch_summary.py profiles/r02_ncu/launches_c4.csv
"""
import collections
import csv
import re
import sys


def main():
    rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").replace("unnamed>::", "")
        name = re.sub(r"^.*::", "", name)
        t = float(r[iv].replace(",", ""))
        c, s = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, s + t)
    tot = sum(s for _, s in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'mean us':>10s} {'share':>7s}")
    for k, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {c:8d} {s / 1e6:10.3f} {s / c / 1e3:10.1f} {100 * s / tot:6.1f}%")


if __name__ == "__main__":
    main()
