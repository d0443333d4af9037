"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/ncu_launch_table.py gpurun_out/launches_x.csv [--regex NAME]

Prints one row per kernel name: launches, total us, mean us, share of the listed time.
"""
import csv
import io
import re
import sys
from collections import OrderedDict


def load(path):
    txt = open(path, errors="replace").read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    out = []
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = v / 1e3 if unit in ("nsecond", "ns") else v * 1e3 if unit in ("msecond", "ms") else v
        out.append((r[ki], us))
    return out


def main():
    path = sys.argv[1]
    rx = re.compile(sys.argv[sys.argv.index("--regex") + 1]) if "--regex" in sys.argv else None
    launches = load(path)
    agg = OrderedDict()
    for name, us in launches:
        short = name.split("(")[0][:70]
        if rx and not rx.search(name):
            continue
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':70s} {'n':>5s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:70s} {c:5d} {t:10.1f} {t / c:9.2f} {100 * t / tot:5.1f}%")
    print(f"{'TOTAL':70s} {sum(a[0] for a in agg.values()):5d} {tot:10.1f}")


if __name__ == "__main__":
    main()
