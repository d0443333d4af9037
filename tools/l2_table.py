"""Summarise gpurun_out/l2_<arm>.csv (tools/gpu/l2reuse.sh): per kernel, the mean of the last
three launches' duration (us), DRAM read (MB) and L2 sector hit rate (%)."""
import collections
import csv
import io
import sys

arm = sys.argv[1]
txt = open(f"gpurun_out/l2_{arm}.csv").read().splitlines()
i = [k for k, l in enumerate(txt) if l.startswith('"ID"')][0]
agg = collections.defaultdict(list)
for r in csv.DictReader(io.StringIO("\n".join(txt[i:]))):
    agg[(r["Kernel Name"].split("(")[0].replace("void ", "")[:16], r["Metric Name"])].append(
        float(r["Metric Value"].replace(",", "")))
out = {}
for (k, m), v in sorted(agg.items()):
    out.setdefault(k, {})[m] = sum(v[-3:]) / len(v[-3:])
print(arm, {k: (round(v["gpu__time_duration.sum"] / 1e3, 1), round(v["dram__bytes_read.sum"] / 1e6, 1),
                round(v["lts__t_sector_hit_rate.pct"], 1)) for k, v in out.items()})
