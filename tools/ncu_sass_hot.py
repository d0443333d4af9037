"""Top SASS instructions of an ncu report by warp-stall samples (needs --set full / source).

    python tools/ncu_sass_hot.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
si, ai, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
data = []
for k, r in enumerate(rows[1:]):
    try:
        data.append((int(r[si] or 0), k, r[ai].strip(), int(r[ei] or 0)))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot}, instructions {len(data)}")
for smp, k, src, ex in sorted(data, reverse=True)[:top]:
    print(f"{100 * smp / tot:5.1f}%  #{k:5d}  exec {ex:9d}  {src[:90]}")
