"""Compact view of an ncu report's details page: kernel, section, metric, value.

    python tools/ncu_brief.py report.ncu-rep [--grep REGEX]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
rx = re.compile(sys.argv[sys.argv.index("--grep") + 1]) if "--grep" in sys.argv else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
ki, si, mi, ui, vi = (h.index(c) for c in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
last = None
for r in rows[1:]:
    if len(r) <= vi:
        continue
    if r[ki] != last:
        print("==", r[ki][:100])
        last = r[ki]
    line = f"{r[si][:28]:28s} {r[mi][:48]:48s} {r[vi]:>14s} {r[ui]}"
    if rx is None or rx.search(line):
        print(line)
