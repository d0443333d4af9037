"""Summarise ncu reports brought back in gpurun_out/ into profiles/ (tracked).

    python tools/ncu_summary.py <round-tag> [config]

Reads gpurun_out/prof_*.ncu-rep (--set full captures) and gpurun_out/launches_*.csv (the
gpu__time_duration launch list), writes profiles/<tag>_ncu_summary.md, copies the launch list
to profiles/<tag>_launches.csv and records per-launch DRAM traffic in profiles/ncu_traffic.json
(bench.py's roofline "traffic" field).
"""
import csv
import glob
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2:]


def main(tag, config="3d_1m"):
    os.makedirs(OUT, exist_ok=True)
    lines = [f"# ncu summary — {tag} ({config})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(gpurun), driver `tools/iter_driver.py` (standalone launches of one factor-PCG "
             "iteration's kernels). ncu flushes caches before each profiled launch, so these are "
             "cold-cache numbers; compare shares, not absolutes, with the in-graph bench.", ""]
    traffic = {}
    for rep in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "prof_*.ncu-rep"))):
        hdr, units, rows = raw(rep)
        stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
        for r in rows:
            name = r[hdr.index("Kernel Name")]
            lines += [f"## `{name}`", "", "| metric | value |", "|---|---|"]
            for m, label in METRICS:
                if m in hdr:
                    lines.append(f"| {label} (`{m}`) | {r[hdr.index(m)]} {units[hdr.index(m)]} |")
            top = sorted(((float(r[hdr.index(h)] or 0), h) for h in stalls), reverse=True)[:4]
            lines.append("| top stalls (warps per issue) | " + ", ".join(
                f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
                for v, h in top) + " |")
            lines.append("")
            short = name.split("(")[0].replace("void ", "").split("<")[0]
            try:
                rd = float(r[hdr.index("dram__bytes_read.sum")])
                wr = float(r[hdr.index("dram__bytes_write.sum")])
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd *= scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
                wr *= scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
                traffic.setdefault(short, rd + wr)
            except (ValueError, KeyError):
                pass
    for f in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "launches_*.csv"))):
        dst = os.path.join(OUT, f"{tag}_{os.path.basename(f)}")
        shutil.copy(f, dst)
        lines.append(f"Launch list: `{os.path.relpath(dst, ROOT)}`")
    open(os.path.join(OUT, f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    tj = os.path.join(OUT, "ncu_traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    d[config] = {k: v for k, v in traffic.items()}
    d[config]["_source"] = f"{tag} ncu --set full captures (cold cache), bytes per launch"
    json.dump(d, open(tj, "w"), indent=1)
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01", sys.argv[2] if len(sys.argv) > 2 else "3d_1m")
