#!/bin/bash
# GPU frame generator: parity tests + timing + per-kernel launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_framegen.py -q -x --timeout 60 2>&1 | tail -15 > gpurun_out/framegen_tests.txt
cat gpurun_out/framegen_tests.txt
timeout 180 python tools/framegen_bench.py --reps 5 > gpurun_out/framegen_bench.jsonl 2> gpurun_out/framegen_bench.err
cat gpurun_out/framegen_bench.jsonl; tail -5 gpurun_out/framegen_bench.err
cat > /tmp/fg1.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_2605_13343_b200 as H
d = H.Device(0)
d.frame_gpu(1 << 20, 0, 1); d.frame_gpu(1 << 20, 0, 2)
d.frame_gpu_3d(256, 256, 256, 0, 1)
PY
timeout 180 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/framegen_launches.csv python /tmp/fg1.py > /dev/null 2>&1
python - <<'PY'
import csv
rows = [r for r in csv.DictReader(l for l in open("gpurun_out/framegen_launches.csv") if l.startswith('"'))]
for r in rows:
    print(r["ID"], r["Kernel Name"][:50], r["Metric Value"])
PY
