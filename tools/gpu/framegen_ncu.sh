#!/bin/bash
# per-kernel device times of the GPU frame generator (2D 1M and 3D 256^3)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_framegen.py -q -k "regenerate or errors" 2>&1 | tail -3
cat > /tmp/fg1.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_2605_13343_b200 as H
d = H.Device(0)
d.frame_gpu(1 << 20, 0, 1); d.frame_gpu(1 << 20, 0, 2)
d.frame_gpu_3d(256, 256, 256, 0, 1)
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/framegen_launches.csv python /tmp/fg1.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.DictReader(l for l in open("gpurun_out/framegen_launches.csv") if l.startswith('"'))]
for r in rows:
    print(r["ID"], r["Kernel Name"][:60], r["Metric Value"])
PY
