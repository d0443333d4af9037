#!/bin/bash
# Training kernels: bit-exact tests, then loss+gradient timings -> gpurun_out/train.jsonl
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py -x -q -m gpu 2>&1 | tail -3
for n in 8192 65536; do timeout 600 python tools/bench_train.py --n $n >> gpurun_out/train.jsonl 2>>gpurun_out/train.err; done
cat gpurun_out/train.jsonl | cut -c1-300; tail -5 gpurun_out/train.err
# per-stage launch list of the same run (times under ncu are serialised, cold-cache)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/train_launches.csv python tools/bench_train.py --n 65536 --cpu 0 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.DictReader(open("gpurun_out/train_launches.csv")) if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = collections.OrderedDict()
for r in rows:
    k = r["Kernel Name"][:90]
    agg.setdefault(k, [0, 0.0]); agg[k][0] += 1; agg[k][1] += float(r["Metric Value"].replace(",", ""))
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t/1e3:10.1f} us  x{c:3d}  {k}")
PY
