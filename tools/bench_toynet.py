"""Time the GPU toy-network forward (d128_L3_hw) and the inference -> PCG pipeline at N.

    python tools/bench_toynet.py [--n 65536] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_13343_b200 as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
fr = H.make_frame(a.n, 2024, 0)
p = H.build_partition(a.n, 128)
dev = H.Device(0)
dev.load_csr(fr.A)
times, dev_ms = [], []
for i in range(a.reps + 1):
    tr = H.ToynetTrace()
    t0 = time.perf_counter()
    H.toynet_forward(fr, p, 32, device=dev, load=True, trace=tr if i else None)
    times.append((time.perf_counter() - t0) * 1e3)
    tr2 = H.ToynetTrace(timing_only=True)
    H.toynet_forward(fr, p, 32, device=dev, load=True, trace=tr2)
    dev_ms.append(tr2.ms)
print(json.dumps({"n": a.n, "host_wall_ms": times, "device_ms_timing_only": dev_ms}))
