"""GPU frame generator timing vs the host generator (make_frame / make_frame_3d).

python tools/framegen_bench.py [--reps 5] -> one JSON line per size: device generate_ms
(median, events on the handle's stream), wall ms of the ABI call, host make_frame ms."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_13343_b200 as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--host", type=int, default=1)
args = ap.parse_args()
dev = H.Device(0)
for spec in [65536, 1 << 20, 1 << 22, (100, 100, 100), (128, 128, 128), (256, 256, 256)]:
    gen = (lambda f: dev.frame_gpu_3d(*spec, 0, f)) if isinstance(spec, tuple) else (lambda f: dev.frame_gpu(spec, 0, f))
    gen(0)
    dms, wms = [], []
    for r in range(args.reps):
        t = time.perf_counter()
        g = gen(r + 1)
        wms.append((time.perf_counter() - t) * 1e3)
        dms.append(g.generate_ms)
    out = {"spec": spec, "n": g.n, "nnz": g.nnz, "gpu_generate_ms": sorted(dms)[len(dms) // 2],
           "gpu_call_wall_ms": sorted(wms)[len(wms) // 2]}
    if args.host:
        t = time.perf_counter()
        (H.make_frame_3d(*spec, 0, 1) if isinstance(spec, tuple) else H.make_frame(spec, 0, 1))
        out["host_make_frame_ms"] = (time.perf_counter() - t) * 1e3
        out["host_cores"] = os.cpu_count()
    print(json.dumps(out), flush=True)
