"""IC(0)-PCG (ic0.cpp, the paper's classical baseline) on the GPU vs the reference's CPU path.

    python tools/bench_ic0.py [--config 3d_1m|2d_65536|...] [--steps 3] [--cpu-iters 10]

GPU: host factorization (bit-identical to ic0_factorize; set-up, timed separately), then the
whole IC(0)-PCG as one CUDA graph (sync-free triangular sweeps), device-timed with CUDA events.
CPU: the reference's own pcg_solve + ic0_applier (oracle/_ref, 1 core) on a bounded sample of
iterations, scaled by the GPU iteration count. Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2605_13343_b200 as H  # noqa: E402
from paper_2605_13343_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="3d_1m")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--cpu-iters", type=int, default=10)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
fr, _ = bench.make_inputs(cfg, 0)
t0 = time.perf_counter()
fac = H.ic0_factorize(fr.A)
fact_ms = (time.perf_counter() - t0) * 1e3
ic = H.ic0_applier(fac)
dev = ic.bind(fr.A)
import torch  # noqa: E402  (device buffers only)
b = torch.from_numpy(fr.b).cuda()
x = torch.empty_like(b)
sc = H.SolveConfig()
dev.solve_ptr(b.data_ptr(), x.data_ptr(), sc, None, N.DEVICE)  # warm-up (graph build)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = torch.cuda.ExternalStream(dev.stream())
e0.record(st)
for _ in range(a.steps):
    rep = dev.solve_ptr(b.data_ptr(), x.data_ptr(), sc, None, N.DEVICE)
e1.record(st)
e1.synchronize()
gpu_ms = e0.elapsed_time(e1) / a.steps
its = int(rep.iterations)
# one standalone apply (two sweeps), CUDA events around hfpg_ic0_apply on device buffers
r = torch.from_numpy(np.random.default_rng(0).standard_normal(fr.n)).cuda()
z = torch.empty_like(r)
N.check(N.lib.hfpg_ic0_apply(dev.h, r.data_ptr(), z.data_ptr(), N.DEVICE))
t1 = time.perf_counter()
for _ in range(5):
    N.check(N.lib.hfpg_ic0_apply(dev.h, r.data_ptr(), z.data_ptr(), N.DEVICE))
apply_ms = (time.perf_counter() - t1) * 1e3 / 5
line = {"metric": "IC(0)-PCG solve ms to 1e-8 rel. residual", "config": a.config, "n": fr.n,
        "iterations": its, "converged": bool(rep.converged), "gpu_ms_per_solve": gpu_ms,
        "gpu_ms_per_iteration": gpu_ms / max(its, 1), "gpu_apply_ms_host_timed": apply_ms,
        "host_factorization_ms": fact_ms}
try:
    from oracle.oracle import Ref
    ref = Ref()
    csr = (np.ascontiguousarray(fr.A.row_offsets, np.uint64), np.ascontiguousarray(fr.A.col_indices, np.uint32),
           np.ascontiguousarray(fr.A.values, np.float64))
    rr, _, _ = ref.pcg_solve(csr, fr.b, 3, rtol=1e-300, max_iters=a.cpu_iters)
    ms_it = rr["wall_ms"] / a.cpu_iters
    line["cpu_baseline"] = {"value": ms_it * its, "unit": "ms/solve", "cores": 1, "kind": "reference",
                            "sample": f"{a.cpu_iters} iterations of the reference pcg_solve + ic0_applier "
                                      f"(oracle/_ref, 1 core) x {its} iterations", "ms_per_iteration": ms_it}
except Exception as e:  # noqa: BLE001
    line["cpu_baseline"] = {"unavailable": str(e)}
print(json.dumps(line))
