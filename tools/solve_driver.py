"""Run persistent (or graph) solves of a bench config, for ncu / compute-sanitizer captures.

    python tools/solve_driver.py [--config 2d_65536] [--max-iters 200] [--reps 2] [--graph]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_13343_b200 as H  # noqa: E402
from paper_2605_13343_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="2d_65536")
ap.add_argument("--max-iters", type=int, default=200)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--graph", action="store_true")
a = ap.parse_args()
if a.config == "3d_1m":
    fr, sigma = H.make_frame_3d(128, 128, 64, 2024, 0), 1e-3
elif a.config == "2d_262144":
    fr, sigma = H.make_frame(262144, 2024, H.test_frame_id(262144, 0)), 1e-2
else:
    fr, sigma = H.make_frame(int(a.config.split("_")[1]), 2024, 0), 1e-2
f = H.init_factors(H.build_partition(fr.n, 128), 32, H.FactorInit.jacobi_seed, sigma,
                   H.RngStream(2024, fr.frame_index, H.RngPurpose.factor_init))
dev = H.Device(0)
dev.load_csr(fr.A)
dev.load_factors(f)
dev.set_precond(2)
dev.set_solver(N.SOLVER_GRAPH if a.graph else N.SOLVER_PERSISTENT)
x = np.empty(fr.n)
for _ in range(a.reps):
    rep = dev.solve_ptr(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(max_iters=a.max_iters), None,
                        N.HOST)
print("iterations", rep.iterations, "ms", rep.wall_ms)
