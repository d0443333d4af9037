"""Small driver for ncu: builds the bench workload, runs one short solve (max_iters=4) and
then `reps` standalone factor-PCG iterations (hfpg_profile_iteration), so a profiler sees
k_spmv_tma / k_leaf_fast / k_coarse_coop / k_prolong_tma launches in isolation.

    python tools/iter_driver.py [--config 3d_1m] [--reps 3]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2605_13343_b200 as H  # noqa: E402
from paper_2605_13343_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="3d_1m")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
fr, f = bench.make_inputs(bench.CONFIGS[a.config], 0)
dev = H.Device(0)
dev.load_csr(fr.A)
dev.load_factors(f)
dev.set_precond(2)
x = np.empty(fr.n)
dev.solve_ptr(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(max_iters=4), None, N.HOST)
ms = np.zeros(4, np.float32)
N.check(N.lib.hfpg_profile_iteration(dev.h, a.reps, ms.ctypes.data))
print("per-kernel ms (spmv, leaf, coarse, prolong):", ms.tolist())
