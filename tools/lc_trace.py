"""Per-CTA phase timeline of k_leaf_coarse (HFPG_LEAF_COARSE=1) at 3D 1M: %globaltimer at the
start, end of phase 1 and end of each CTA (hfpg_set_trace), from standalone iterations."""
import json
import os
import sys

os.environ["HFPG_LEAF_COARSE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2605_13343_b200 as H  # noqa: E402
from paper_2605_13343_b200 import _native as N  # noqa: E402

fr, f = bench.make_inputs(bench.CONFIGS["3d_1m"], 0)
dev = H.Device(0)
dev.load_csr(fr.A)
dev.load_factors(f)
dev.set_precond(2)
x = np.empty(fr.n)
dev.solve_ptr(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(max_iters=4), None, N.HOST)
N.check(N.lib.hfpg_set_trace(dev.h, 12 * 148))
ms = np.zeros(4, np.float32)
N.check(N.lib.hfpg_profile_iteration(dev.h, 1, ms.ctypes.data))
tr = np.zeros(12 * 148, np.uint64)
N.check(N.lib.hfpg_get_trace(dev.h, tr.ctypes.data, 12 * 148))
t = tr.reshape(148, 12).astype(np.int64)
t0 = t[:, 0].min()
p1 = (t[:, 1] - t0) / 1e3
end = (t[:, 2] - t0) / 1e3
start = (t[:, 0] - t0) / 1e3
print(json.dumps({"kernel_ms": ms.tolist(), "start_us": [float(start.min()), float(start.max())],
                  "phase1_end_us": [float(p1.min()), float(np.median(p1)), float(p1.max())],
                  "end_us": [float(end.min()), float(np.median(end)), float(end.max())],
                  "f_leaves": [int(t[:, 3].min()), int(t[:, 3].max())],
                  "unit_us_median": {k: float(np.median(t[:, 4 + q]) / 1e3)
                                     for q, k in enumerate(["F", "sum", "tile", "F_wait"])},
                  "f_sub_cycles_per_leaf": {k: float(np.median(t[:, 8 + q] / t[:, 3]))
                                            for q, k in enumerate(["issue", "chain", "fc"])},
                  "sm_ghz": float(np.median(t[:, 11] / (t[:, 2] - t[:, 0]))),
                  "unit_us_max": {k: float(t[:, 4 + q].max() / 1e3)
                                  for q, k in enumerate(["F", "sum", "tile", "F_wait"])}}))
