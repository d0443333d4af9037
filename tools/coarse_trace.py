"""Per-CTA phase timeline of k_coarse_coop at 3D 1M (hfpg_set_trace): %globaltimer at entry,
after the group roots (A), after the group-internal tiles (B), after the grid wait, after the
tiles above the groups (C) and at exit; medians / maxima over the CTAs, µs from the first entry."""
import json
import os
import sys

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
G = 296
N.check(N.lib.hfpg_set_trace(dev.h, 8 * G))
ms = np.zeros(4, np.float32)
N.check(N.lib.hfpg_profile_iteration(dev.h, 1, ms.ctypes.data))
tr = np.zeros(8 * G, np.uint64)
N.check(N.lib.hfpg_get_trace(dev.h, tr.ctypes.data, 8 * G))
t = tr.reshape(G, 8).astype(np.int64)
t0 = t[:, 0].min()
rel = (t[:, :6] - t0) / 1e3
names = ["entry", "after_A", "after_B", "after_wait", "after_C", "exit"]
out = {"kernel_ms": ms.tolist()}
for q, nm in enumerate(names):
    col = rel[:, q][t[:, q] > 0]
    out[nm] = [round(float(col.min()), 2), round(float(np.median(col)), 2), round(float(col.max()), 2)] if len(col) else None
print(json.dumps(out))
