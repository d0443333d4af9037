"""Per-phase device time of the persistent solver (k_solve) from its %globaltimer barrier trace.

    python tools/phase_trace.py [--config 2d_65536|3d_1m|2d_8192|2d_262144]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_13343_b200 as H  # noqa: E402
from paper_2605_13343_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="2d_65536")
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
dev.set_solver(N.SOLVER_PERSISTENT)
cap = 1 << 16
N.check(N.lib.hfpg_set_trace(dev.h, cap))
x = np.empty(fr.n)
for _ in range(2):
    rep = dev.solve_ptr(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(), None, N.HOST)
t = np.zeros(cap, np.uint64)
N.check(N.lib.hfpg_get_trace(dev.h, t.ctypes.data, cap))
its = int(rep.iterations)
# barriers: init [leaf, (sums,) coarse, prolong]; per iteration [spmv, leaf, (sums,) coarse, prolong] —
# K <= 1024 leaves run the coarse stage as one phase (p_coarse_phase), larger K as sums + tiles
merged = fr.n // 128 <= 1024
NI, NP = (3, 4) if merged else (4, 5)
n_bar = min(NI + NP * (its - 1) + 2, cap - 1)
t = t[: n_bar + 1].astype(np.float64)
d = np.diff(t) / 1e3  # us
init = d[:NI]
loop = d[NI: NI + NP * ((n_bar - NI) // NP)].reshape(-1, NP)
names = ["spmv", "leaf", "coarse", "prolong"] if merged else ["spmv", "leaf", "sums", "tiles", "prolong"]
out = {"config": a.config, "n": fr.n, "iterations": its, "solve_ms": rep.wall_ms,
       "init_us": dict(zip(names[1:], init.round(2).tolist())),
       "loop_us_median": dict(zip(names, np.median(loop, 0).round(2).tolist())),
       "loop_us_mean": dict(zip(names, loop.mean(0).round(2).tolist())),
       "iteration_us_median": float(np.median(loop.sum(1)))}
tp = np.zeros(cap, np.uint64)
N.check(N.lib.hfpg_get_trace(dev.h, tp.ctypes.data, cap))
pr = tp[cap - 64:].astype(np.float64)
base = pr[0] if pr[0] else 0
out["probes_us"] = {i: round((pr[i] - base) / 1e3, 2) for i in list(range(40)) + list(range(44, 60)) if pr[i]}
out["probe_cycles"] = {i: int(pr[i]) for i in range(40, 44) if pr[i]}
print(json.dumps(out))
