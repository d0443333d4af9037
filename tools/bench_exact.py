"""Cost of the bit-exact PCG (hfpg_pcg_solve_exact) against the graph solve on one config.

    python tools/bench_exact.py [--config 3d_1m] [--precond factor|ic0|jacobi]
Prints one JSON line: iterations and device ms per solve for both modes (same inputs)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2605_13343_b200 as H  # noqa: E402
from paper_2605_13343_b200 import _native as N  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="3d_1m")
ap.add_argument("--precond", default="factor")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
fr, f = bench.make_inputs(cfg, 0)
if a.precond == "factor":
    dev = H.factor_applier(f, fr.A).bind(fr.A)
elif a.precond == "ic0":
    dev = H.ic0_applier(H.ic0_factorize(fr.A)).bind(fr.A)
else:
    dev = H.jacobi_applier(fr.A).bind(fr.A)
b = torch.from_numpy(fr.b).cuda()
x = torch.empty_like(b)
sc = H.SolveConfig()
line = {"config": a.config, "precond": a.precond, "n": fr.n}
for name, exact in (("graph", False), ("exact", True)):
    dev.solve_ptr(b.data_ptr(), x.data_ptr(), sc, None, N.DEVICE, exact=exact)  # warm-up
    rep = dev.solve_ptr(b.data_ptr(), x.data_ptr(), sc, None, N.DEVICE, exact=exact)
    line[name] = {"iterations": int(rep.iterations), "ms": float(rep.wall_ms),
                  "ms_per_iteration": float(rep.wall_ms) / max(1, int(rep.iterations))}
print(json.dumps(line))
