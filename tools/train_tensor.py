"""Train a factor tensor on the GPU (train_factors, train.cpp:29-217) and write it as HFTC.

    python tools/train_tensor.py --n 1024 --steps 2000 [--frames 4] [--lr 2e-3] [--out ck.hftc]

Frames: train_frame_id(n, i), i < frames (frame.hpp:85-87); held-out: test_frame_id(n, 0).
Prints one JSON line: the log, wall time, and the held-out iterations of the trained tensor
against Jacobi (graph PCG on the same frame)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2605_13343_b200 as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--steps", type=int, default=2000)
ap.add_argument("--frames", type=int, default=4)
ap.add_argument("--lr", type=float, default=2e-3)
ap.add_argument("--contexts", type=int, default=4)
ap.add_argument("--log-every", type=int, default=100)
ap.add_argument("--seed", type=int, default=2024)
ap.add_argument("--out", default="")
ap.add_argument("--acceptance", action="store_true",
                help="the reference's acceptance criterion 10 (acceptance.cpp:378-420): make_frame(n, 2024, 0), "
                     "default TrainConfig, 20000 steps max, eval every 200 steps, stop at half Jacobi's iterations")
a = ap.parse_args()
if a.acceptance:
    f0 = H.make_frame(a.n, 2024, 0)
    jac0 = H.pcg_solve(f0.A, f0.b, H.jacobi_applier(f0.A))
    fr, ev = [f0], f0
    cfg = H.TrainConfig(max_steps=20000, log_every=100, eval_every_logs=2, stop_at_iters=jac0.iterations // 2)
    a.seed = 2024
else:
    fr = [H.make_frame(a.n, 2024, H.train_frame_id(a.n, i)) for i in range(a.frames)]
    ev = H.make_frame(a.n, 2024, H.test_frame_id(a.n, 0))
    cfg = H.TrainConfig(max_steps=a.steps, log_every=a.log_every, lr=a.lr, contexts_per_step=a.contexts)
t0 = time.perf_counter()
res = H.train_factors(fr, cfg, seed=a.seed, eval_frame=ev)
wall = time.perf_counter() - t0
jac = H.pcg_solve(ev.A, ev.b, H.jacobi_applier(ev.A))
trained = H.pcg_solve(ev.A, ev.b, H.factor_applier(res.factors, ev.A))
if a.out:
    H.write_checkpoint(res.factors, a.out, json.dumps({"trained": True, "n": a.n, "seed": a.seed, "frames": a.frames,
                                                      "steps": res.history.total_steps}))
print(json.dumps({"n": a.n, "acceptance": a.acceptance, "reached_target": res.history.reached_target,
                  "steps": res.history.total_steps, "wall_s": wall, "ms_per_step": 1e3 * wall / max(1, res.history.total_steps),
                  "jacobi_iterations": jac.iterations, "trained_iterations": trained.iterations,
                  "trained_converged": trained.converged, "auto_stopped": res.history.auto_stopped,
                  "log": [e.__dict__ for e in res.history.entries]}))
