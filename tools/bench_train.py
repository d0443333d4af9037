"""One training context (probe batch -> loss + gradient, adjoint.cpp:250) on the GPU vs the
reference CPU loss_gradient, and the AdamW step. Prints one JSON line.

    python tools/bench_train.py [--n 65536] [--kz 0 (= probe_count(n))] [--kind 0|1]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_13343_b200 as H  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--kz", type=int, default=0)
ap.add_argument("--kind", type=int, default=0)
ap.add_argument("--cpu", type=int, default=1)
a = ap.parse_args()
n = a.n
kz = a.kz or max(64, math.ceil(math.sqrt(n)))  # probes.cpp:8-12 probe_count
fr = H.make_frame(n, 2024, 0)
dev = H.Device(0)
dev.load_csr(fr.A)
f = H.init_factors(H.build_partition(n, 128), 32, H.FactorInit.jacobi_seed, 1e-2,
                   H.RngStream(2024, 0, H.RngPurpose.factor_init))
P = f.data.astype(np.float64)
Z = np.random.default_rng(1).standard_normal(n * kz)
H.loss_gradient(P, Z, kz, H.LossKind(a.kind), dev, norm_a=8.0)  # warm-up
torch.cuda.synchronize()
t = time.perf_counter()
reps = 3
for _ in range(reps):
    r = H.loss_gradient(P, Z, kz, H.LossKind(a.kind), dev, norm_a=8.0)
gpu_ms = (time.perf_counter() - t) * 1e3 / reps
# the same call on device-resident arrays (where = DEVICE): the kernels alone, no PCIe copies
import ctypes as C  # noqa: E402
from paper_2605_13343_b200 import _native as N  # noqa: E402
dP, dZ = torch.from_numpy(P).cuda(), torch.from_numpy(Z).cuda()
dG = torch.empty_like(dP)
lo, dg = N.dbl(), N.i32()
def dev_call():
    rc = N.lib.hfpg_loss_gradient(dev.h, dP.data_ptr(), 128, 32, 0.0, dZ.data_ptr(), kz, a.kind, 8.0,
                                  C.byref(lo), C.byref(dg), dG.data_ptr(), N.DEVICE)
    assert rc == 0, rc
dev_call()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(reps):
    dev_call()
torch.cuda.synchronize()
dev_ms = (time.perf_counter() - t) * 1e3 / reps
assert np.array_equal(dG.cpu().numpy(), r.grad)
# forward-pass FLOPs (2 per multiply-add): leaf 2 x 2 L^2 n/L kz... summed per stage
K = n // 128
fwd = 2 * kz * (2 * K * 128 * 128 + 2 * 2 * K * 128 * 32 + 4 * (K - 1) * 32 * 16)
line = {"metric": "loss_gradient ms per probe batch (host arrays in/out)", "n": n, "kz": kz, "kind": a.kind,
        "gpu_ms": gpu_ms, "gpu_device_ms": dev_ms, "loss": r.loss, "approx_gflop": 3 * fwd / 1e9}
if a.cpu:
    try:
        from oracle.oracle import Ref
        ref = Ref()
        csr = (np.ascontiguousarray(fr.A.row_offsets, np.uint64), np.ascontiguousarray(fr.A.col_indices, np.uint32),
               np.ascontiguousarray(fr.A.values, np.float64))
        t = time.perf_counter()
        loss, _, g = ref.loss_gradient(csr, P, Z, kz, a.kind, 8.0)
        line["cpu_baseline"] = {"ms": (time.perf_counter() - t) * 1e3, "cores": 1, "kind": "reference",
                                "loss": loss, "grad_rel_diff": float(np.linalg.norm(g - r.grad) / np.linalg.norm(g))}
    except Exception as e:  # noqa: BLE001
        line["cpu_baseline"] = {"unavailable": str(e)}
# AdamW on the packed width, device buffers
tp, tg, m1, m2 = (torch.from_numpy(x).cuda() for x in (P.copy(), r.grad.copy(), np.zeros_like(P), np.zeros_like(P)))
H.adamw_step(dev, tp.data_ptr(), tg.data_ptr(), m1.data_ptr(), m2.data_ptr(), len(P), 1, 1e-3)
torch.cuda.synchronize()
t = time.perf_counter()
H.adamw_step(dev, tp.data_ptr(), tg.data_ptr(), m1.data_ptr(), m2.data_ptr(), len(P), 2, 1e-3)
line["adamw_ms"] = (time.perf_counter() - t) * 1e3
print(json.dumps(line))
