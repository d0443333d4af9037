"""Small invocations of every device path, for compute-sanitizer (memcheck / racecheck /
synccheck): fast + generic apply, SpMV, graph and persistent PCG, a 2-rank partitioned group
solve, the toy-network forward (tcgen05 GEMMs + attention), the IC(0) sweeps, the GPU crc32 and
the MPPF / HFTC device loaders.

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py [--only NAME]
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
ap.add_argument("--only", default="")
a = ap.parse_args()


def seeded(n, seed=7, frame=0, L=128, Ls=32):
    return H.init_factors(H.build_partition(n, L), Ls, H.FactorInit.jacobi_seed, 1e-2,
                          H.RngStream(seed, frame, H.RngPurpose.factor_init))


def run(name, fn):
    if a.only and a.only != name:
        return
    fn()
    print("ok", name, flush=True)


def apply_fast():
    fr = H.make_frame(4096, 7, 0)
    ap_ = H.factor_applier(seeded(4096), fr.A)
    ap_(fr.b)
    ap_.dev.spmv(fr.b)


def apply_generic():
    fr = H.make_frame(2048, 7, 1)
    f = H.init_factors(H.build_partition(2048, 64), 16, H.FactorInit.jacobi_seed, 1e-2,
                       H.RngStream(7, 1, H.RngPurpose.factor_init))
    H.factor_applier(f, fr.A)(fr.b)


def solve(kind, n=8192):
    def go():
        fr = H.make_frame(n, 7, 2)
        d = H.Device(0)
        d.load_csr(fr.A)
        d.load_factors(seeded(n, frame=2))
        d.set_precond(2)
        d.set_solver(kind)
        x = np.empty(fr.n)
        d.solve_ptr(fr.b.ctypes.data, x.ctypes.data, H.SolveConfig(max_iters=6), None, N.HOST)
    return go


def iteration_kernels():
    # the graph's loop kernels (spmv<loop>, leaf<loop>, sums, tiles, prolong<loop>) launched
    # standalone: racecheck / synccheck do not follow conditional-node graph bodies
    fr = H.make_frame(8192, 7, 5)
    d = H.Device(0)
    d.load_csr(fr.A)
    d.load_factors(seeded(8192, frame=5))
    d.set_precond(2)
    ms = np.zeros(4, np.float32)
    N.check(N.lib.hfpg_profile_iteration(d.h, 2, ms.ctypes.data))


def group_apply():
    fr = H.make_frame(8192, 7, 6)
    H.PartitionGroup(fr.A, 4, factors=seeded(8192, frame=6)).apply(fr.b)


def group():
    fr = H.make_frame(8192, 7, 3)
    g = H.PartitionGroup(fr.A, 2, factors=seeded(8192, frame=3))
    g.solve(fr.b, H.SolveConfig(max_iters=6))
    g.apply(fr.b)


def toynet():
    fr = H.make_frame(1024, 7, 4)
    H.toynet_forward(fr, H.build_partition(1024, 128), 32, H.ToynetConfig(), weight_seed=0,
                     trace=H.ToynetTrace())


def ic0():
    fr = H.make_frame(4096, 7, 8)
    ap_ = H.ic0_applier(H.ic0_factorize(fr.A))
    ap_.bind(fr.A)
    ap_(fr.b)
    H.pcg_solve(fr.A, fr.b, ap_, H.SolveConfig(max_iters=5))


def io():
    import tempfile
    import torch
    d = H.Device(0)
    x = torch.arange(100000, dtype=torch.uint8, device="cuda")
    d.crc32((x.data_ptr() + 3, 99990))
    fr = H.make_frame(4096, 7, 9)
    with tempfile.TemporaryDirectory() as t:
        H.write_mppf(fr, os.path.join(t, "f.mppf"))
        d.load_mppf(os.path.join(t, "f.mppf"))
        f = seeded(4096, frame=9)
        H.write_checkpoint(f, os.path.join(t, "m.hftc"))
        d.load_checkpoint(os.path.join(t, "m.hftc"))


run("apply_fast", apply_fast)
run("apply_generic", apply_generic)
run("solve_graph", solve(N.SOLVER_GRAPH))
run("solve_persistent", solve(N.SOLVER_PERSISTENT))
run("solve_persistent_pipe", solve(N.SOLVER_PERSISTENT, 65536))  # 3-4 leaves per CTA: the pipelined leaf phase
run("iteration_kernels", iteration_kernels)
run("group_apply", group_apply)
run("group", group)
run("toynet", toynet)
run("ic0", ic0)
run("io", io)
