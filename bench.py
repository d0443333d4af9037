#!/usr/bin/env python
"""Benchmark: one step = one PCG solve to rel. residual 1e-8 of a synthetic pressure-Poisson
system with the hierarchical-factor preconditioner, on B200 through libhfpg's C ABI.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3d_1m|2d_65536|2d_8192]
                  [--impl ours|reference]

Default workload (N=1): BASELINE.json configs[2] — N = 1,048,576 (128x128x64 3D 7-point
Neumann Laplacian, the bandwidth-bound apply + SpMV regime the metric's "precond-apply HBM GB/s
vs peak" half is quoted on), seeded jacobi_seed sigma=1e-2 factor tensor (L=128, L_s=32).
Under torchrun (N>1) every rank solves its own frame (frame index = rank): independent systems,
no collective on the data path ("scaling": "weak"); the barrier + max-over-ranks timing is the
only communication. `--impl reference` times the reference's own CPU code (oracle/_ref, the
unmodified reference sources) on a bounded sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG solve ms to 1e-8 rel. residual at N"
UNIT = "ms/solve"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
ITERS = os.path.join(ROOT, "tests", "golden", "ref_iterations.json")
TRAFFIC = os.path.join(ROOT, "profiles", "ncu_traffic.json")

CONFIGS = {
    "3d_1m": dict(desc="BASELINE configs[2]: N=1,048,576 3D 128x128x64 7-point pressure-Poisson "
                       "(Morton order), seeded jacobi_seed sigma=1e-3 factor tensor (sigma=1e-2 "
                       "does not converge at this N, see DESIGN.md), L=128, L_s=32",
                  dims=(128, 128, 64), sigma=1e-3, ref_key="3d_1m_s1e-3"),
    "2d_65536": dict(desc="BASELINE configs[1] solve half: N=65,536 2D make_frame(65536, 2024, 0), "
                          "seeded sigma=1e-2 factor tensor, L=128, L_s=32 (inference not included)",
                     n=65536, sigma=1e-2, ref_key="2d_65536"),
    "2d_8192": dict(desc="BASELINE configs[0] system: make_frame(8192, 2024, 0), seeded tensor",
                    n=8192, sigma=1e-2, ref_key="2d_8192"),
}


def make_inputs(cfg: dict, frame_index: int):
    import paper_2605_13343_b200 as H
    if "dims" in cfg:
        fr = H.make_frame_3d(*cfg["dims"], 2024, frame_index)
    else:
        fr = H.make_frame(cfg["n"], 2024, frame_index)
    f = H.init_factors(H.build_partition(fr.n, 128), 32, H.FactorInit.jacobi_seed, cfg["sigma"],
                       H.RngStream(2024, frame_index, H.RngPurpose.factor_init))
    return fr, f


def peaks():
    try:
        p = json.load(open(PEAKS))
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ref_iterations(key):
    try:
        return json.load(open(ITERS))[key]["factor"]["iterations"]
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "samples": len(sms), "reasons": sorted(reasons)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if os.environ.get("HFPG_BENCH_GLOO") is None else "gloo")
    return world, rank, local


def max_over_ranks(v: float, world: int, local: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------------- reference arm


def cpu_sample(cfg, fr, f, budget_s: float):
    """Time the reference's own pcg_solve loop (oracle/_ref) for a bounded number of
    iterations; returns (ms per iteration, iterations run)."""
    from oracle.oracle import Ref
    r = Ref()
    csr = (fr.A.row_offsets, fr.A.col_indices, fr.A.values)
    ms = r.pcg_time_iters(csr, fr.b, 128, 32, f.data, 3) / 3.0
    iters = max(3, int(budget_s * 1000.0 / max(ms, 1e-3)))
    total = r.pcg_time_iters(csr, fr.b, 128, 32, f.data, iters)
    return total / iters, iters


def run_reference(args, cfg):
    world, rank, local = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return
    fr, f = make_inputs(cfg, 0)
    its = ref_iterations(cfg["ref_key"])
    vals = []
    for step in range(args.warmup + args.steps):
        ms_it, n_it = cpu_sample(cfg, fr, f, args.ref_budget)
        if step >= args.warmup:
            vals.append(ms_it)
    ms_it = statistics.median(vals)
    value = ms_it * its if its else None
    sample = (f"reference pcg_solve (oracle/_ref, unmodified sources) with factor_applier, "
              f"{n_it} iterations per step timed by the reference's own steady_clock; "
              f"ms/solve = ms/iteration x {its} reference iterations (tests/golden/ref_iterations.json)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_it * n_it,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32/f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "n": fr.n, "nnz": int(fr.A.nnz())},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                             "sample": sample, "ms_per_iteration": ms_it, "nproc": os.cpu_count()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- our arm


def run_ours(args, cfg):
    world, rank, local = dist_init()
    import torch
    torch.cuda.set_device(local)
    import paper_2605_13343_b200 as H
    from paper_2605_13343_b200 import _native as N

    fr, f = make_inputs(cfg, rank)
    n = fr.n
    dev = H.Device(local)
    dev.load_csr(fr.A)
    dev.load_factors(f)
    dev.set_precond(2)
    assert dev.fast_path(), "fast sm_100a path not selected"
    sc = H.SolveConfig()
    b_d = torch.from_numpy(fr.b).to(f"cuda:{local}")
    x_d = torch.empty_like(b_d)
    stream = torch.cuda.ExternalStream(dev.stream(), device=f"cuda:{local}")

    def solve():
        return dev.solve_ptr(b_d.data_ptr(), x_d.data_ptr(), sc, None, N.DEVICE)

    for _ in range(args.warmup):
        rep = solve()
    iters = []
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            rep = solve()
            iters.append(int(rep.iterations))
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    t_ms = e0.elapsed_time(e1)
    t_max = max_over_ranks(t_ms, world, local)
    value = t_max / (args.steps * world)
    status = rep.status

    # end to end through the public C ABI with pinned host buffers (H2D b, D2H x + report)
    hb, hx = N.vp(), N.vp()
    N.check(N.lib.hfpg_host_alloc(8 * n, hb))
    N.check(N.lib.hfpg_host_alloc(8 * n, hx))
    import ctypes
    b_h = np.ctypeslib.as_array(ctypes.cast(hb, ctypes.POINTER(ctypes.c_double)), shape=(n,))
    b_h[:] = fr.b
    e2e_steps = max(1, min(args.steps, 5))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        dev.solve_ptr(hb.value, hx.value, sc, None, N.HOST)
    e2e_ms = (time.perf_counter() - t0) * 1000.0
    e2e_max = max_over_ranks(e2e_ms, world, local)
    N.lib.hfpg_host_free(hb)
    N.lib.hfpg_host_free(hx)

    per_iter, per_apply = dev.launch_counts()
    # per-kernel device times (standalone launches of the iteration's kernels, CUDA events on
    # the library stream) -> roofline of the dominant kernel
    ms4 = np.zeros(4, np.float32)
    N.check(N.lib.hfpg_profile_iteration(dev.h, 20, ms4.ctypes.data))
    ms_spmv, ms_leaf, ms_coarse, ms_prol = (float(v) for v in ms4)
    K = n // 128
    nnz = int(fr.A.nnz())
    # algorithmic bytes per launch
    leaf_bytes = 4 * (K * 128 * 128 + 2 * n * 32) + 48 * n
    prol_bytes = 4 * (2 * n * 32 + n) + 40 * n  # bridges + gate; y_loc, r, a_diag in, z out
    spmv_bytes = 12 * nnz + 8 * (n // 32 + 1) + 40 * n  # SELL vals+cols, z/p_prev in, p/ap out
    coarse_bytes = 4 * (K - 1) * 32 * 32 + 4 * K * 64
    b_apply = 4 * f.layout.total + 24 * n
    peak, peak_src = peaks()
    achieved = leaf_bytes / (ms_leaf * 1e-3) / 1e9
    traffic = None
    try:
        traffic = json.load(open(TRAFFIC)).get(args.config, {}).get("k_leaf_fast")
    except Exception:
        pass
    iter_ms = ms_spmv + ms_leaf + ms_coarse + ms_prol
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "n": n, "nnz": nnz, "leaf": 128, "coarse": 32,
                   "iterations": iters[-1], "status": status, "rtol": 1e-8,
                   "ref_iterations": ref_iterations(cfg["ref_key"]),
                   "l2": "inputs larger than L2 (4P = %.0f MB of factors streamed per iteration)"
                         % (4 * f.layout.total / 1e6) if n >= 262144 else
                         "factor tensor fits in L2 (%.0f MB); solve-time number is L2-resident"
                         % (4 * f.layout.total / 1e6),
                   "parallelism": f"replicas x{world} (one independent system per GPU)"},
        "roofline": {"bound": "hbm", "kernel": "k_leaf_fast", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": leaf_bytes,
                     "kernel_ms": {"k_spmv": ms_spmv, "k_leaf_fast": ms_leaf,
                                   "k_coarse": ms_coarse, "k_prolong_fast": ms_prol},
                     "apply_GBps": b_apply / ((ms_leaf + ms_coarse + ms_prol) * 1e-3) / 1e9,
                     "spmv_GBps": spmv_bytes / (ms_spmv * 1e-3) / 1e9,
                     "prolong_GBps": prol_bytes / (ms_prol * 1e-3) / 1e9,
                     "iteration_ms": iter_ms,
                     "solve_ms_per_iteration": (t_max / args.steps) / max(iters[-1], 1)},
        "e2e": {"value": e2e_max / (e2e_steps * world), "unit": UNIT,
                "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n + 96},
        "gpu_launches": args.steps * (1 + per_apply + per_iter * iters[-1]),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ms_it, n_it = cpu_sample(cfg, fr, f, args.ref_budget)
        its = ref_iterations(cfg["ref_key"]) or iters[-1]
        line["cpu_baseline"] = {
            "value": ms_it * its, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{n_it} iterations of the reference pcg_solve loop (oracle/_ref, "
                      f"factor_applier) on 1 host core, scaled by {its} iterations",
            "ms_per_iteration": ms_it, "nproc": os.cpu_count()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="3d_1m", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-budget", type=float, default=10.0, help="CPU seconds per sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        args.ref_budget = min(args.ref_budget, 4.0)
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
