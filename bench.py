#!/usr/bin/env python
"""Benchmark: one step = one PCG solve to rel. residual 1e-8 of a synthetic pressure-Poisson
system with the hierarchical-factor preconditioner, on B200 through libhfpg's C ABI.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 3d_1m|2d_65536|2d_262144|2d_8192|batch_262k|part_16m]

Default workload (N=1): BASELINE.json configs[2] — N = 1,048,576 (128x128x64 3D 7-point
Neumann Laplacian, the bandwidth-bound apply + SpMV regime the metric's "precond-apply HBM GB/s
vs peak" half is quoted on), seeded jacobi_seed sigma=1e-2 factor tensor (L=128, L_s=32).
Under torchrun (N>1) every rank solves its own frame (frame index = rank): independent systems,
no collective on the data path ("scaling": "weak"); the barrier + max-over-ranks timing is the
only communication. The other BASELINE configs are named workloads:
  batch_262k  configs[3]: 64 independent N=262,144 frames sharded over the ranks (64/N each);
              value = batch time / 64 ("scaling": "strong", total work fixed)
  part_16m    configs[4]: one N=16,777,216 system (3D 256^3) row-partitioned over the ranks,
              peers over CUDA IPC / NVLink (the whole system on one GPU at N=1)
`--impl reference` times the reference's own CPU code (oracle/_ref, the
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
    "2d_262144": dict(desc="one frame of BASELINE configs[3]: N=262,144 2D make_frame(262144, 2024, "
                           "test_frame_id(262144, 0)), seeded sigma=1e-2 tensor, L=128, L_s=32",
                      n=262144, sigma=1e-2, ref_key="2d_262144_t0_s1e-2", test_frame=True),
    "2d_8192": dict(desc="BASELINE configs[0] system: make_frame(8192, 2024, 0), seeded tensor",
                    n=8192, sigma=1e-2, ref_key="2d_8192"),
    "batch_262k": dict(kind="batch", frames=64,
                       desc="BASELINE configs[3]: 64 independent frames make_frame(262144, 2024, "
                            "test_frame_id(262144, i)), i = 0..63, each with its seeded sigma=1e-3 "
                            "tensor (RngStream(2024, frame_id, factor_init); sigma=1e-2 leaves "
                            "frames at max_iters, DESIGN.md), sharded over the GPUs",
                       n=262144, sigma=1e-3, ref_key="2d_262144_t0_s1e-3"),
    "2d_65536_infer": dict(kind="infer", n=65536,
                           desc="BASELINE configs[1]: N=65,536 (make_frame(65536, 2024, 0) generated on the GPU), "
                                "full toynet d128_L3_hw inference into the packed factor tensor + graph PCG; "
                                "step = generate + forward + solve (device times)"),
    "part_16m": dict(kind="part",
                     desc="BASELINE configs[4]: N=16,777,216 3D 256^3 7-point pressure-Poisson, "
                          "seeded sigma=1e-3 tensor, row-partitioned over the GPUs along the "
                          "bisection tree (mailbox exchange over CUDA IPC / NVLink)",
                     dims=(256, 256, 256), sigma=1e-3, ref_key=None),
}


def make_inputs(cfg: dict, frame_index: int):
    import paper_2605_13343_b200 as H
    if "dims" in cfg:
        fr = H.make_frame_3d(*cfg["dims"], 2024, frame_index)
    else:
        fid = H.test_frame_id(cfg["n"], frame_index) if cfg.get("test_frame") or cfg.get("kind") == "batch" else frame_index
        fr = H.make_frame(cfg["n"], 2024, fid)
    f = H.init_factors(H.build_partition(fr.n, 128), 32, H.FactorInit.jacobi_seed, cfg["sigma"],
                       H.RngStream(2024, fr.frame_index, H.RngPurpose.factor_init))
    return fr, f


def make_ref_inputs(cfg: dict, frame_index: int):
    """The reference arm's inputs, built without the product library: the reference's own
    make_frame (frame.cpp:161-181) / the oracle-side 3D frame (oracle/frame3d_ref.cpp, reference
    RngStream + sample_rhs) and the reference's init_factors (factor_tensor.cpp:30-39), all from
    oracle/_ref. Returns (csr tuple, b, packed factors, n)."""
    from oracle.oracle import Ref
    r = Ref()
    if "dims" in cfg:
        fr = r.make_frame_3d(*cfg["dims"], 2024, frame_index)
        fid = frame_index
    else:
        n = cfg["n"]
        fid = ((n << 24) | (1 << 20) | frame_index) if cfg.get("test_frame") or cfg.get("kind") == "batch" \
            else frame_index  # frame.hpp:88-90 test_frame_id
        fr = r.make_frame(n, 2024, fid)
    packed = r.init_factors(fr["n"], 128, 32, cfg["sigma"], 2024, fid)
    return (fr["row_offsets"], fr["col_indices"], fr["values"]), fr["b"], packed, fr["n"]


def config_of(cfg: dict, n: int, nnz: int) -> dict:
    """The `config` object both arms print (same keys, same values)."""
    return {"workload": cfg["desc"], "n": int(n), "nnz": int(nnz)}


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
    dev = "cpu" if dist.get_backend() == "gloo" else f"cuda:{local}"  # gloo: the CPU multi-process tests
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def frames_of(rank: int, world: int, frames: int) -> list:
    """configs[3]'s sharding: frame i on rank i mod N (no collective on the solve path)."""
    return list(range(rank, frames, world))


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------------- reference arm


def cpu_sample_raw(csr, b, packed, budget_s: float):
    """Time the reference's own pcg_solve loop (oracle/_ref) for a bounded number of
    iterations; returns (ms per iteration, iterations run)."""
    from oracle.oracle import Ref
    r = Ref()
    ms = r.pcg_time_iters(csr, b, 128, 32, packed, 3) / 3.0
    iters = max(3, int(budget_s * 1000.0 / max(ms, 1e-3)))
    total = r.pcg_time_iters(csr, b, 128, 32, packed, iters)
    return total / iters, iters


def cpu_sample(cfg, fr, f, budget_s: float):
    return cpu_sample_raw((fr.A.row_offsets, fr.A.col_indices, fr.A.values), fr.b, f.data, budget_s)


def run_reference(args, cfg):
    world, rank, local = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return
    if cfg.get("kind") in ("part", "infer"):
        print(json.dumps({"impl": "reference", "unavailable": f"--config {args.config}: the reference "
                          "has no row-partitioned solve / its forward is timed in the parity tests"}), flush=True)
        return
    csr, b, packed, n = make_ref_inputs(cfg, 0)
    its = ref_iterations(cfg["ref_key"])
    vals = []
    for step in range(args.warmup + args.steps):
        ms_it, n_it = cpu_sample_raw(csr, b, packed, args.ref_budget)
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
            "config": config_of(cfg, n, len(csr[2])),
            "config_details": {"inputs": "built by oracle/_ref (reference make_frame / oracle-side 3D "
                                         "frame, reference init_factors); the product library is not loaded"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                             "sample": sample, "ms_per_iteration": ms_it, "nproc": os.cpu_count()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------ configs[1]: inference + graph PCG


def toynet_flops(n: int, L: int = 128, Ls: int = 32, d: int = 128, layers: int = 3, feat: int = 19) -> int:
    """Dense-contraction FLOPs of one toynet forward as the reference computes it
    (toy_net.cpp:225-586): encoder MLP + GCN, per layer QKV / QK^T / PV / O-projection / 4d FFN
    (K = 4d, the glob slice included) for both streams, decoder heads. 2 FLOPs per MAC."""
    K = n // L
    mt = (K - 1) * Ls  # tile tokens

    def stream(rows, T):
        return rows * (d * 3 * d + 2 * T * d + d * d + 4 * d * 4 * d + 4 * d * d)

    macs = n * (feat * d + d * d) + 2 * n * d * d  # encoder + 2 GCN layers
    macs += layers * (stream(n, L) + stream(mt, Ls))
    macs += n * (d * d + d * L + d * (2 * Ls + 1)) + mt * d * Ls  # decoder heads
    return 2 * macs


def run_inference(local: int, steps: int, warmup: int, n: int = 65536, solve: bool = True) -> dict:
    """BASELINE configs[1]: the N=65,536 frame generated on the GPU (make_frame(n, 2024, 0)),
    the d128_L3_hw toy network (seeded weights, toy_net.cpp:170-223) writing the packed factor
    tensor straight into the handle, then the graph PCG on that tensor. Device times (CUDA
    events on the handle's stream)."""
    import paper_2605_13343_b200 as H
    from paper_2605_13343_b200 import _native as N
    import torch
    dev = H.Device(local)
    gen_ms, inf_ms = [], []
    for i in range(warmup + steps):
        gf = dev.frame_gpu(n, 2024, 0)
        tr = H.ToynetTrace(timing_only=True)
        H.toynet_forward_gpu_frame(gf, 32, trace=tr, load=True)
        if i >= warmup:
            gen_ms.append(gf.generate_ms)
            inf_ms.append(tr.ms)
    fl = toynet_flops(n)
    peak_bf16 = None
    try:
        peak_bf16 = float(json.load(open(PEAKS))["bf16_tflops_sustained"])
        peak_src = "0.5 x MEASURED_PEAKS.json bf16_tflops_sustained (kind::tf32 runs at half the bf16 rate)"
    except Exception:
        peak_bf16 = 2250.0 * 0.85
        peak_src = "0.5 x fallback bf16 dense (B200_PROFILING.md)"
    peak = 0.5 * peak_bf16
    ms = statistics.median(inf_ms)
    out = {"workload": "BASELINE configs[1]: make_frame(65536, 2024, 0) generated on the GPU, toynet "
                       "d128_L3_hw (d=128, 3 layers, 8 heads, L=128, L_s=32, weight seed 0) -> packed "
                       "factor tensor on the device -> graph PCG",
           "n": n, "generate_ms": statistics.median(gen_ms), "inference_ms": ms,
           "inference_ms_all": inf_ms, "inference_flops": fl,
           "roofline": {"bound": "tensor", "achieved": fl / (ms * 1e-3) / 1e12, "peak": peak,
                        "unit": "TFLOP/s", "frac": fl / (ms * 1e-3) / 1e12 / peak,
                        "peak_source": peak_src, "precision": "kind::tf32 products, fp32 accumulation"}}
    if solve:
        dev.set_precond(2)
        x = torch.empty(n, dtype=torch.float64, device=f"cuda:{local}")
        rep = dev.solve_ptr(gf.b, x.data_ptr(), H.SolveConfig(), None, N.DEVICE)
        out.update({"solve_ms": float(rep.wall_ms), "solve_iterations": int(rep.iterations),
                    "solve_status": H.SolveStatus(int(rep.status)).name,
                    "solve_note": "the seeded-weight tensor is not a convergent preconditioner "
                                  "(SURVEY.md section 0 fact 2: the reference stagnates / NaNs), so the "
                                  "solve runs to max_iters exactly as the reference's does"})
    return out


TRAINED = os.path.join(ROOT, "tests", "golden", "trained_8192.hftc")


def run_trained(local: int, reps: int = 5) -> dict:
    """BASELINE configs[0]'s system (make_frame(8192, 2024, 0)) with a TRAINED factor tensor —
    tests/golden/trained_8192.hftc, produced by the GPU train_factors on the reference's
    acceptance recipe (acceptance.cpp:378-420; tools/train_tensor.py --acceptance --n 8192) — next
    to Jacobi on the same graph: graph-PCG device times, the exact solver's count against the
    reference's own pcg_solve with the same checkpoint (tests/golden/ref_iterations.json)."""
    import paper_2605_13343_b200 as H
    from paper_2605_13343_b200 import _native as N
    import torch
    fr = H.make_frame(8192, 2024, 0)
    dev = H.Device(local)
    dev.load_csr(fr.A)
    dev.load_checkpoint(TRAINED)
    b = torch.from_numpy(fr.b).to(f"cuda:{local}")
    x = torch.empty_like(b)
    sc = H.SolveConfig()
    out = {"workload": "make_frame(8192, 2024, 0) (BASELINE configs[0]) with the trained tensor "
                       "tests/golden/trained_8192.hftc vs Jacobi, graph PCG to 1e-8"}
    for name, kind in (("trained", 2), ("jacobi", 1)):
        dev.set_precond(kind)
        ms, its = [], 0
        for _ in range(reps + 1):
            rep = dev.solve_ptr(b.data_ptr(), x.data_ptr(), sc, None, N.DEVICE)
            ms.append(float(rep.wall_ms))
            its = int(rep.iterations)
        out[name] = {"iterations": its, "ms": statistics.median(ms[1:])}
    dev.set_precond(2)
    rx = dev.solve_ptr(b.data_ptr(), x.data_ptr(), sc, None, N.DEVICE, exact=True)
    want = None
    try:
        want = json.load(open(ITERS))["2d_8192_trained"]
    except Exception:
        pass
    out["trained"]["exact_iterations"] = int(rx.iterations)
    out["reference_iterations"] = {"trained": want["factor"]["iterations"], "jacobi": want["jacobi"]["iterations"]} if want else None
    return out


def run_infer_config(args, cfg):
    world, rank, local = dist_init()
    import torch
    torch.cuda.set_device(local)
    with Clocks(local) as clk:
        res = run_inference(local, args.steps, args.warmup, cfg["n"], solve=True)
    step_ms = res["generate_ms"] + res["inference_ms"] + res["solve_ms"]
    line = {"metric": METRIC, "value": step_ms, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (tf32 MMA) / f64", "data": "synthetic",
            "config": config_of(cfg, cfg["n"], 0),
            "roofline": res.pop("roofline"), "inference": res, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- our arm


def launches_per_solve(dev, iterations: int) -> int:
    """Kernels one solve launches: one k_solve (persistent driver) or the graph's init + loop."""
    per_iter, per_apply = dev.launch_counts()
    if per_iter == 0:
        return 1
    return 1 + per_apply + per_iter * iterations


def run_ours(args, cfg):
    if cfg.get("kind") == "batch":
        return run_batch(args, cfg)
    if cfg.get("kind") == "part":
        return run_part(args, cfg)
    if cfg.get("kind") == "infer":
        return run_infer_config(args, cfg)
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
    # every rank solves its own independent system (weak scaling): the metric is the per-solve
    # latency, max over ranks; the aggregate rate across GPUs is reported beside it
    value = t_max / args.steps
    status = rep.status

    # end to end through the public C ABI with pinned host buffers (H2D b, D2H x + report)
    hb, hx = N.vp(), N.vp()
    N.check(N.lib.hfpg_host_alloc(8 * n, hb))
    N.check(N.lib.hfpg_host_alloc(8 * n, hx))
    import ctypes
    b_h = np.ctypeslib.as_array(ctypes.cast(hb, ctypes.POINTER(ctypes.c_double)), shape=(n,))
    b_h[:] = fr.b
    # interleaved pairs (device-resident solve timed by CUDA events, then the host-buffer solve
    # timed by the wall clock around the blocking C-ABI call), medians of each: box noise hits
    # both arms alike, so e2e - device is the copy cost, not run-to-run drift
    e2e_steps = max(5, min(args.steps, 9))
    dev_ms_pairs, e2e_ms_pairs = [], []
    barrier(world)
    for _ in range(e2e_steps):
        e0.record(stream)
        solve()
        e1.record(stream)
        torch.cuda.synchronize()
        dev_ms_pairs.append(e0.elapsed_time(e1))
        t0 = time.perf_counter()
        dev.solve_ptr(hb.value, hx.value, sc, None, N.HOST)
        e2e_ms_pairs.append((time.perf_counter() - t0) * 1000.0)
    e2e_med = max_over_ranks(statistics.median(e2e_ms_pairs), world, local)
    dev_med = max_over_ranks(statistics.median(dev_ms_pairs), world, local)
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
    apply_ms = ms_leaf + ms_coarse + ms_prol
    apply_gbps = b_apply / (apply_ms * 1e-3) / 1e9
    traffic = apply_traffic = spmv_traffic = None
    try:
        tj = json.load(open(TRAFFIC)).get(args.config, {})
        traffic = tj.get("k_leaf_fast")
        parts = [tj.get(k) for k in ("k_leaf_fast", "k_coarse_coop", "k_prolong_tma")]
        apply_traffic = sum(parts) if all(p is not None for p in parts) else None
        spmv_traffic = tj.get("k_spmv_tma")
    except Exception:
        pass
    iter_ms = ms_spmv + ms_leaf + ms_coarse + ms_prol
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": config_of(cfg, n, nnz),
        "config_details": {"leaf": 128, "coarse": 32,
                   "iterations": iters[-1], "status": status, "rtol": 1e-8,
                   "ref_iterations": ref_iterations(cfg["ref_key"]),
                   "l2": "inputs larger than L2 (4P = %.0f MB of factors streamed per iteration)"
                         % (4 * f.layout.total / 1e6) if n >= 262144 else
                         "factor tensor fits in L2 (%.0f MB); solve-time number is L2-resident"
                         % (4 * f.layout.total / 1e6),
                   "parallelism": f"replicas x{world} (one independent system per GPU)"},
        # headline: the whole preconditioner apply (the metric's "precond-apply HBM GB/s vs
        # peak"): B_apply = 4P + 24N algorithmic bytes over the summed device time
        # of its launches (leaf + coarse + prolongation); the dominant kernel below
        "roofline": {"bound": "hbm", "kernel": "apply (k_leaf_fast + k_coarse_coop + k_prolong_tma)",
                     "achieved": apply_gbps, "peak": peak, "unit": "GB/s", "frac": apply_gbps / peak,
                     "traffic": apply_traffic, "peak_source": peak_src, "algorithmic_bytes_per_launch": b_apply,
                     "traffic_note": "ncu DRAM read+write bytes of the apply's three launches (cold-cache standalone "
                                     "launches: the bridges are read twice, once per side of the coarse stage)",
                     "dominant_kernel": {"kernel": "k_leaf_fast", "achieved": achieved, "frac": achieved / peak,
                                         "algorithmic_bytes_per_launch": leaf_bytes, "traffic": traffic},
                     "kernel_ms": {"k_spmv": ms_spmv, "k_leaf_fast": ms_leaf,
                                   "k_coarse": ms_coarse, "k_prolong": ms_prol},
                     "apply_GBps": apply_gbps,
                     "spmv_GBps": spmv_bytes / (ms_spmv * 1e-3) / 1e9,
                     # sustained DRAM rate: the ncu bytes the launches actually move (the apply reads
                     # the bridges twice, which B_apply does not count) over the same device times
                     "apply_dram_GBps": apply_traffic / (apply_ms * 1e-3) / 1e9 if apply_traffic else None,
                     "spmv_dram_GBps": spmv_traffic / (ms_spmv * 1e-3) / 1e9 if spmv_traffic else None,
                     "prolong_GBps": prol_bytes / (ms_prol * 1e-3) / 1e9,
                     "iteration_ms": iter_ms,
                     "solve_ms_per_iteration": (t_max / args.steps) / max(iters[-1], 1)},
        "aggregate_solves_per_s": world * args.steps / (t_max * 1e-3),
        "e2e": {"value": e2e_med, "unit": UNIT,
                "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n + 96,
                "device_ms_median_interleaved": dev_med, "pairs": e2e_steps,
                "how": "median of interleaved pairs: device-resident solve (CUDA events) / host-buffer solve "
                       "through hfpg_pcg_solve (wall clock around the blocking call)"},
        "gpu_launches": args.steps * launches_per_solve(dev, iters[-1]),
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_parity:
        # outside the timed region: the bit-exact loop (hfpg_pcg_solve_exact) on the same system,
        # against the reference's own run at this size (tests/golden/ref_iterations.json)
        want = None
        try:
            want = json.load(open(ITERS))[cfg["ref_key"]]["factor"]
        except Exception:
            pass
        hist_d = torch.empty(sc.max_iters, dtype=torch.float64, device=f"cuda:{local}")
        xr = torch.empty_like(b_d)
        rx = dev.solve_ptr(b_d.data_ptr(), xr.data_ptr(), sc, hist_d.data_ptr(), N.DEVICE, exact=True)
        last = float(hist_d[int(rx.history_len) - 1].item()) if rx.history_len else None
        line["parity"] = {
            "graph_iterations": iters[-1], "exact_iterations": int(rx.iterations),
            "reference_iterations": want["iterations"] if want else None,
            "exact_final_rel": last, "reference_final_rel": want["final_rel"] if want else None,
            "exact_bit_identical_to_reference": bool(want) and int(rx.iterations) == want["iterations"]
                                               and last == want["final_rel"],
            "exact_ms": float(rx.wall_ms),
            "how": "hfpg_pcg_solve_exact (sequential dots emulated exactly, apply<float> bit for bit) "
                   "vs the reference's own pcg_solve run at this size"}
    if rank == 0 and not args.no_inference:
        # BASELINE configs[1] (N=65,536 inference + graph PCG), outside the timed region
        line["inference"] = run_inference(local, 3, 1, 65536, solve=True)
        # a trained tensor (GPU train_factors) on configs[0]'s system, against Jacobi
        if os.path.exists(TRAINED):
            line["trained"] = run_trained(local)
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


# ------------------------------------------------------------- configs[3]: batched frames


def run_batch(args, cfg):
    """64 independent frames, frame i on rank i mod N; one step = every rank solves its share
    (each solve one graph / one persistent launch on the whole GPU); value = max-over-ranks step
    time / 64 frames."""
    world, rank, local = dist_init()
    import torch
    torch.cuda.set_device(local)
    import paper_2605_13343_b200 as H
    from paper_2605_13343_b200 import _native as N
    mine = frames_of(rank, world, cfg["frames"])
    devs, bs, xs, its = [], [], [], []
    fr0 = f0 = None
    for i in mine:
        fr, f = make_inputs(cfg, i)
        d = H.Device(local)
        d.load_csr(fr.A)
        d.load_factors(f)
        d.set_precond(2)
        devs.append(d)
        bs.append(torch.from_numpy(fr.b).to(f"cuda:{local}"))
        xs.append(torch.empty_like(bs[-1]))
        if i == 0:
            fr0, f0 = fr, f
    sc = H.SolveConfig()

    # every frame of this rank in flight at once (one handle + stream each): independent
    # latency-bound solves fill each other's gaps; the step starts on s0 and ends when all
    # streams have joined it again
    streams = [torch.cuda.ExternalStream(d.stream(), device=f"cuda:{local}") for d in devs]
    s0 = streams[0]
    ev_start = torch.cuda.Event()
    ev_done = [torch.cuda.Event() for _ in devs]

    def step():
        ev_start.record(s0)
        for d, st, b, x in zip(devs, streams, bs, xs):
            st.wait_event(ev_start)
            d.solve_async(b.data_ptr(), x.data_ptr(), sc, N.DEVICE)
        out = []
        for d, st, ev in zip(devs, streams, ev_done):
            ev.record(st)
            s0.wait_event(ev)
        for d in devs:
            out.append(int(d.wait().iterations))
        return out

    for _ in range(args.warmup):
        its = step()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(s0)
        for _ in range(args.steps):
            its = step()
        e1.record(s0)
        torch.cuda.synchronize()
    barrier(world)
    t_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, local)
    value = t_ms / cfg["frames"]
    # end to end through the C ABI: each frame's b from pinned host memory in, x out
    import ctypes
    n = bs[0].numel()
    hb, hx = N.vp(), N.vp()
    N.check(N.lib.hfpg_host_alloc(8 * n, hb))
    N.check(N.lib.hfpg_host_alloc(8 * n, hx))
    b_np = np.ctypeslib.as_array(ctypes.cast(hb, ctypes.POINTER(ctypes.c_double)), shape=(n,))
    host_b = [b.cpu().numpy() for b in bs]
    barrier(world)
    t0 = time.perf_counter()
    for d, bh in zip(devs, host_b):
        b_np[:] = bh
        d.solve_ptr(hb.value, hx.value, sc, None, N.HOST)
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1000.0, world, local)
    N.lib.hfpg_host_free(hb)
    N.lib.hfpg_host_free(hx)
    all_its = its
    if world > 1:
        import torch.distributed as dist
        gathered = [None] * world
        dist.all_gather_object(gathered, its)
        all_its = [v for g in gathered for v in g]
    peak, peak_src = peaks()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": config_of(cfg, n, int(fr0.A.nnz()) if fr0 is not None else 0),
        "config_details": {"frames": cfg["frames"], "frames_per_gpu": len(mine),
                   "iterations_mean": float(np.mean(all_its)), "iterations_min": int(min(all_its)),
                   "iterations_max": int(max(all_its)), "ref_iterations_frame0": ref_iterations(cfg["ref_key"]),
                   "solver": "persistent" if devs[0].solver_in_use() == N.SOLVER_PERSISTENT else "graph",
                   "l2": "per-frame factor tensor 211 MB > L2 (streamed every iteration)",
                   "parallelism": f"frames sharded {cfg['frames']}/{world} per GPU, all of a GPU's frames in flight "
                                  f"concurrently (one handle + stream each), no collective"},
        "e2e": {"value": e2e_ms / cfg["frames"], "unit": UNIT,
                "h2d_bytes_per_step": 8 * n * cfg["frames"], "d2h_bytes_per_step": 8 * n * cfg["frames"]},
        "gpu_launches": args.steps * sum(launches_per_solve(devs[0], k) for k in its),
        "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "peak": peak, "peak_source": peak_src, "unit": "GB/s"},
    }
    if rank == 0:
        # dominant kernel of the per-stage path on frame 0 (standalone launches, CUDA events)
        ms4 = np.zeros(4, np.float32)
        devs[0].solve_ptr(bs[0].data_ptr(), xs[0].data_ptr(), sc, None, N.DEVICE)
        N.check(N.lib.hfpg_profile_iteration(devs[0].h, 20, ms4.ctypes.data))
        K = n // 128
        leaf_bytes = 4 * (K * 128 * 128 + 2 * n * 32) + 48 * n
        achieved = leaf_bytes / (float(ms4[1]) * 1e-3) / 1e9
        line["roofline"].update({"kernel": "k_leaf_fast", "achieved": achieved, "frac": achieved / peak,
                                 "traffic": None, "algorithmic_bytes_per_launch": leaf_bytes,
                                 "kernel_ms": dict(zip(["k_spmv", "k_leaf_fast", "k_coarse", "k_prolong"],
                                                       map(float, ms4)))})
        if world == 1 and not args.no_cpu_baseline:
            ms_it, n_it = cpu_sample(cfg, fr0, f0, args.ref_budget)
            rits = ref_iterations(cfg["ref_key"]) or all_its[0]
            line["cpu_baseline"] = {
                "value": ms_it * rits, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"{n_it} iterations of the reference pcg_solve on frame 0 (oracle/_ref, 1 host core), "
                          f"x {rits} iterations = ms per frame solve",
                "ms_per_iteration": ms_it, "nproc": os.cpu_count()}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ------------------------------------------------------ configs[4]: row-partitioned system


def run_part(args, cfg):
    """One N=16.7M system; rank r of N holds rows [r N/G, (r+1) N/G) and the matching subtree of
    the factor tensor (drawn per slice); peers are mapped through CUDA IPC handles all-gathered
    over torch.distributed. One step = one partitioned solve; value = max-over-ranks ms."""
    world, rank, local = dist_init()
    import torch
    torch.cuda.set_device(local)
    import paper_2605_13343_b200 as H
    from paper_2605_13343_b200 import _native as N
    t_setup = time.perf_counter()
    fr = H.make_frame_3d(*cfg["dims"], 2024, 0)
    n = fr.n
    sc = H.SolveConfig()
    if world == 1:
        f = H.init_factors(H.build_partition(n, 128), 32, H.FactorInit.jacobi_seed, cfg["sigma"],
                           H.RngStream(2024, 0, H.RngPurpose.factor_init))
        dev = H.Device(local)
        dev.load_csr(fr.A)
        dev.load_factors(f)
        dev.set_precond(2)
        del f
        nl, r0 = n, 0
    else:
        import torch.distributed as dist

        def allgather(blob):
            out = [None] * world
            dist.all_gather_object(out, blob)
            return out

        rs = H.RankSolver(fr.A, world, rank, allgather, sigma=cfg["sigma"], seed=2024, frame=0,
                          device=local)
        dev, nl, r0 = rs.dev, rs.n_local, rs.row_begin
    b = torch.from_numpy(fr.b[r0:r0 + nl].copy()).to(f"cuda:{local}")
    x = torch.empty_like(b)
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.ExternalStream(dev.stream(), device=f"cuda:{local}")

    def solve():
        return dev.solve_ptr(b.data_ptr(), x.data_ptr(), sc, None, N.DEVICE)

    for _ in range(args.warmup):
        rep = solve()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            rep = solve()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    t_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, local)
    # end to end: host slices of b in, x out
    hb = fr.b[r0:r0 + nl].copy()
    hx = np.empty(nl)
    barrier(world)
    t0 = time.perf_counter()
    dev.solve_ptr(hb.ctypes.data, hx.ctypes.data, sc, None, N.HOST)
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1000.0, world, local)
    its = int(rep.iterations)
    K = nl // 128
    nnz = int(fr.A.nnz())
    b_iter = (4 * (K * 128 * 128 + (K - 1) * 1024 + 2 * nl * 32 + nl) + 24 * nl) + (12 * nnz // world + 24 * nl) + 64 * nl
    peak, peak_src = peaks()
    achieved = b_iter * its / (t_ms * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": t_ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
            "config": config_of(cfg, n, nnz),
            "config_details": {"rows_per_gpu": nl, "iterations": its,
                       "status": int(rep.status), "rtol": 1e-8, "setup_s": setup_s,
                       "parallelism": f"row partition over {world} GPU(s)" + (
                           ", mailboxes + z halo over CUDA IPC (NVLink P2P)" if world > 1 else ""),
                       "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "kernel": "whole solve (per GPU, algorithmic B_iter x iterations)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "peak_source": peak_src, "algorithmic_bytes_per_iteration": b_iter},
            "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": 8 * nl, "d2h_bytes_per_step": 8 * nl},
            "gpu_launches": args.steps * launches_per_solve(dev, its),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run with N ranks
    (one per GPU, rendezvous on 127.0.0.1), the driver's own launch line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def check_launch(args):
    """--check-launch: the N-rank plumbing only (rendezvous, barrier, max over ranks, the
    configs[3] frame sharding) — one JSON line from rank 0; runs on CPU with HFPG_BENCH_GLOO=1."""
    world, rank, local = dist_init()
    barrier(world)
    t = max_over_ranks(float(rank + 1), world, local)
    frames = frames_of(rank, world, 64)
    if world > 1:
        import torch.distributed as dist
        got = [None] * world
        dist.all_gather_object(got, frames)
        frames = sorted(f for g in got for f in g)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"check_launch": True, "n_gpus": world, "gpus_requested": args.gpus,
                          "max_over_ranks": t, "frames_covered": frames == list(range(64))}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="3d_1m", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-budget", type=float, default=10.0, help="CPU seconds per sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the bit-exact parity solve")
    ap.add_argument("--no-inference", action="store_true", help="skip the configs[1] inference object")
    ap.add_argument("--check-launch", action="store_true", help="N-rank plumbing only (no solve)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    if args.check_launch:
        return check_launch(args)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        args.ref_budget = min(args.ref_budget, 4.0)
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
