"""ctypes binding of include/hfpg.h (the C ABI of libhfpg.so).

The library is loaded from this package directory only (built in-tree by build.py). There is
no CPU fallback: if the shared object is missing this module raises at import.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libhfpg.so")
# development A/B only: HFPG_SO_VARIANT=<name> loads the in-tree variants/libhfpg_<name>.so built
# by tools/build_variant.sh (same sources, different compile-time constants)
if os.environ.get("HFPG_SO_VARIANT"):
    SO_PATH = os.path.join(HERE, "variants", "libhfpg_%s.so" % os.environ["HFPG_SO_VARIANT"])

HFPG_OK, HFPG_EINVAL, HFPG_EIO, HFPG_ECUDA, HFPG_ENCCL = range(5)
HOST, DEVICE = 0, 1
SOLVER_AUTO, SOLVER_GRAPH, SOLVER_PERSISTENT = 0, 1, 2

u64, i32, dbl, vp = C.c_uint64, C.c_int32, C.c_double, C.c_void_p


class Tile(C.Structure):
    _fields_ = [("id", u64), ("span", u64), ("row_begin", u64), ("col_begin", u64),
                ("depth", u64)]


class Layout(C.Structure):
    _fields_ = [(k, u64) for k in ("n", "leaf_size", "coarse_size", "coupling_rank",
                                   "leaf_count", "tile_count", "leaf_base", "tile_base",
                                   "bridge_base", "gate_base", "total")]


class SolveConfigC(C.Structure):
    _fields_ = [("rtol", dbl), ("max_iters", u64)]


class ReportC(C.Structure):
    _fields_ = [("n", u64), ("iterations", u64), ("converged", i32), ("status", i32),
                ("breakdown_iter", u64), ("history_len", u64), ("wall_ms", dbl)]


class ToynetConfigC(C.Structure):
    _fields_ = [(k, u64) for k in ("d", "layers", "heads", "gcn_layers", "d_global",
                                   "edge_hidden")]


class ToynetTraceC(C.Structure):
    _fields_ = [("max_attention_row_sum_error", dbl), ("highway_max_deviation", dbl),
                ("leaf_attention_dispatches", u64), ("tile_attention_dispatches", u64),
                ("ms", dbl), ("timing_only", i32)]


class FrameViewC(C.Structure):
    _fields_ = [("n", u64), ("width", u64), ("height", u64), ("cell_order", vp), ("rho", vp),
                ("rho_heavy", dbl), ("row_offsets", vp), ("col_indices", vp), ("values", vp)]


class TrainFrameC(C.Structure):
    _fields_ = [("view", FrameViewC), ("b", vp), ("frame_index", u64)]


class TrainConfigC(C.Structure):
    _fields_ = [("lr", dbl), ("weight_decay", dbl), ("clip_norm", dbl), ("plateau_factor", dbl),
                ("plateau_patience", u64), ("plateau_rel_threshold", dbl), ("max_steps", u64),
                ("autostop_window", u64), ("probe_omega", dbl), ("probe_smooth_steps", u64),
                ("contexts_per_step", u64), ("loss", i32), ("log_every", u64), ("init_sigma", dbl),
                ("leaf_size", u64), ("coarse_size", u64), ("eval_every_logs", u64), ("solve_rtol", dbl),
                ("solve_max_iters", u64), ("stop_at_iters", u64)]


class TrainLogC(C.Structure):
    _fields_ = [("step", u64), ("train_loss", dbl), ("sai_heldout", dbl), ("pcg_iters_heldout", u64),
                ("lr", dbl), ("wall_s", dbl)]


class TrainSummaryC(C.Structure):
    _fields_ = [("total_steps", u64), ("auto_stopped", i32), ("aborted_divergence", i32),
                ("reached_target", i32), ("n_entries", u64), ("leaf_size", u64), ("packed_width", u64)]


class FrameDeviceC(C.Structure):
    _fields_ = [("n", u64), ("nnz", u64), ("width", u64), ("height", u64), ("depth", u64),
                ("rho_heavy", dbl), ("cell_order", vp), ("rho", vp), ("row_offsets", vp),
                ("col_indices", vp), ("values", vp), ("b", vp), ("a_diag", vp),
                ("generate_ms", C.c_float), ("frobenius", dbl)]


class CudaError(RuntimeError):
    """A CUDA failure inside libhfpg (HFPG_ECUDA)."""


_PROTOS = {
    "hfpg_version": (C.c_char_p, []),
    "hfpg_last_error": (C.c_char_p, []),
    "hfpg_packed_width": (C.c_int, [u64, u64, u64, C.POINTER(u64)]),
    "hfpg_build_partition": (C.c_int, [u64, u64, vp, u64, C.POINTER(u64)]),
    "hfpg_factor_layout": (C.c_int, [u64, u64, u64, C.POINTER(Layout)]),
    "hfpg_init_factors": (C.c_int, [u64, u64, u64, dbl, u64, u64, vp]),
    "hfpg_read_checkpoint": (C.c_int, [C.c_char_p, C.POINTER(Layout), vp, C.POINTER(i32),
                                       C.POINTER(dbl), C.c_char_p, u64]),
    "hfpg_write_checkpoint": (C.c_int, [C.c_char_p, u64, u64, u64, vp, i32, dbl, C.c_char_p]),
    "hfpg_frame_2d": (C.c_int, [u64, u64, u64, C.POINTER(vp)]),
    "hfpg_frame_3d": (C.c_int, [u64, u64, u64, u64, u64, C.POINTER(vp)]),
    "hfpg_frame_info": (C.c_int, [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64),
                                  C.POINTER(u64), C.POINTER(u64), C.POINTER(dbl)]),
    "hfpg_frame_copy": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "hfpg_frame_gpu_2d": (C.c_int, [vp, u64, u64, u64]),
    "hfpg_frame_gpu_3d": (C.c_int, [vp, u64, u64, u64, u64, u64]),
    "hfpg_frame_gpu_view": (C.c_int, [vp, C.POINTER(FrameDeviceC)]),
    "hfpg_seq_sum": (C.c_int, [vp, vp, u64, i32, C.c_int, C.POINTER(dbl)]),
    "hfpg_frame_gpu_copy": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "hfpg_frame_free": (None, [vp]),
    "hfpg_host_alloc": (C.c_int, [u64, C.POINTER(vp)]),
    "hfpg_host_free": (C.c_int, [vp]),
    "hfpg_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "hfpg_destroy": (C.c_int, [vp]),
    "hfpg_get_stream": (C.c_int, [vp, C.POINTER(vp)]),
    "hfpg_load_csr": (C.c_int, [vp, u64, vp, vp, vp, C.c_int]),
    "hfpg_load_factors": (C.c_int, [vp, u64, u64, u64, vp, u64, i32, dbl, C.c_int]),
    "hfpg_set_diag": (C.c_int, [vp, u64, vp, C.c_int]),
    "hfpg_set_precond": (C.c_int, [vp, C.c_int]),
    "hfpg_apply": (C.c_int, [vp, vp, vp, C.c_int]),
    "hfpg_precond_apply": (C.c_int, [vp, vp, vp, C.c_int]),
    "hfpg_probes_device": (C.c_int, [vp, u64, u64, u64, dbl, u64, vp]),
    "hfpg_train_factors": (C.c_int, [C.POINTER(TrainFrameC), u64, C.POINTER(TrainFrameC), C.POINTER(TrainConfigC),
                                     u64, C.c_int, vp, C.POINTER(TrainLogC), u64, C.POINTER(TrainSummaryC)]),
    "hfpg_spmv": (C.c_int, [vp, vp, vp, C.c_int]),
    "hfpg_ic0_factor_host": (C.c_int, [u64, vp, vp, vp, i32, vp, vp, vp, u64, C.POINTER(u64),
                                       C.POINTER(dbl)]),
    "hfpg_load_ic0": (C.c_int, [vp, u64, vp, vp, vp]),
    "hfpg_crc32": (C.c_int, [vp, vp, u64, C.c_int, C.POINTER(C.c_uint32)]),
    "hfpg_payload_crc32": (C.c_int, [vp, u64, C.POINTER(C.c_uint32)]),
    "hfpg_load_checkpoint": (C.c_int, [vp, C.c_char_p]),
    "hfpg_write_mppf": (C.c_int, [vp, C.c_char_p]),
    "hfpg_read_mppf": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "hfpg_frame_meta": (C.c_int, [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(C.c_uint32), vp, C.c_uint32]),
    "hfpg_frame_create": (C.c_int, [u64, u64, u64, u64, u64, u64, dbl, C.c_uint32, vp, vp, vp, vp, vp, vp, vp,
                                    C.POINTER(vp)]),
    "hfpg_load_mppf": (C.c_int, [vp, C.c_char_p]),
    "hfpg_batch_apply": (C.c_int, [vp, vp, u64, u64, dbl, vp, u64, vp, C.c_int]),
    "hfpg_batch_adjoint": (C.c_int, [vp, vp, vp, vp, C.c_int]),
    "hfpg_loss_gradient": (C.c_int, [vp, vp, u64, u64, dbl, vp, u64, i32, dbl, C.POINTER(dbl),
                                     C.POINTER(i32), vp, C.c_int]),
    "hfpg_adamw_step": (C.c_int, [vp, vp, vp, vp, vp, u64, u64, dbl, dbl, dbl, dbl, dbl, dbl,
                                  C.POINTER(dbl)]),
    "hfpg_ic0_apply": (C.c_int, [vp, vp, vp, C.c_int]),
    "hfpg_apply_exact": (C.c_int, [vp, vp, vp, C.c_int]),
    "hfpg_set_residual_callback": (C.c_int, [vp, vp, vp]),
    "hfpg_pcg_solve": (C.c_int, [vp, vp, C.POINTER(SolveConfigC), vp, vp, C.POINTER(ReportC),
                                 C.c_int]),
    "hfpg_pcg_solve_exact": (C.c_int, [vp, vp, C.POINTER(SolveConfigC), vp, vp, C.POINTER(ReportC),
                                       C.c_int]),
    "hfpg_set_solver": (C.c_int, [vp, C.c_int]),
    "hfpg_solver_in_use": (C.c_int, [vp, C.POINTER(i32)]),
    "hfpg_set_trace": (C.c_int, [vp, C.c_uint32]),
    "hfpg_get_trace": (C.c_int, [vp, vp, C.c_uint32]),
    "hfpg_part_load": (C.c_int, [vp, C.c_uint32, C.c_uint32, u64, vp, vp, vp, u64, u64, vp, dbl, u64,
                                 u64, i32, dbl]),
    "hfpg_part_info": (C.c_int, [vp, vp]),
    "hfpg_part_mailbox": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp)]),
    "hfpg_part_connect": (C.c_int, [vp, vp, vp]),
    "hfpg_part_ipc_get": (C.c_int, [vp, vp]),
    "hfpg_part_ipc_connect": (C.c_int, [vp, vp]),
    "hfpg_group_pcg_solve": (C.c_int, [vp, C.c_uint32, vp, C.POINTER(SolveConfigC), vp, vp,
                                       C.POINTER(ReportC)]),
    "hfpg_group_apply": (C.c_int, [vp, C.c_uint32, vp, vp]),
    "hfpg_part_plan": (C.c_int, [u64, vp, vp, vp, u64, C.c_uint32, C.c_uint32, vp, vp, vp, vp, vp,
                                 vp]),
    "hfpg_part_factors": (C.c_int, [u64, u64, u64, C.c_uint32, C.c_uint32, vp, dbl, u64, u64, vp,
                                    vp]),
    "hfpg_pcg_solve_async": (C.c_int, [vp, vp, C.POINTER(SolveConfigC), vp, C.c_int]),
    "hfpg_pcg_solve_wait": (C.c_int, [vp, vp, C.POINTER(ReportC), C.c_int]),
    "hfpg_launch_counts": (C.c_int, [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "hfpg_fast_path": (C.c_int, [vp, C.POINTER(i32)]),
    "hfpg_profile_iteration": (C.c_int, [vp, C.c_uint32, vp]),
    "hfpg_gemm_tf32": (C.c_int, [u64, u64, u64, vp, vp, vp]),
    "hfpg_toynet_forward": (C.c_int, [vp, C.POINTER(FrameViewC), u64, u64, C.POINTER(ToynetConfigC),
                                      u64, vp, i32, C.POINTER(ToynetTraceC)]),
    "hfpg_toynet_forward_gpu_frame": (C.c_int, [vp, u64, u64, C.POINTER(ToynetConfigC), u64, vp, i32,
                                                vp]),
}

EXPORTED = sorted(_PROTOS)


def _load() -> C.CDLL:
    if not os.path.exists(SO_PATH):
        raise ImportError(
            f"{SO_PATH} is missing: build the native library first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(SO_PATH)
    for name, (res, args) in _PROTOS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    """Raise the Python analogue of the reference's exception for a failed call."""
    if rc == HFPG_OK:
        return
    msg = lib.hfpg_last_error().decode()
    if rc == HFPG_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == HFPG_ECUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)  # std::runtime_error (I/O, format, checksum)

# pcg.cpp:102 residual_vectors callback (hfpg_residual_fn)
RESIDUAL_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.POINTER(C.c_double), C.c_uint64)
