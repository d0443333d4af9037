"""paper_2605_13343_b200 — B200-native (sm_100a) PCG with the hierarchical-factor
preconditioner of arxiv 2605.13343, behind the reference `hfp` API.

The product is the native library `libhfpg.so` (C ABI in include/hfpg.h, CUDA kernels in
csrc/); this package is the Python mirror of the reference interface over that ABI.
"""
from .api import (Checkpoint, CsrMatrix, Device, FactorInit, FactorLayout, FactorTensor, Frame, GpuFrame,
                  HPartition, Ic0Factor, Ic0Shift, LossGradResult, LossKind, PrecondApplier, RngPurpose, RngStream, SolveConfig, SolveReport,
                  SolveStatus, TileSpec, ToynetConfig, ToynetTrace, adamw_step, apply, build_partition, factor_apply_batch, factor_apply_batch_adjoint, loss_gradient, clamp_leaf_size, factor_applier,
                  ic0_applier, ic0_factorize, identity_applier, init_factors, jacobi_applier, make_factor_layout, make_frame,
                  make_frame_3d, packed_width, pcg_solve, read_checkpoint, read_mppf, test_frame_id,
                  toynet_forward, toynet_forward_gpu_frame, train_frame_id, write_checkpoint, write_mppf,
                  PlateauConfig, TrainConfig, TrainHistory, TrainLogEntry, TrainResult, train_factors)

from .partition import PartitionGroup, RankSolver  # noqa: E402

__all__ = [n for n in dir() if not n.startswith("_")]
