"""Row-partitioned PCG over G ranks (the north star's N=16.7M / 8-GPU configuration).

The system is split along the bisection tree (partition.cpp:9-46): rank r owns leaves
[r K/G, (r+1) K/G) and rows [r N/G, (r+1) N/G); only the G-1 tiles above the rank subtrees span
ranks and every rank recomputes them from exchanged subtree-root strip sums. Per iteration each
rank sends three small f64 messages to every rank through device mailboxes over peer memory
(include/hfpg.h, csrc/comm.cuh) plus its z halo rows; scalars are reduced in rank order so all
ranks take identical decisions.

* `PartitionGroup` — all G ranks in this process on one device, launched as one graph stage by
  stage (the way to run and check a partitioning on a single GPU).
* `RankSolver` — one rank per process / GPU; peers are mapped with CUDA IPC handles that are
  all-gathered through torch.distributed (any backend: the handles are 128 bytes per rank).
* `plan()` / `factor_slice()` — the host-side partition (no GPU needed).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._native import check, lib
from .api import CsrMatrix, Device, FactorTensor, SolveConfig, SolveReport, SolveStatus


@dataclass
class PartPlan:
    """Rank `rank`'s share: local columns (owned c - row0, ghosts n_local + i), ghost global ids,
    and the halo rows it pushes (grouped by peer via send_off) into peer ghost slots."""
    n_local: int
    row_begin: int
    ghost_cols: np.ndarray
    send_rows: np.ndarray
    send_slot: np.ndarray
    send_off: np.ndarray
    local_cols: np.ndarray


def plan(A: CsrMatrix, G: int, rank: int, leaf_size: int = 128) -> PartPlan:
    counts = np.zeros(4, np.uint64)
    args = (A.n_rows, A.row_offsets.ctypes.data, A.col_indices.ctypes.data, A.values.ctypes.data,
            leaf_size, G, rank)
    check(lib.hfpg_part_plan(*args, counts.ctypes.data, None, None, None, None, None))
    nl, ng, ns, nnz = (int(c) for c in counts)
    ghost = np.empty(ng, np.uint32)
    srows = np.empty(ns, np.uint32)
    sslot = np.empty(ns, np.uint32)
    soff = np.empty(G + 1, np.uint64)
    lcols = np.empty(nnz, np.uint32)
    check(lib.hfpg_part_plan(*args, counts.ctypes.data, ghost.ctypes.data, srows.ctypes.data,
                             sslot.ctypes.data, soff.ctypes.data, lcols.ctypes.data))
    return PartPlan(nl, rank * nl, ghost, srows, sslot, soff, lcols)


def factor_slice(n: int, G: int, rank: int, packed: np.ndarray | None = None, sigma: float = 0.0,
                 seed: int = 0, frame: int = 0, leaf_size: int = 128, coarse_size: int = 32):
    """(local packed tensor of size n/G, top tiles (G-1, L_s, L_s)) of rank `rank`."""
    from .api import build_partition, make_factor_layout
    Ll = make_factor_layout(build_partition(n // G, leaf_size), coarse_size)
    local = np.empty(Ll.total, np.float32)
    top = np.empty((G - 1) * coarse_size * coarse_size, np.float32)
    src = None if packed is None else np.ascontiguousarray(packed, np.float32).ctypes.data
    check(lib.hfpg_part_factors(n, leaf_size, coarse_size, G, rank, src, sigma, seed, frame,
                                local.ctypes.data, top.ctypes.data))
    return local, top


def _load(dev: Device, A: CsrMatrix, G: int, rank: int, factors: FactorTensor | None,
          sigma: float, seed: int, frame: int):
    packed = None if factors is None else factors.data.ctypes.data
    spd = (0, 0.0) if factors is None else (int(factors.spd_shift_enabled), float(factors.spd_shift_raw))
    check(lib.hfpg_part_load(dev.h, G, rank, A.n_rows, A.row_offsets.ctypes.data,
                             A.col_indices.ctypes.data, A.values.ctypes.data, 128, 32, packed,
                             sigma, seed, frame, spd[0], spd[1]))


def _report(rep, hist) -> SolveReport:
    return SolveReport(method="hfactor-gpu-partitioned", n=int(rep.n), iterations=int(rep.iterations),
                       converged=bool(rep.converged), status=SolveStatus(rep.status),
                       residual_history=hist[: rep.history_len].tolist(), wall_ms=float(rep.wall_ms),
                       breakdown_iter=int(rep.breakdown_iter))


class PartitionGroup:
    """All G ranks of a row-partitioned system in this process, on one device. The factors come
    from `factors` (the global tensor) or are drawn per slice as init_factors(sigma, seed, frame)."""

    def __init__(self, A: CsrMatrix, G: int, factors: FactorTensor | None = None, sigma: float = 0.0,
                 seed: int = 0, frame: int = 0, device: int = 0):
        self.n, self.G = A.n_rows, G
        self.devs = [Device(device) for _ in range(G)]
        for r, d in enumerate(self.devs):
            _load(d, A, G, r, factors, sigma, seed, frame)
        mb = (C.c_void_p * G)()
        zz = (C.c_void_p * G)()
        for r, d in enumerate(self.devs):
            a, b = N.vp(), N.vp()
            check(lib.hfpg_part_mailbox(d.h, C.byref(a), C.byref(b)))
            mb[r], zz[r] = a.value, b.value
        for d in self.devs:
            check(lib.hfpg_part_connect(d.h, mb, zz))
        self._hs = (C.c_void_p * G)(*[d.h.value for d in self.devs])

    def info(self, rank: int) -> dict:
        out = np.zeros(6, np.uint64)
        check(lib.hfpg_part_info(self.devs[rank].h, out.ctypes.data))
        return dict(zip(["n_local", "row_begin", "n_ghost", "halo_send", "G", "rank"], map(int, out)))

    def solve(self, b, cfg: SolveConfig | None = None):
        """pcg_solve (pcg.cpp:53-126) across the ranks; returns (SolveReport, x)."""
        cfg = cfg or SolveConfig()
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty(self.n)
        hist = np.empty(max(cfg.max_iters, 1))
        rep = N.ReportC()
        c = N.SolveConfigC(cfg.rtol, cfg.max_iters)
        check(lib.hfpg_group_pcg_solve(self._hs, self.G, b.ctypes.data, C.byref(c), x.ctypes.data,
                                       hist.ctypes.data, C.byref(rep)))
        return _report(rep, hist), x

    def apply(self, r) -> np.ndarray:
        """z = M r (apply.cpp:79-174) across the ranks."""
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty(self.n)
        check(lib.hfpg_group_apply(self._hs, self.G, r.ctypes.data, z.ctypes.data))
        return z


class RankSolver:
    """This process's rank of a G-rank partitioned system on `device`; `allgather(bytes) ->
    list[bytes]` exchanges the CUDA IPC handles (e.g. torch.distributed.all_gather_object)."""

    def __init__(self, A: CsrMatrix, G: int, rank: int, allgather, factors: FactorTensor | None = None,
                 sigma: float = 0.0, seed: int = 0, frame: int = 0, device: int = 0):
        self.G, self.rank = G, rank
        self.dev = Device(device)
        _load(self.dev, A, G, rank, factors, sigma, seed, frame)
        mine = (C.c_char * 128)()
        check(lib.hfpg_part_ipc_get(self.dev.h, mine))
        table = allgather(bytes(mine))
        allh = (C.c_char * (128 * G)).from_buffer_copy(b"".join(table))
        check(lib.hfpg_part_ipc_connect(self.dev.h, allh))
        out = np.zeros(6, np.uint64)
        check(lib.hfpg_part_info(self.dev.h, out.ctypes.data))
        self.n_local, self.row_begin = int(out[0]), int(out[1])

    def solve_ptr(self, b_ptr, x_ptr, cfg: SolveConfig, hist_ptr=None, where=N.DEVICE):
        """Local slices b[row_begin : row_begin + n_local] in, x out (pcg.cpp:53-126)."""
        return self.dev.solve_ptr(b_ptr, x_ptr, cfg, hist_ptr, where)

    def solve(self, b_local, cfg: SolveConfig | None = None):
        cfg = cfg or SolveConfig()
        b = np.ascontiguousarray(b_local, np.float64)
        x = np.empty(self.n_local)
        hist = np.empty(max(cfg.max_iters, 1))
        rep = self.dev.solve_ptr(b.ctypes.data, x.ctypes.data, cfg, hist.ctypes.data, N.HOST)
        return _report(rep, hist), x
