"""Python mirror of the reference `hfp` API on the hot path, backed by libhfpg (sm_100a).

Names, argument meaning and error behaviour follow the reference headers so parity tests read
like the reference's own tests:

  partition.hpp     TileSpec, HPartition, build_partition, packed_width, clamp_leaf_size
  factor_tensor.hpp FactorLayout, make_factor_layout, FactorTensor (PackedFactors<float>),
                    FactorInit, init_factors
  rng.hpp           RngPurpose, RngStream (key only; draws happen natively)
  csr.hpp           CsrMatrix
  frame.hpp         make_frame (+ make_frame_3d, new)
  apply.hpp         apply
  pcg.hpp           SolveConfig, SolveStatus, SolveReport, identity_applier, jacobi_applier,
                    factor_applier, pcg_solve
  checkpoint.hpp    write_checkpoint, read_checkpoint, Checkpoint

std::invalid_argument maps to ValueError, std::runtime_error to RuntimeError. Every numeric
operation runs in libhfpg: the appliers and pcg_solve execute on the GPU, the partition /
layout / seeded initialisation / frame generation in the library's native host code.
"""
from __future__ import annotations

import ctypes as C
import json
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import check, lib

# ---------------------------------------------------------------------------- partition.hpp


@dataclass
class TileSpec:
    id: int
    span: int
    row_begin: int
    col_begin: int
    depth: int


@dataclass
class HPartition:
    n: int
    leaf_size: int
    leaf_count: int
    tiles: list
    admissibility: int = 1
    row_tiles_of_leaf: list = field(default_factory=list)
    col_tiles_of_leaf: list = field(default_factory=list)

    def tile_count(self) -> int:
        return len(self.tiles)

    def leaf_begin(self, k: int) -> int:
        return k * self.leaf_size


def build_partition(n: int, leaf_size: int) -> HPartition:
    """partition.cpp:9-46."""
    cnt = N.u64()
    check(lib.hfpg_build_partition(n, leaf_size, None, 0, C.byref(cnt)))
    arr = (N.Tile * max(cnt.value, 1))()
    check(lib.hfpg_build_partition(n, leaf_size, arr, cnt.value, C.byref(cnt)))
    k = n // leaf_size
    tiles = [TileSpec(t.id, t.span, t.row_begin, t.col_begin, t.depth)
             for t in arr[: cnt.value]]
    p = HPartition(n, leaf_size, k, tiles)
    p.row_tiles_of_leaf = [[] for _ in range(k)]
    p.col_tiles_of_leaf = [[] for _ in range(k)]
    for t in tiles:
        for s in range(t.span):
            p.row_tiles_of_leaf[t.row_begin + s].append(t.id)
            p.col_tiles_of_leaf[t.col_begin + s].append(t.id)
    return p


def packed_width(p: HPartition, coarse_size: int) -> int:
    """partition.cpp:48-53."""
    out = N.u64()
    check(lib.hfpg_packed_width(p.n, p.leaf_size, coarse_size, C.byref(out)))
    return out.value


def clamp_leaf_size(n: int, leaf_size: int) -> int:
    """partition.hpp:48-50."""
    return n // 2 if n < 2 * leaf_size else leaf_size


# ------------------------------------------------------------------------ factor_tensor.hpp


@dataclass
class FactorLayout:
    n: int
    leaf_size: int
    coarse_size: int
    coupling_rank: int
    leaf_count: int
    tile_count: int
    leaf_base: int
    tile_base: int
    bridge_base: int
    gate_base: int
    total: int
    tiles: list

    def leaf_factor(self, k):
        return self.leaf_base + k * self.leaf_size * self.leaf_size

    def tile_u(self, m):
        return self.tile_base + m * self.coarse_size * self.coarse_size

    def tile_v(self, m):
        return self.tile_u(m) + self.coarse_size * self.coupling_rank

    def bridge_u(self, k):
        return self.bridge_base + k * 2 * self.leaf_size * self.coarse_size

    def bridge_v(self, k):
        return self.bridge_u(k) + self.leaf_size * self.coarse_size

    def gate(self):
        return self.gate_base


def make_factor_layout(partition: HPartition, coarse_size: int) -> FactorLayout:
    """factor_tensor.cpp:7-28."""
    lay = N.Layout()
    check(lib.hfpg_factor_layout(partition.n, partition.leaf_size, coarse_size, C.byref(lay)))
    return FactorLayout(*(getattr(lay, f) for f, _ in N.Layout._fields_), tiles=partition.tiles)


class FactorTensor:
    """PackedFactors<float> (factor_tensor.hpp:57-112): one contiguous float32 array."""

    def __init__(self, layout: FactorLayout, data: np.ndarray | None = None):
        self.layout = layout
        self.data = (np.zeros(layout.total, np.float32) if data is None
                     else np.ascontiguousarray(data, dtype=np.float32))
        if self.data.shape != (layout.total,):
            raise ValueError("factor tensor: packed width mismatch")
        self.spd_shift_enabled = False
        self.spd_shift_raw = 0.0

    def spd_shift(self) -> float:
        return math.log1p(math.exp(self.spd_shift_raw)) if self.spd_shift_enabled else 0.0

    def _sec(self, off, cnt, shape):
        return self.data[off: off + cnt].reshape(shape)

    def leaf_factor(self, k):
        L = self.layout
        return self._sec(L.leaf_factor(k), L.leaf_size ** 2, (L.leaf_size, L.leaf_size))

    def tile_u(self, m):
        L = self.layout
        return self._sec(L.tile_u(m), L.coarse_size * L.coupling_rank,
                         (L.coarse_size, L.coupling_rank))

    def tile_v(self, m):
        L = self.layout
        return self._sec(L.tile_v(m), L.coarse_size * L.coupling_rank,
                         (L.coarse_size, L.coupling_rank))

    def bridge_u(self, k):
        L = self.layout
        return self._sec(L.bridge_u(k), L.leaf_size * L.coarse_size, (L.leaf_size, L.coarse_size))

    def bridge_v(self, k):
        L = self.layout
        return self._sec(L.bridge_v(k), L.leaf_size * L.coarse_size, (L.leaf_size, L.coarse_size))

    def gate(self):
        return self.data[self.layout.gate_base: self.layout.total]

    def copy(self) -> "FactorTensor":
        f = FactorTensor(self.layout, self.data.copy())
        f.spd_shift_enabled, f.spd_shift_raw = self.spd_shift_enabled, self.spd_shift_raw
        return f


class RngPurpose(enum.IntEnum):
    """rng.hpp:12-20 (frozen values)."""
    density = 1
    rhs = 2
    probes = 3
    factor_init = 4
    net_weights = 5
    power_iter = 6
    test = 7


@dataclass
class RngStream:
    """rng.hpp:37-41 key. Draws are made natively at counter 0.. by the consumer."""
    seed: int
    frame: int
    purpose: RngPurpose


class FactorInit(enum.Enum):
    jacobi_seed = 0
    random = 1


def init_factors(partition: HPartition, coarse_size: int, mode: FactorInit, sigma: float,
                 stream: RngStream) -> FactorTensor:
    """factor_tensor.cpp:30-39 (bit-identical; drawn in parallel from the counter stream)."""
    if stream.purpose != RngPurpose.factor_init:
        raise ValueError("init_factors: native draws use the factor_init purpose key")
    lay = make_factor_layout(partition, coarse_size)
    out = np.empty(lay.total, np.float32)
    check(lib.hfpg_init_factors(partition.n, partition.leaf_size, coarse_size, float(sigma),
                                stream.seed, stream.frame, out.ctypes.data))
    return FactorTensor(lay, out)


# ---------------------------------------------------------------------------------- csr.hpp


class CsrMatrix:
    """csr.hpp:11-30: u64 row offsets, u32 columns, f64 values."""

    def __init__(self, n_rows, n_cols, row_offsets, col_indices, values):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_offsets = np.ascontiguousarray(row_offsets, np.uint64)
        self.col_indices = np.ascontiguousarray(col_indices, np.uint32)
        self.values = np.ascontiguousarray(values, np.float64)

    def nnz(self) -> int:
        return len(self.values)

    def diagonal(self) -> np.ndarray:
        """csr.cpp:52-58."""
        d = np.zeros(self.n_rows)
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_offsets).astype(np.int64))
        m = self.col_indices == rows
        d[rows[m]] = self.values[m]
        return d


@dataclass
class Frame:
    """frame.hpp:26-40 (what the path consumes)."""
    n: int
    width: int
    height: int
    depth: int
    cell_order: np.ndarray
    rho: np.ndarray
    A: CsrMatrix
    b: np.ndarray
    rho_heavy: float
    master_seed: int = 0
    frame_index: int = 0
    barriers: list = field(default_factory=list)  # frame.hpp:37: (orientation, center, thickness, gap)


def _frame_from_handle(h, seed, fidx) -> Frame:
    n, nnz, w, hh, d = (N.u64() for _ in range(5))
    rh = N.dbl()
    check(lib.hfpg_frame_info(h, C.byref(n), C.byref(nnz), C.byref(w), C.byref(hh), C.byref(d),
                              C.byref(rh)))
    co = np.empty(n.value, np.uint32)
    rho = np.empty(n.value)
    ro = np.empty(n.value + 1, np.uint64)
    ci = np.empty(nnz.value, np.uint32)
    v = np.empty(nnz.value)
    b = np.empty(n.value)
    check(lib.hfpg_frame_copy(h, co.ctypes.data, rho.ctypes.data, ro.ctypes.data,
                              ci.ctypes.data, v.ctypes.data, b.ctypes.data))
    sd, fi, nb = N.u64(), N.u64(), C.c_uint32()
    bars = np.zeros(4 * 8)
    check(lib.hfpg_frame_meta(h, C.byref(sd), C.byref(fi), C.byref(nb), bars.ctypes.data, 8))
    lib.hfpg_frame_free(h)
    seed = sd.value if seed is None else seed
    fidx = fi.value if fidx is None else fidx
    return Frame(n.value, w.value, hh.value, d.value, co, rho,
                 CsrMatrix(n.value, n.value, ro, ci, v), b, rh.value, seed, fidx,
                 [tuple(float(x) for x in bars[4 * i:4 * i + 4]) for i in range(min(nb.value, 8))])


def write_mppf(frame: Frame, path: str) -> None:
    """mppf.cpp:48-100 (MPPF v1; per-section zlib crc32; 2D frames)."""
    bars = np.array([x for bar in frame.barriers for x in bar], np.float64) if frame.barriers else np.zeros(1)
    co = np.ascontiguousarray(frame.cell_order, np.uint32)
    rho = np.ascontiguousarray(frame.rho, np.float64)
    ro = np.ascontiguousarray(frame.A.row_offsets, np.uint64)
    ci = np.ascontiguousarray(frame.A.col_indices, np.uint32)
    v = np.ascontiguousarray(frame.A.values, np.float64)
    b = np.ascontiguousarray(frame.b, np.float64)
    h = N.vp()
    check(lib.hfpg_frame_create(frame.n, frame.width, frame.height, frame.depth, frame.master_seed,
                                frame.frame_index, frame.rho_heavy, len(frame.barriers), bars.ctypes.data,
                                co.ctypes.data, rho.ctypes.data, ro.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                b.ctypes.data, C.byref(h)))
    try:
        check(lib.hfpg_write_mppf(h, str(path).encode()))
    finally:
        lib.hfpg_frame_free(h)


def read_mppf(path: str) -> Frame:
    """mppf.cpp:102-177: checksums, CSR invariants (ValueError, like std::invalid_argument),
    format errors (RuntimeError), Morton cell order recomputed."""
    h = N.vp()
    check(lib.hfpg_read_mppf(str(path).encode(), C.byref(h)))
    return _frame_from_handle(h, None, None)


def make_frame(n: int, master_seed: int, frame_index: int) -> Frame:
    """frame.cpp:161-181 (bit-identical native generator)."""
    h = N.vp()
    check(lib.hfpg_frame_2d(n, master_seed, frame_index, C.byref(h)))
    return _frame_from_handle(h, master_seed, frame_index)


def make_frame_3d(nx: int, ny: int, nz: int, master_seed: int, frame_index: int) -> Frame:
    """3D analogue of make_frame (new; see include/hfpg.h)."""
    h = N.vp()
    check(lib.hfpg_frame_3d(nx, ny, nz, master_seed, frame_index, C.byref(h)))
    return _frame_from_handle(h, master_seed, frame_index)


def train_frame_id(scale: int, i: int) -> int:
    return (scale << 24) | i


def test_frame_id(scale: int, i: int) -> int:
    return (scale << 24) | (1 << 20) | i


# --------------------------------------------------------------------------- device handle


@dataclass
class GpuFrame:
    """A frame generated on the device (Device.frame_gpu / frame_gpu_3d) and loaded as that
    device's system; `b`, `rho`, ... are device pointers, valid until the next frame."""
    n: int
    nnz: int
    width: int
    height: int
    depth: int
    rho_heavy: float
    cell_order: int
    rho: int
    row_offsets: int
    col_indices: int
    values: int
    b: int
    a_diag: int
    generate_ms: float
    frobenius: float
    master_seed: int
    frame_index: int
    device: "Device"

    def to_host(self) -> Frame:
        """Download as a host Frame (same fields as make_frame / make_frame_3d)."""
        co = np.empty(self.n, np.uint32)
        rho = np.empty(self.n)
        ro = np.empty(self.n + 1, np.uint64)
        ci = np.empty(self.nnz, np.uint32)
        v = np.empty(self.nnz)
        b = np.empty(self.n)
        check(lib.hfpg_frame_gpu_copy(self.device.h, co.ctypes.data, rho.ctypes.data, ro.ctypes.data,
                                      ci.ctypes.data, v.ctypes.data, b.ctypes.data))
        return Frame(self.n, self.width, self.height, self.depth, co, rho,
                     CsrMatrix(self.n, self.n, ro, ci, v), b, self.rho_heavy, self.master_seed,
                     self.frame_index)


class Device:
    """One hfpg handle: a CUDA stream + device-resident operator, factors and workspace."""

    def __init__(self, device: int = 0):
        h = N.vp()
        check(lib.hfpg_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.csr_id = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib.hfpg_destroy(h)
            self.h = None

    def load_csr(self, A: CsrMatrix):
        check(lib.hfpg_load_csr(self.h, A.n_rows, A.row_offsets.ctypes.data,
                                A.col_indices.ctypes.data, A.values.ctypes.data, N.HOST))
        self.csr_id = id(A)
        # content snapshot: a solve must use the A it is handed (pcg.cpp:53), even if the caller
        # edited the arrays in place or a new matrix reuses a freed object's id
        self._csr_snap = (A.n_rows, A.row_offsets.copy(), A.col_indices.copy(), A.values.view(np.uint64).copy())

    def holds_csr(self, A: CsrMatrix) -> bool:
        """True when the device operator is bit-identical to A (structure and values)."""
        snap = getattr(self, "_csr_snap", None)
        if snap is None or snap[0] != A.n_rows or len(snap[3]) != len(A.values):
            return False
        return (np.array_equal(snap[1], A.row_offsets) and np.array_equal(snap[2], A.col_indices)
                and np.array_equal(snap[3], A.values.view(np.uint64)))

    def _gpu_frame(self, seed, fidx) -> GpuFrame:
        v = N.FrameDeviceC()
        check(lib.hfpg_frame_gpu_view(self.h, C.byref(v)))
        self.csr_id = ("gpu_frame", seed, fidx)
        self._csr_snap = None
        return GpuFrame(v.n, v.nnz, v.width, v.height, v.depth, v.rho_heavy, v.cell_order or 0,
                        v.rho or 0, v.row_offsets or 0, v.col_indices or 0, v.values or 0, v.b or 0,
                        v.a_diag or 0, float(v.generate_ms), float(v.frobenius), seed, fidx, self)

    def frame_gpu(self, n: int, master_seed: int, frame_index: int) -> GpuFrame:
        """make_frame (frame.cpp:161-181) generated on this device and loaded as its system."""
        check(lib.hfpg_frame_gpu_2d(self.h, n, master_seed, frame_index))
        return self._gpu_frame(master_seed, frame_index)

    def frame_gpu_3d(self, nx: int, ny: int, nz: int, master_seed: int, frame_index: int) -> GpuFrame:
        """make_frame_3d generated on this device and loaded as its system."""
        check(lib.hfpg_frame_gpu_3d(self.h, nx, ny, nz, master_seed, frame_index))
        return self._gpu_frame(master_seed, frame_index)

    def load_csr_device(self, n, ro_ptr, ci_ptr, v_ptr):
        check(lib.hfpg_load_csr(self.h, n, ro_ptr, ci_ptr, v_ptr, N.DEVICE))
        self.csr_id = ("device", ro_ptr, ci_ptr, v_ptr)
        self._csr_snap = None

    def load_mppf(self, path: str) -> "GpuFrame":
        """read_mppf on the device (pinned streaming, GPU crc32 and CSR checks); the frame becomes
        this handle's system and GPU frame."""
        check(lib.hfpg_load_mppf(self.h, str(path).encode()))
        g = self._gpu_frame(None, None)
        self.csr_id = ("mppf", str(path))
        return g

    def load_checkpoint(self, path: str):
        """read_checkpoint straight into device memory (pinned streaming, GPU crc32)."""
        check(lib.hfpg_load_checkpoint(self.h, str(path).encode()))

    def crc32(self, data, where: int | None = None) -> int:
        """zlib crc32 of a numpy array (host, zlib) or a device pointer + size (GPU)."""
        out = C.c_uint32()
        if isinstance(data, np.ndarray):
            a = np.ascontiguousarray(data)
            check(lib.hfpg_crc32(self.h, a.ctypes.data, a.nbytes, N.HOST, C.byref(out)))
        else:
            ptr, nbytes = data
            check(lib.hfpg_crc32(self.h, ptr, nbytes, N.DEVICE if where is None else where, C.byref(out)))
        return out.value

    def load_factors(self, f: FactorTensor):
        L = f.layout
        check(lib.hfpg_load_factors(self.h, L.n, L.leaf_size, L.coarse_size, f.data.ctypes.data,
                                    L.total, int(f.spd_shift_enabled), float(f.spd_shift_raw),
                                    N.HOST))

    def set_diag(self, a_diag: np.ndarray):
        a = np.ascontiguousarray(a_diag, np.float64)
        check(lib.hfpg_set_diag(self.h, len(a), a.ctypes.data, N.HOST))

    def set_precond(self, kind: int):
        check(lib.hfpg_set_precond(self.h, kind))

    def apply(self, r: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        check(lib.hfpg_apply(self.h, r.ctypes.data, z.ctypes.data, N.HOST))
        return z

    def apply_ptr(self, r_ptr: int, z_ptr: int, where: int = N.DEVICE):
        check(lib.hfpg_apply(self.h, r_ptr, z_ptr, where))

    def apply_exact(self, r: np.ndarray) -> np.ndarray:
        """apply<float> bit for bit (hfpg_apply_exact; the exact PCG's factor preconditioner)."""
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        check(lib.hfpg_apply_exact(self.h, r.ctypes.data, z.ctypes.data, N.HOST))
        return z

    def spmv(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        check(lib.hfpg_spmv(self.h, x.ctypes.data, y.ctypes.data, N.HOST))
        return y

    def spmv_ptr(self, x_ptr: int, y_ptr: int, where: int = N.DEVICE):
        check(lib.hfpg_spmv(self.h, x_ptr, y_ptr, where))

    def solve_ptr(self, b_ptr, x_ptr, cfg: "SolveConfig", hist_ptr=None, where=N.DEVICE, exact: bool = False):
        rep = N.ReportC()
        c = N.SolveConfigC(cfg.rtol, cfg.max_iters)
        fn = lib.hfpg_pcg_solve_exact if exact else lib.hfpg_pcg_solve
        check(fn(self.h, b_ptr, C.byref(c), x_ptr, hist_ptr, C.byref(rep), where))
        return rep

    def solve_async(self, b_ptr, x_ptr, cfg: "SolveConfig", where=N.DEVICE):
        """Enqueue a solve on this handle's stream (hfpg_pcg_solve_async); finish with wait()."""
        c = N.SolveConfigC(cfg.rtol, cfg.max_iters)
        check(lib.hfpg_pcg_solve_async(self.h, b_ptr, C.byref(c), x_ptr, where))

    def wait(self, hist_ptr=None, where=N.DEVICE):
        rep = N.ReportC()
        check(lib.hfpg_pcg_solve_wait(self.h, hist_ptr, C.byref(rep), where))
        return rep

    def set_solver(self, kind: int):
        """N.SOLVER_AUTO / SOLVER_GRAPH / SOLVER_PERSISTENT (include/hfpg.h hfpg_solver)."""
        check(lib.hfpg_set_solver(self.h, kind))

    def solver_in_use(self) -> int:
        v = N.i32()
        check(lib.hfpg_solver_in_use(self.h, C.byref(v)))
        return v.value

    def stream(self) -> int:
        s = N.vp()
        check(lib.hfpg_get_stream(self.h, C.byref(s)))
        return s.value or 0

    def fast_path(self) -> bool:
        v = N.i32()
        check(lib.hfpg_fast_path(self.h, C.byref(v)))
        return bool(v.value)

    def launch_counts(self):
        a, b = C.c_uint32(), C.c_uint32()
        check(lib.hfpg_launch_counts(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value


# ---------------------------------------------------------------------------------- pcg.hpp


@dataclass
class SolveConfig:
    rtol: float = 1e-8
    max_iters: int = 20000


class SolveStatus(enum.Enum):
    converged = 0
    max_iters = 1
    breakdown = 2


@dataclass
class SolveReport:
    method: str = ""
    n: int = 0
    iterations: int = 0
    converged: bool = False
    status: SolveStatus = SolveStatus.max_iters
    residual_history: list = field(default_factory=list)
    wall_ms: float = 0.0
    frame_id: str = ""
    breakdown_iter: int = 0

    def to_json(self) -> str:
        """pcg.cpp:12-26 (same keys; breakdown_iter only on breakdown)."""
        import json
        j = {"method": self.method, "n": self.n, "iterations": self.iterations, "converged": self.converged,
             "status": self.status.name, "wall_ms": self.wall_ms, "frame_id": self.frame_id}
        if self.status == SolveStatus.breakdown:
            j["breakdown_iter"] = self.breakdown_iter
        j["residual_history"] = list(self.residual_history)
        return json.dumps(j, separators=(",", ":"))


class PrecondApplier:
    """pcg.hpp:36: callable z = M r (host arrays; H2D -> device apply -> D2H, for parity and
    plug compatibility). pcg_solve runs the same preconditioner device-resident."""

    kind = N.vp  # overridden

    def __init__(self, device: Device | None):
        self.dev = device

    def bind(self, A: CsrMatrix) -> Device:
        if self.dev is None:
            self.dev = Device(0)
        if not self.dev.holds_csr(A):
            self.dev.load_csr(A)
        self.dev.set_precond(self.kind)
        return self.dev


class _Identity(PrecondApplier):
    kind = 0
    method = "none"

    def __call__(self, r):
        return np.array(r, dtype=np.float64, copy=True)


class _Jacobi(PrecondApplier):
    kind = 1
    method = "jacobi"

    def __init__(self, A: CsrMatrix):
        super().__init__(Device(0))
        self.dev.load_csr(A)
        self.dev.set_precond(1)  # throws ValueError on a nonpositive diagonal (pcg.cpp:36-38)

    def __call__(self, r):
        """pcg.cpp:40: z_i = r_i / a_ii, on the device (hfpg_precond_apply)."""
        r = np.ascontiguousarray(r, np.float64)
        if len(r) != self.dev_n():
            raise ValueError("apply: length mismatch")
        z = np.empty_like(r)
        self.dev.set_precond(self.kind)
        check(lib.hfpg_precond_apply(self.dev.h, r.ctypes.data, z.ctypes.data, N.HOST))
        return z

    def dev_n(self) -> int:
        return len(self.dev._csr_snap[1]) - 1


class _Factor(PrecondApplier):
    kind = 2
    method = "hfactor-gpu"

    def __init__(self, factors: FactorTensor, A: CsrMatrix):
        super().__init__(Device(0))
        self.dev.load_csr(A)
        self.dev.load_factors(factors)

    def __call__(self, r):
        return self.dev.apply(r)


# ------------------------------------------------------------------ adjoint.hpp / train.cpp


class LossKind(enum.IntEnum):
    """loss.hpp: cosine (1 - cos(Z, M A Z)) or sai (|(1/normA) A M Z - Z|_F^2)."""
    cosine = 0
    sai = 1


def _f64(a):
    return np.ascontiguousarray(a, np.float64)


def factor_apply_batch(params, x, kz: int, device: "Device", shift: float = 0.0) -> np.ndarray:
    """adjoint.cpp:44-127: Y = M X (row-major n x kz, double precision, stages stashed on the
    device for factor_apply_batch_adjoint). diag(A) is the device's loaded system's."""
    x = _f64(x)
    y = np.empty_like(x)
    p = _f64(params)
    check(lib.hfpg_batch_apply(device.h, p.ctypes.data, 128, 32, float(shift), x.ctypes.data, kz,
                               y.ctypes.data, N.HOST))
    return y


def factor_apply_batch_adjoint(params, bar_y, device: "Device") -> np.ndarray:
    """adjoint.cpp:129-248: d(loss)/d(params) for the upstream adjoint bar_y of the last batch."""
    p = _f64(params)
    by = _f64(bar_y)
    g = np.empty_like(p)
    check(lib.hfpg_batch_adjoint(device.h, p.ctypes.data, by.ctypes.data, g.ctypes.data, N.HOST))
    return g


@dataclass
class LossGradResult:
    loss: float
    degenerate: bool
    grad: np.ndarray


def loss_gradient(params, z, kz: int, kind: LossKind, device: "Device", norm_a: float = 1.0,
                  shift: float = 0.0) -> LossGradResult:
    """adjoint.cpp:250-292 on the device's loaded system."""
    p = _f64(params)
    z = _f64(z)
    g = np.empty_like(p)
    loss, deg = N.dbl(), N.i32()
    check(lib.hfpg_loss_gradient(device.h, p.ctypes.data, 128, 32, float(shift), z.ctypes.data, kz,
                                 int(kind), float(norm_a), C.byref(loss), C.byref(deg), g.ctypes.data, N.HOST))
    return LossGradResult(float(loss.value), bool(deg.value), g)


def adamw_step(device: "Device", params_ptr: int, grad_ptr: int, m1_ptr: int, m2_ptr: int, count: int,
               step: int, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
               weight_decay: float = 0.0, clip_norm: float = float("inf")) -> float:
    """train.cpp:136-160 on device buffers (global clip, AdamW); returns the gradient norm."""
    gn = N.dbl()
    check(lib.hfpg_adamw_step(device.h, params_ptr, grad_ptr, m1_ptr, m2_ptr, count, step, lr, beta1, beta2,
                              eps, weight_decay, clip_norm, C.byref(gn)))
    return float(gn.value)


@dataclass
class PlateauConfig:
    """train.hpp:12-17."""
    factor: float = 0.5
    patience: int = 5
    rel_threshold: float = 5e-3


@dataclass
class TrainConfig:
    """train.hpp:19-40 (defaults as the reference's)."""
    lr: float = 2e-4
    weight_decay: float = 1e-4
    clip_norm: float = 1.0
    plateau: PlateauConfig = field(default_factory=PlateauConfig)
    max_steps: int = 100000
    autostop_window: int = 10
    probe_omega: float = 0.6
    probe_smooth_steps: int = 2
    contexts_per_step: int = 4
    loss: LossKind = LossKind.cosine
    log_every: int = 100
    init_sigma: float = 1e-2
    leaf_size: int = 128
    coarse_size: int = 32
    eval_every_logs: int = 1
    solve_rtol: float = 1e-8
    solve_max_iters: int = 20000
    stop_at_iters: int = 0

    def to_c(self) -> "N.TrainConfigC":
        return N.TrainConfigC(self.lr, self.weight_decay, self.clip_norm, self.plateau.factor, self.plateau.patience,
                              self.plateau.rel_threshold, self.max_steps, self.autostop_window, self.probe_omega,
                              self.probe_smooth_steps, self.contexts_per_step, int(self.loss), self.log_every,
                              self.init_sigma, self.leaf_size, self.coarse_size, self.eval_every_logs,
                              self.solve_rtol, self.solve_max_iters, self.stop_at_iters)


@dataclass
class TrainLogEntry:
    """train.hpp:42-49."""
    step: int = 0
    train_loss: float = 0.0
    sai_heldout: float = 0.0
    pcg_iters_heldout: int = 0
    lr: float = 0.0
    wall_s: float = 0.0


@dataclass
class TrainHistory:
    """train.hpp:51-58; to_jsonl as train.cpp:13-27."""
    entries: list = field(default_factory=list)
    auto_stopped: bool = False
    aborted_divergence: bool = False
    reached_target: bool = False
    total_steps: int = 0

    def to_jsonl(self) -> str:
        return "".join(json.dumps({"step": e.step, "train_loss": e.train_loss, "sai_heldout": e.sai_heldout,
                                   "pcg_iters_heldout": e.pcg_iters_heldout, "lr": e.lr, "wall_s": e.wall_s},
                                  separators=(",", ":")) + "\n" for e in self.entries)


@dataclass
class TrainResult:
    """train.hpp:60-63."""
    factors: "FactorTensor"
    history: TrainHistory


def _train_frame(fr: Frame) -> "N.TrainFrameC":
    v = _frame_view(fr)
    t = N.TrainFrameC(v, fr.b.ctypes.data, int(fr.frame_index))
    t._keep = (v, fr)
    return t


def train_factors(frames, cfg: TrainConfig | None = None, seed: int = 0, eval_frame: Frame | None = None,
                  device: int = 0) -> TrainResult:
    """train.cpp:29-217 on the GPU (train_loop.cu): AdamW with decoupled weight decay, global
    clip, reduce-on-plateau, min-lr auto-stop, divergence abort; each step averages
    contexts_per_step fresh smoothed probe batches; the held-out evaluation runs the exact PCG."""
    cfg = cfg or TrainConfig()
    frames = list(frames)
    if not frames:
        raise ValueError("train_factors: no frames")
    tf = (N.TrainFrameC * len(frames))(*[_train_frame(f) for f in frames])
    keep = [f for f in frames]
    ev = _train_frame(eval_frame) if eval_frame is not None else None
    n = frames[0].n
    leaf = clamp_leaf_size(n, cfg.leaf_size)
    lay = make_factor_layout(build_partition(n, leaf), cfg.coarse_size)
    out = np.empty(lay.total, np.float32)
    cap = max(1, cfg.max_steps // max(cfg.log_every, 1) + 1)
    logs = (N.TrainLogC * cap)()
    summ = N.TrainSummaryC()
    c = cfg.to_c()
    check(lib.hfpg_train_factors(tf, len(frames), C.byref(ev) if ev is not None else None, C.byref(c), seed,
                                 device, out.ctypes.data, logs, cap, C.byref(summ)))
    del keep
    hist = TrainHistory([TrainLogEntry(int(e.step), float(e.train_loss), float(e.sai_heldout),
                                       int(e.pcg_iters_heldout), float(e.lr), float(e.wall_s))
                         for e in logs[: min(int(summ.n_entries), cap)]],
                        bool(summ.auto_stopped), bool(summ.aborted_divergence), bool(summ.reached_target),
                        int(summ.total_steps))
    return TrainResult(FactorTensor(lay, out), hist)


class Ic0Shift(enum.IntEnum):
    """ic0.hpp:7: scaled factors A + 1e-8 max(diag) I."""
    none = 0
    scaled = 1


@dataclass
class Ic0Factor:
    """ic0.hpp:10-13: the lower factor (pattern = lower triangle of A, diagonal last) + shift."""
    lower: "CsrMatrix"
    shift: float = 0.0


def ic0_factorize(A: "CsrMatrix", policy: Ic0Shift = Ic0Shift.scaled) -> Ic0Factor:
    """ic0.cpp:10-69 (host C++ in libhfpg, bit-identical to the reference). Raises ValueError on
    a non-square matrix and RuntimeError on a nonpositive pivot, like the reference's
    std::invalid_argument / std::runtime_error."""
    if A.n_rows != A.n_cols:
        raise ValueError("ic0_factorize: matrix not square")
    n = A.n_rows
    ro = np.ascontiguousarray(A.row_offsets, np.uint64)
    ci = np.ascontiguousarray(A.col_indices, np.uint32)
    v = np.ascontiguousarray(A.values, np.float64)
    cap = int(ro[-1]) + n
    lro = np.empty(n + 1, np.uint64)
    lci = np.empty(max(cap, 1), np.uint32)
    lv = np.empty(max(cap, 1), np.float64)
    nnz = N.u64()
    shift = N.dbl()
    rc = N.lib.hfpg_ic0_factor_host(n, ro.ctypes.data, ci.ctypes.data, v.ctypes.data, int(policy),
                                    lro.ctypes.data, lci.ctypes.data, lv.ctypes.data, cap,
                                    N.C.byref(nnz), N.C.byref(shift))
    N.check(rc)
    k = int(nnz.value)
    return Ic0Factor(CsrMatrix(n, n, lro, lci[:k].copy(), lv[:k].copy()), float(shift.value))


class _Ic0(PrecondApplier):
    kind = 3
    method = "ic0"

    def __init__(self, factor: Ic0Factor, A: "CsrMatrix | None" = None):
        super().__init__(Device(0))
        self.factor = factor
        if A is not None:
            self.bind(A)

    def bind(self, A: "CsrMatrix") -> Device:
        if not self.dev.holds_csr(A):
            self.dev.load_csr(A)
        L = self.factor.lower
        lro = np.ascontiguousarray(L.row_offsets, np.uint64)
        lci = np.ascontiguousarray(L.col_indices, np.uint32)
        lv = np.ascontiguousarray(L.values, np.float64)
        N.check(N.lib.hfpg_load_ic0(self.dev.h, L.n_rows, lro.ctypes.data, lci.ctypes.data, lv.ctypes.data))
        self.dev.set_precond(self.kind)
        return self.dev

    def __call__(self, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty_like(r)
        if self.dev.csr_id is None:  # a bare applier: the factor alone defines the operator
            L = self.factor.lower
            self.bind(CsrMatrix(L.n_rows, L.n_cols, L.row_offsets, L.col_indices, L.values))
        N.check(N.lib.hfpg_ic0_apply(self.dev.h, r.ctypes.data, z.ctypes.data, N.HOST))
        return z


def ic0_applier(factor: Ic0Factor) -> PrecondApplier:
    """ic0.cpp:72-99: z = (L L^T)^{-1} r — two sync-free triangular sweeps on the GPU. Bind it
    to the system (pcg_solve does) to run the device-resident IC(0)-PCG."""
    return _Ic0(factor)


def identity_applier() -> PrecondApplier:
    return _Identity(None)


def jacobi_applier(A: CsrMatrix) -> PrecondApplier:
    return _Jacobi(A)


def factor_applier(factors: FactorTensor, A: CsrMatrix) -> PrecondApplier:
    """pcg.cpp:44-51: owning copy of the tensor and diag(A) — on the GPU."""
    return _Factor(factors, A)


def pcg_solve(A: CsrMatrix, b, precond: PrecondApplier, cfg: SolveConfig | None = None,
              x_out: list | None = None, exact: bool = False,
              residual_vectors: list | None = None) -> SolveReport:
    """pcg.cpp:53-126, whole loop in one CUDA graph. If x_out is a list, the solution is
    appended to it (the reference's optional std::vector<double>* out-parameter).
    exact=True: every dot product as the reference's sequential loop (hfpg_pcg_solve_exact), so
    x, the history and the iteration count are the reference's bit for bit (slower).
    residual_vectors: a list receiving r_k after every iteration (pcg.cpp:102); delivered by the
    host-driven exact loop, so it implies exact=True."""
    cfg = cfg or SolveConfig()
    if cfg.rtol <= 0.0:
        raise ValueError("pcg_solve: rtol must be positive")
    b = np.ascontiguousarray(b, np.float64)
    if b.shape != (A.n_rows,):
        raise ValueError("pcg_solve: rhs length mismatch")
    dev = precond.bind(A)
    x = np.empty(A.n_rows)
    hist = np.empty(max(cfg.max_iters, 1))
    if residual_vectors is not None:
        exact = True
        cb = N.RESIDUAL_FN(lambda _u, _k, r, n: residual_vectors.append(np.ctypeslib.as_array(r, (n,)).copy()))
        check(lib.hfpg_set_residual_callback(dev.h, C.cast(cb, C.c_void_p), None))
    try:
        rep = dev.solve_ptr(b.ctypes.data, x.ctypes.data, cfg, hist.ctypes.data, N.HOST, exact=exact)
    finally:
        if residual_vectors is not None:
            check(lib.hfpg_set_residual_callback(dev.h, None, None))
    if x_out is not None:
        x_out.append(x)
    return SolveReport(method=getattr(precond, "method", ""), n=int(rep.n),
                       iterations=int(rep.iterations), converged=bool(rep.converged),
                       status=SolveStatus(rep.status),
                       residual_history=hist[: rep.history_len].tolist(),
                       wall_ms=float(rep.wall_ms), breakdown_iter=int(rep.breakdown_iter))


# ------------------------------------------------------------------------------ toy_net.hpp


@dataclass
class ToynetConfig:
    """toy_net.hpp:12-19. The GPU forward implements the production width (d = 128, head dim
    16, i.e. the d128_L3_hw config: layers=3, heads=8)."""
    d: int = 128
    layers: int = 3
    heads: int = 8
    gcn_layers: int = 2
    d_global: int = 12
    edge_hidden: int = 8


@dataclass
class ToynetTrace:
    """toy_net.hpp:64-74."""
    leaf_attention_dispatches: int = 0
    tile_attention_dispatches: int = 0
    max_attention_row_sum_error: float = 0.0
    highway_max_deviation: float = 0.0
    ms: float = 0.0
    timing_only: bool = False  # input: time the forward without the audits

    def attention_kernel_families(self) -> int:
        return int(self.leaf_attention_dispatches > 0) + int(self.tile_attention_dispatches > 0)


def _frame_view(frame: Frame) -> "N.FrameViewC":
    A = frame.A
    v = N.FrameViewC(frame.n, frame.width, frame.height, frame.cell_order.ctypes.data,
                     frame.rho.ctypes.data, float(frame.rho_heavy), A.row_offsets.ctypes.data,
                     A.col_indices.ctypes.data, A.values.ctypes.data)
    v._keep = (frame,)
    return v


def toynet_forward(frame: Frame, partition: HPartition, coarse_size: int,
                   cfg: ToynetConfig | None = None, weight_seed: int = 0,
                   trace: ToynetTrace | None = None, device: Device | None = None,
                   load: bool = False) -> FactorTensor:
    """toy_net.cpp:170 init_weights(cfg, layout, weight_seed) + :322 forward on the GPU
    (tcgen05 tf32 GEMMs). With load=True the tensor also becomes `device`'s factor tensor."""
    cfg = cfg or ToynetConfig()
    if frame.depth != 1:
        raise ValueError("toynet: 2D frames only (frame.hpp)")
    dev = device or Device(0)
    lay = make_factor_layout(partition, coarse_size)
    out = np.empty(lay.total, np.float32)
    c = N.ToynetConfigC(cfg.d, cfg.layers, cfg.heads, cfg.gcn_layers, cfg.d_global, cfg.edge_hidden)
    tr = N.ToynetTraceC()
    tr.timing_only = int(bool(trace is not None and trace.timing_only))
    view = _frame_view(frame)
    check(lib.hfpg_toynet_forward(dev.h, C.byref(view), partition.leaf_size, coarse_size, C.byref(c),
                                  weight_seed, out.ctypes.data, int(load),
                                  C.byref(tr) if trace is not None else None))
    if trace is not None:
        trace.max_attention_row_sum_error = tr.max_attention_row_sum_error
        trace.highway_max_deviation = tr.highway_max_deviation
        trace.leaf_attention_dispatches = tr.leaf_attention_dispatches
        trace.tile_attention_dispatches = tr.tile_attention_dispatches
        trace.ms = tr.ms
    return FactorTensor(lay, out)


def toynet_forward_gpu_frame(frame: "GpuFrame", coarse_size: int, cfg: ToynetConfig | None = None,
                             weight_seed: int = 0, trace: ToynetTrace | None = None,
                             leaf_size: int = 128, load: bool = True,
                             copy_out: bool = False) -> FactorTensor | None:
    """toynet forward from a GPU frame (Device.frame_gpu): inputs never leave the device. With
    load=True the factors become the frame's device's factor tensor (generate -> infer -> solve
    on the GPU); copy_out=True also returns them as a host FactorTensor."""
    cfg = cfg or ToynetConfig()
    if frame.depth != 1:
        raise ValueError("toynet: 2D frames only (frame.hpp)")
    lay = make_factor_layout(build_partition(frame.n, leaf_size), coarse_size)
    out = np.empty(lay.total, np.float32) if copy_out else None
    c = N.ToynetConfigC(cfg.d, cfg.layers, cfg.heads, cfg.gcn_layers, cfg.d_global, cfg.edge_hidden)
    tr = N.ToynetTraceC()
    tr.timing_only = int(bool(trace is not None and trace.timing_only))
    check(lib.hfpg_toynet_forward_gpu_frame(frame.device.h, leaf_size, coarse_size, C.byref(c), weight_seed,
                                            out.ctypes.data if copy_out else None, int(load),
                                            C.byref(tr) if trace is not None else None))
    if trace is not None:
        trace.max_attention_row_sum_error = tr.max_attention_row_sum_error
        trace.highway_max_deviation = tr.highway_max_deviation
        trace.leaf_attention_dispatches = tr.leaf_attention_dispatches
        trace.tile_attention_dispatches = tr.tile_attention_dispatches
        trace.ms = tr.ms
    return FactorTensor(lay, out) if copy_out else None


# -------------------------------------------------------------------------------- apply.hpp


def apply(factors: FactorTensor, a_diag, r, device: Device | None = None) -> np.ndarray:
    """apply.cpp:79-174 apply<float> on the GPU: y = M r."""
    dev = device or Device(0)
    dev.load_factors(factors)
    dev.set_diag(np.asarray(a_diag, np.float64))
    r = np.asarray(r, np.float64)
    if r.shape != (factors.layout.n,):
        raise ValueError("apply: length mismatch")
    return dev.apply(r)


# --------------------------------------------------------------------------- checkpoint.hpp


@dataclass
class Checkpoint:
    factors: FactorTensor
    metadata_json: str


def write_checkpoint(factors: FactorTensor, path: str, metadata_json: str = "{}") -> None:
    """checkpoint.cpp:17-43 (HFTC v1)."""
    L = factors.layout
    check(lib.hfpg_write_checkpoint(str(path).encode(), L.n, L.leaf_size, L.coarse_size,
                                    factors.data.ctypes.data, int(factors.spd_shift_enabled),
                                    float(factors.spd_shift_raw), metadata_json.encode()))


def read_checkpoint(path: str) -> Checkpoint:
    """checkpoint.cpp:45-85 (magic, version, packed width and crc32 validated)."""
    lay = N.Layout()
    check(lib.hfpg_read_checkpoint(str(path).encode(), C.byref(lay), None, None, None, None, 0))
    data = np.empty(lay.total, np.float32)
    en, raw = N.i32(), N.dbl()
    meta = C.create_string_buffer(1 << 16)
    check(lib.hfpg_read_checkpoint(str(path).encode(), C.byref(lay), data.ctypes.data,
                                   C.byref(en), C.byref(raw), meta, len(meta)))
    p = build_partition(lay.n, lay.leaf_size)
    f = FactorTensor(make_factor_layout(p, lay.coarse_size), data)
    f.spd_shift_enabled, f.spd_shift_raw = bool(en.value), float(raw.value)
    return Checkpoint(f, meta.value.decode())
