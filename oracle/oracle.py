"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracle.

Two checkers live here:

* ``Oracle``  — the plain-C restatement (``oracle/hfp_oracle.c`` -> ``oracle/liboracle.so``);
* ``Ref``     — the UNMODIFIED reference library compiled from ``/root/reference/proj/src``
  (``oracle/_ref/libhfpref.so``, via ``oracle/Makefile``) behind a pointer-only shim.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhfpref.so")
REF_SRC = "/root/reference/proj/src/apply.cpp"

_u64 = C.c_uint64
_p = C.c_void_p


def build() -> None:
    """Build the checkers (the reference .so only where /root/reference is mounted)."""
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_p)


def _check(rc: int, lib, what: str) -> None:
    if rc != 0:
        msg = lib.ref_last_error().decode() if hasattr(lib, "ref_last_error") else ""
        raise ValueError(f"{what} failed ({rc}) {msg}")


class _Base:
    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)

    # -- shared signatures (same names modulo prefix) -----------------------------------
    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def packed_width(self, n: int, leaf: int, ls: int) -> int:
        out = _u64()
        _check(self._f("packed_width")(_u64(n), _u64(leaf), _u64(ls), C.byref(out)), self.lib,
               "packed_width")
        return out.value

    def partition(self, n: int, leaf: int) -> np.ndarray:
        k = n // leaf
        out = np.zeros((max(k - 1, 0), 5), np.uint64)
        _check(self._f("partition")(_u64(n), _u64(leaf), _ptr(out)), self.lib, "partition")
        return out

    def init_factors(self, n, leaf, ls, sigma, seed, frame) -> np.ndarray:
        out = np.empty(self.packed_width(n, leaf, ls), np.float32)
        f = self._f("init_factors_f32")
        f.argtypes = [_u64, _u64, _u64, C.c_double, _u64, _u64, _p]
        _check(f(n, leaf, ls, sigma, seed, frame, _ptr(out)), self.lib, "init_factors")
        return out

    def spmv(self, csr, x: np.ndarray) -> np.ndarray:
        ro, ci, v = csr
        n = len(ro) - 1
        y = np.empty(n, np.float64)
        self._f("spmv")(_u64(n), _ptr(ro), _ptr(ci), _ptr(v), _ptr(x), _ptr(y))
        return y

    def apply_f32(self, n, leaf, ls, packed, a_diag, r, spd_enabled=0, spd_raw=0.0):
        y = np.empty(n, np.float64)
        f = self._f("apply_f32")
        f.argtypes = [_u64, _u64, _u64, _p, C.c_int, C.c_double, _p, _p, _p]
        _check(f(n, leaf, ls, _ptr(np.ascontiguousarray(packed, np.float32)), spd_enabled,
                 spd_raw, _ptr(a_diag), _ptr(r), _ptr(y)), self.lib, "apply_f32")
        return y

    def pcg_solve(self, csr, b, kind: int, leaf=0, ls=0, packed=None, rtol=1e-8,
                  max_iters=20000, spd_enabled=0, spd_raw=0.0):
        """kind: 0 identity, 1 jacobi, 2 factor, 3 ic0 (Ref only). Returns (report dict, x, history)."""
        ro, ci, v = csr
        n = len(ro) - 1
        x = np.empty(n, np.float64)
        hist = np.empty(max(max_iters, 1), np.float64)
        rep = np.zeros(6, np.float64)
        f = self._f("pcg_solve")
        f.argtypes = [_u64, _p, _p, _p, _p, C.c_int, _u64, _u64, _p, C.c_int, C.c_double,
                      C.c_double, _u64, _p, _p, _p]
        _check(f(n, _ptr(ro), _ptr(ci), _ptr(v), _ptr(b), kind, leaf, ls,
                 _ptr(packed) if packed is not None else None, spd_enabled, spd_raw, rtol,
                 max_iters, _ptr(x), _ptr(hist), _ptr(rep)), self.lib, "pcg_solve")
        status = {0: "converged", 1: "max_iters", 2: "breakdown"}[int(rep[2])]
        report = dict(iterations=int(rep[0]), converged=bool(rep[1]), status=status,
                      breakdown_iter=int(rep[3]), wall_ms=float(rep[5]))
        return report, x, hist[: int(rep[4])].copy()


class Oracle(_Base):
    """The C restatement (oracle/hfp_oracle.c)."""

    prefix = "orc_"

    def __init__(self):
        super().__init__(ORACLE_SO)
        self.lib.orc_apply_f64.argtypes = [_u64, _u64, _u64, _p, C.c_int, C.c_double, _p, _p,
                                           _p]

    def apply_f64(self, n, leaf, ls, packed64, a_diag, r, spd_enabled=0, spd_raw=0.0):
        y = np.empty(n, np.float64)
        _check(self.lib.orc_apply_f64(n, leaf, ls, _ptr(np.ascontiguousarray(packed64,
                                                                             np.float64)),
                                      spd_enabled, spd_raw, _ptr(a_diag), _ptr(r), _ptr(y)),
               self.lib, "apply_f64")
        return y

    def seq_sum(self, x, squares: bool) -> float:
        x = np.ascontiguousarray(x, np.float64)
        self.lib.orc_seq_sum.restype = C.c_double
        self.lib.orc_seq_sum.argtypes = [_p, _u64, C.c_int]
        return float(self.lib.orc_seq_sum(_ptr(x), len(x), int(squares)))

    def rng(self, seed, frame, purpose, count):
        class S(C.Structure):
            _fields_ = [("key", _u64), ("counter", _u64)]

        s = S()
        self.lib.orc_rng_init(C.byref(s), _u64(seed), _u64(frame), _u64(purpose))
        self.lib.orc_rng_bits.restype = _u64
        self.lib.orc_rng_normal.restype = C.c_double
        bits = np.array([self.lib.orc_rng_bits(C.byref(s)) for _ in range(count)], np.uint64)
        self.lib.orc_rng_init(C.byref(s), _u64(seed), _u64(frame), _u64(purpose))
        normals = np.array([self.lib.orc_rng_normal(C.byref(s)) for _ in range(count)])
        return bits, normals


class Ref(_Base):
    """The reference itself, compiled from /root/reference by oracle/Makefile."""

    prefix = "ref_"

    def apply_batch_adjoint(self, n, packed64, a_diag, x, kz, bar_y=None, spd_enabled=0, spd_raw=0.0):
        """adjoint.cpp:44 factor_apply_batch (+ :129 adjoint when bar_y is given) -> (y, grad)."""
        y = np.empty(n * kz)
        grad = np.empty(len(packed64))
        f = self._f("apply_batch_adjoint")
        f.argtypes = [_u64, _u64, _u64, _p, C.c_int, C.c_double, _p, _p, _u64, _p, _p, _p]
        _check(f(n, 128, 32, _ptr(np.ascontiguousarray(packed64, np.float64)), spd_enabled, spd_raw,
                 _ptr(np.ascontiguousarray(a_diag, np.float64)), _ptr(np.ascontiguousarray(x, np.float64)), kz,
                 _ptr(np.ascontiguousarray(bar_y, np.float64)) if bar_y is not None else None, _ptr(y),
                 _ptr(grad)), self.lib, "apply_batch_adjoint")
        return y, (grad if bar_y is not None else None)

    def loss_gradient(self, csr, packed64, z, kz, kind, norm_a=1.0):
        """adjoint.cpp:250 loss_gradient -> (loss, degenerate, grad)."""
        ro, ci, v = csr
        n = len(ro) - 1
        grad = np.empty(len(packed64))
        loss = C.c_double()
        deg = C.c_int()
        f = self._f("loss_gradient")
        f.argtypes = [_u64, _p, _p, _p, _u64, _u64, _p, _p, _u64, C.c_int, C.c_double, _p, _p, _p]
        _check(f(n, _ptr(ro), _ptr(ci), _ptr(v), 128, 32, _ptr(np.ascontiguousarray(packed64, np.float64)),
                 _ptr(np.ascontiguousarray(z, np.float64)), kz, kind, norm_a, C.byref(loss), C.byref(deg),
                 _ptr(grad)), self.lib, "loss_gradient")
        return loss.value, bool(deg.value), grad

    def ic0_factorize(self, csr, policy=1):
        """ic0.cpp:10 -> (lro u64[n+1], lci u32[nnz], lv f64[nnz], shift)."""
        ro, ci, v = csr
        n = len(ro) - 1
        cap = int(ro[-1]) + n
        lro = np.empty(n + 1, np.uint64)
        lci = np.empty(cap, np.uint32)
        lv = np.empty(cap, np.float64)
        nnz = C.c_uint64()
        shift = C.c_double()
        f = self._f("ic0_factorize")
        f.argtypes = [_u64, _p, _p, _p, C.c_int, _p, _p, _p, _u64, _p, _p]
        _check(f(n, _ptr(ro), _ptr(ci), _ptr(v), policy, _ptr(lro), _ptr(lci), _ptr(lv), cap,
                 C.byref(nnz), C.byref(shift)), self.lib, "ic0_factorize")
        return lro, lci[: nnz.value].copy(), lv[: nnz.value].copy(), shift.value

    def ic0_apply(self, csr, r, policy=1):
        """ic0_applier(ic0_factorize(A)) on r (ic0.cpp:72-99)."""
        ro, ci, v = csr
        n = len(ro) - 1
        z = np.empty(n, np.float64)
        f = self._f("ic0_apply")
        f.argtypes = [_u64, _p, _p, _p, C.c_int, _p, _p]
        _check(f(n, _ptr(ro), _ptr(ci), _ptr(v), policy, _ptr(np.ascontiguousarray(r, np.float64)),
                 _ptr(z)), self.lib, "ic0_apply")
        return z

    def __init__(self):
        super().__init__(REF_SO)
        self.lib.ref_last_error.restype = C.c_char_p
        self.lib.ref_frame_create.restype = _p
        self.lib.ref_frame_create.argtypes = [_u64, _u64, _u64]
        self.lib.ref_morton_encode.restype = C.c_uint32
        self.lib.ref_morton_encode.argtypes = [C.c_uint32, C.c_uint32]

    def make_frame(self, n: int, seed: int, frame_index: int) -> dict:
        """frame.cpp:161 make_frame -> dict of numpy arrays."""
        h = self.lib.ref_frame_create(n, seed, frame_index)
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        return self._frame_dict(h)

    def make_frame_3d(self, nx: int, ny: int, nz: int, seed: int, frame_index: int) -> dict:
        """The 3D benchmark frame built from the reference's RngStream / sample_rhs / stencil
        rules (oracle/frame3d_ref.cpp) -> dict of numpy arrays."""
        L = self.lib
        L.ref_frame3d_create.restype = _p
        L.ref_frame3d_create.argtypes = [_u64] * 5
        L.ref_frame3d_last_error.restype = C.c_char_p
        h = L.ref_frame3d_create(nx, ny, nz, seed, frame_index)
        if not h:
            raise ValueError(L.ref_frame3d_last_error().decode())
        nn, nnz, rh = _u64(), _u64(), C.c_double()
        L.ref_frame3d_sizes(_p(h), C.byref(nn), C.byref(nnz), C.byref(rh))
        fr = dict(n=nn.value, width=nx, height=ny, depth=nz, rho_heavy=rh.value,
                  cell_order=np.empty(nn.value, np.uint32), rho=np.empty(nn.value),
                  row_offsets=np.empty(nn.value + 1, np.uint64),
                  col_indices=np.empty(nnz.value, np.uint32), values=np.empty(nnz.value),
                  b=np.empty(nn.value))
        L.ref_frame3d_fill(_p(h), _ptr(fr["cell_order"]), _ptr(fr["rho"]), _ptr(fr["row_offsets"]),
                           _ptr(fr["col_indices"]), _ptr(fr["values"]), _ptr(fr["b"]))
        L.ref_frame3d_free(_p(h))
        return fr

    def write_mppf(self, n: int, seed: int, frame_index: int, path: str) -> None:
        """mppf.cpp:48 write_mppf(make_frame(n, seed, frame_index), path)."""
        f = self._f("write_mppf")
        f.argtypes = [_u64, _u64, _u64, C.c_char_p]
        _check(f(n, seed, frame_index, path.encode()), self.lib, "write_mppf")

    def read_mppf(self, path: str) -> dict:
        """mppf.cpp:102 read_mppf -> dict of numpy arrays (+ seeds, barriers)."""
        self.lib.ref_read_mppf.restype = _p
        self.lib.ref_read_mppf.argtypes = [C.c_char_p]
        h = self.lib.ref_read_mppf(path.encode())
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        seed, fidx, nb = _u64(), _u64(), C.c_uint32()
        bars = np.zeros(12)
        self.lib.ref_frame_meta(_p(h), C.byref(seed), C.byref(fidx), C.byref(nb), _ptr(bars))
        fr = self._frame_dict(h)
        fr.update(master_seed=seed.value, frame_index=fidx.value,
                  barriers=[tuple(bars[4 * i:4 * i + 4]) for i in range(nb.value)])
        return fr

    def _frame_dict(self, h) -> dict:
        nn, nnz, w, hh = _u64(), _u64(), _u64(), _u64()
        rh = C.c_double()
        self.lib.ref_frame_sizes(_p(h), C.byref(nn), C.byref(nnz), C.byref(w), C.byref(hh),
                                 C.byref(rh))
        fr = dict(n=nn.value, width=w.value, height=hh.value, rho_heavy=rh.value,
                  cell_order=np.empty(nn.value, np.uint32), rho=np.empty(nn.value),
                  row_offsets=np.empty(nn.value + 1, np.uint64),
                  col_indices=np.empty(nnz.value, np.uint32), values=np.empty(nnz.value),
                  b=np.empty(nn.value))
        self.lib.ref_frame_fill(_p(h), _ptr(fr["cell_order"]), _ptr(fr["rho"]),
                                _ptr(fr["row_offsets"]), _ptr(fr["col_indices"]),
                                _ptr(fr["values"]), _ptr(fr["b"]))
        self.lib.ref_frame_free(_p(h))
        return fr

    def rng(self, seed, frame, purpose, count):
        bits = np.empty(count, np.uint64)
        normals = np.empty(count)
        self.lib.ref_rng_draws(_u64(seed), _u64(frame), _u64(purpose), _u64(count), _ptr(bits),
                               _ptr(normals))
        return bits, normals

    def apply_f64_of_f32(self, n, leaf, ls, packed, a_diag, r, spd_enabled=0, spd_raw=0.0):
        y = np.empty(n, np.float64)
        f = self.lib.ref_apply_f64_of_f32
        f.argtypes = [_u64, _u64, _u64, _p, C.c_int, C.c_double, _p, _p, _p]
        _check(f(n, leaf, ls, _ptr(packed), spd_enabled, spd_raw, _ptr(a_diag), _ptr(r),
                 _ptr(y)), self.lib, "apply_f64")
        return y

    def assemble_dense(self, n, leaf, ls, packed, a_diag, spd_enabled=0, spd_raw=0.0):
        out = np.empty((n, n), np.float64)
        f = self.lib.ref_assemble_dense_f32
        f.argtypes = [_u64, _u64, _u64, _p, C.c_int, C.c_double, _p, _p]
        _check(f(n, leaf, ls, _ptr(packed), spd_enabled, spd_raw, _ptr(a_diag), _ptr(out)),
               self.lib, "assemble_dense")
        return out

    def time_apply_f32(self, n, leaf, ls, packed, a_diag, r, reps):
        ms = C.c_double()
        f = self.lib.ref_time_apply_f32
        f.argtypes = [_u64, _u64, _u64, _p, _p, _p, _u64, _p]
        _check(f(n, leaf, ls, _ptr(packed), _ptr(a_diag), _ptr(r), reps, C.byref(ms)),
               self.lib, "time_apply")
        return ms.value

    def pcg_time_iters(self, csr, b, leaf, ls, packed, iters):
        ro, ci, v = csr
        ms = C.c_double()
        f = self.lib.ref_pcg_time_iters
        f.argtypes = [_u64, _p, _p, _p, _p, _u64, _u64, _p, _u64, _p]
        _check(f(len(ro) - 1, _ptr(ro), _ptr(ci), _ptr(v), _ptr(b), leaf, ls, _ptr(packed),
                 iters, C.byref(ms)), self.lib, "pcg_time_iters")
        return ms.value

    def write_checkpoint(self, path, n, leaf, ls, packed, spd_enabled=0, spd_raw=0.0,
                         metadata="{}"):
        f = self.lib.ref_write_checkpoint
        f.argtypes = [C.c_char_p, _u64, _u64, _u64, _p, C.c_int, C.c_double, C.c_char_p]
        _check(f(path.encode(), n, leaf, ls, _ptr(packed), spd_enabled, spd_raw,
                 metadata.encode()), self.lib, "write_checkpoint")

    def read_checkpoint(self, path):
        n, leaf, ls, tot = _u64(), _u64(), _u64(), _u64()
        f = self.lib.ref_read_checkpoint
        f.argtypes = [C.c_char_p, _p, _p, _p, _p, _p]
        _check(f(path.encode(), C.byref(n), C.byref(leaf), C.byref(ls), C.byref(tot), None),
               self.lib, "read_checkpoint")
        out = np.empty(tot.value, np.float32)
        _check(f(path.encode(), C.byref(n), C.byref(leaf), C.byref(ls), C.byref(tot),
                 _ptr(out)), self.lib, "read_checkpoint")
        return dict(n=n.value, leaf=leaf.value, ls=ls.value), out

    def train_factors(self, n, frame_seed, frame_indices, eval_index, cfg_c, seed, log_cap=4096):
        """train.cpp:29 train_factors on make_frame(n, frame_seed, i) frames; cfg_c is the
        product's TrainConfigC (same C layout). Returns (factors, [log dicts], summary dict)."""
        from paper_2605_13343_b200 import _native as PN  # struct layouts only
        idx = np.asarray(frame_indices, np.uint64)
        summ = PN.TrainSummaryC()
        logs = (PN.TrainLogC * log_cap)()
        width = self.packed_width(n, n // 2 if n < 2 * cfg_c.leaf_size else cfg_c.leaf_size, cfg_c.coarse_size)
        out = np.empty(width, np.float32)
        f = self.lib.ref_train_factors
        f.argtypes = [_u64, _u64, _p, _u64, _u64, _p, _u64, _p, _p, _u64, _p]
        _check(f(n, frame_seed, _ptr(idx), len(idx), eval_index, C.byref(cfg_c), seed, _ptr(out), logs, log_cap,
                 C.byref(summ)), self.lib, "train_factors")
        ents = [dict(step=e.step, train_loss=e.train_loss, sai_heldout=e.sai_heldout,
                     pcg_iters_heldout=e.pcg_iters_heldout, lr=e.lr) for e in logs[: summ.n_entries]]
        return out, ents, dict(total_steps=summ.total_steps, auto_stopped=summ.auto_stopped,
                               aborted_divergence=summ.aborted_divergence, reached_target=summ.reached_target)

    def toynet_forward(self, n, seed, frame_index, leaf=128, ls=32, d=128, layers=3, heads=8,
                       gcn_layers=2, d_global=12, edge_hidden=8, weight_seed=0):
        out = np.empty(self.packed_width(n, leaf, ls), np.float32)
        trace = np.zeros(4)
        ms = C.c_double()
        f = self.lib.ref_toynet_forward
        f.argtypes = [_u64] * 12 + [_p, _p, _p]
        _check(f(n, seed, frame_index, leaf, ls, d, layers, heads, gcn_layers, d_global,
                 edge_hidden, weight_seed, _ptr(out), _ptr(trace), C.byref(ms)), self.lib,
               "toynet_forward")
        return out, trace, ms.value


def ref_available() -> bool:
    return os.path.exists(REF_SO)
