"""GPU frame generator (framegen.cuh) against the host generator (frame.cpp:161-181 and the 3D
analogue), through the C ABI.

* Under HFPG_FRAME_CRMATH=1 the host generator draws its normals with correctly rounded log/cos,
  which is what the device computes: every array (Morton order, CSR, values, rho, b) must then be
  bit-identical.
* Against the default host build (glibc libm, bit-identical to the reference — test_host.py),
  Morton order and CSR structure are bit-identical; rho and b differ by at most 2 ulp (values
  by a few, a diagonal summing perturbed weights) on the ~0.16% of normals glibc rounds
  incorrectly (tools/crmath_check.cpp).
* The generated frame is loaded as the handle's system: solving it from the device rhs gives
  the iterations and the bitwise x of loading the CR host frame through hfpg_load_csr."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES_2D = [4, 1000, 4096, 65536, 100003, 1 << 20]
CASES_3D = [(2, 2, 2), (16, 16, 16), (33, 20, 7), (64, 64, 64)]


def host_frame(H, spec, seed, fidx, crmath):
    old = os.environ.get("HFPG_FRAME_CRMATH")
    os.environ["HFPG_FRAME_CRMATH"] = "1" if crmath else "0"
    try:
        if isinstance(spec, tuple):
            return H.make_frame_3d(*spec, seed, fidx)
        return H.make_frame(spec, seed, fidx)
    finally:
        if old is None:
            del os.environ["HFPG_FRAME_CRMATH"]
        else:
            os.environ["HFPG_FRAME_CRMATH"] = old


def gpu_frame(dev, spec, seed, fidx):
    if isinstance(spec, tuple):
        return dev.frame_gpu_3d(*spec, seed, fidx)
    return dev.frame_gpu(spec, seed, fidx)


def arrays(f):
    return {"cell_order": f.cell_order, "rho": f.rho, "row_offsets": f.A.row_offsets,
            "col_indices": f.A.col_indices, "values": f.A.values, "b": f.b}


@pytest.mark.parametrize("spec", CASES_2D + CASES_3D, ids=str)
def test_bit_identical_to_crmath_host(H, oracle, spec):
    dev = H.Device(0)
    for seed, fidx in [(0, 1), (2024, (3 << 24) | 17)]:
        g = gpu_frame(dev, spec, seed, fidx)
        h = host_frame(H, spec, seed, fidx, True)
        assert (g.n, g.width, g.height, g.depth) == (h.n, h.width, h.height, h.depth)
        assert g.rho_heavy == h.rho_heavy
        got = arrays(g.to_host())
        # |A|_F from the sequential fused sum of squares (csr.cpp:64-68), bit for bit
        assert g.frobenius == np.sqrt(oracle.seq_sum(h.A.values, True))
        for k, want in arrays(h).items():
            assert got[k].dtype == want.dtype and got[k].shape == want.shape, k
            bad = np.flatnonzero(got[k] != want)
            assert bad.size == 0, f"{k}: {bad.size} mismatches, first at {bad[:5]}"


@pytest.mark.parametrize("spec", [65536, 1 << 20, (64, 64, 64)], ids=str)
def test_against_glibc_host(H, spec):
    dev = H.Device(0)
    g = gpu_frame(dev, spec, 7, 5).to_host()
    h = host_frame(H, spec, 7, 5, False)
    for k in ("cell_order", "row_offsets", "col_indices"):
        assert (arrays(g)[k] == arrays(h)[k]).all(), k
    for k in ("rho", "values", "b"):
        a, b = arrays(g)[k], arrays(h)[k]
        diff = a != b
        assert diff.mean() < 0.01, (k, diff.mean())
        # one-ulp normals -> rho within 2 ulp; a diagonal sums up to six perturbed weights
        tol = {"rho": 4.5e-16, "values": 2e-15, "b": 4.5e-16}[k]
        scale = np.maximum(np.abs(b), 1.0 if k == "b" else 0.0)
        assert (np.abs(a - b) <= tol * scale).all(), (k, np.abs(a - b).max())


@pytest.mark.parametrize("spec", [65536, (32, 32, 32)], ids=str)
def test_solve_matches_host_loaded_system(H, spec):
    import torch
    from paper_2605_13343_b200 import _native as N
    h = host_frame(H, spec, 11, 2, True)
    n = h.n
    f = H.init_factors(H.build_partition(n, 128), 32, H.FactorInit.jacobi_seed, 1e-2,
                       H.RngStream(11, 2, H.RngPurpose.factor_init))
    cfg = H.SolveConfig()
    d1 = H.Device(0)
    d1.load_csr(h.A)
    d1.load_factors(f)
    d1.set_precond(2)
    x1 = np.empty(n)
    r1 = d1.solve_ptr(h.b.ctypes.data, x1.ctypes.data, cfg, None, N.HOST)

    d2 = H.Device(0)
    d2.load_factors(f)
    d2.set_precond(2)
    g = gpu_frame(d2, spec, 11, 2)
    x2 = torch.empty(n, dtype=torch.float64, device="cuda")
    r2 = d2.solve_ptr(g.b, x2.data_ptr(), cfg, None, N.DEVICE)
    assert r1.converged and r2.converged
    assert int(r1.iterations) == int(r2.iterations)
    assert (x2.cpu().numpy() == x1).all()


def test_regenerate_on_one_handle(H):
    """Frames of changing size/index on one handle: buffers regrow, the solve graph follows."""
    import torch
    from paper_2605_13343_b200 import _native as N
    dev = H.Device(0)
    for n, fidx in [(65536, 0), (4096, 1), (65536, 2), (1 << 18, 3), (65536, 0)]:
        g = dev.frame_gpu(n, 3, fidx)
        dev.set_precond(1)  # Jacobi: no factors needed
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        rep = dev.solve_ptr(g.b, x.data_ptr(), H.SolveConfig(), None, N.DEVICE)
        h = host_frame(H, n, 3, fidx, True)
        ref = H.pcg_solve(h.A, h.b, H.jacobi_applier(h.A))
        assert rep.converged and int(rep.iterations) == int(ref.iterations)
        assert g.generate_ms > 0.0


def test_errors(H):
    dev = H.Device(0)
    with pytest.raises(ValueError):
        dev.frame_gpu(3, 0, 0)
    with pytest.raises(ValueError):
        dev.frame_gpu_3d(1, 4, 4, 0, 0)
    from paper_2605_13343_b200 import _native as N
    with pytest.raises(ValueError):
        N.check(N.lib.hfpg_frame_gpu_view(H.Device(0).h, None))


def _seq_inputs():
    g = np.random.default_rng(42)
    yield "normals", g.standard_normal(1 << 20), False
    yield "normals_odd_len", g.standard_normal((1 << 16) + 4097), False
    yield "drift", g.standard_normal(300000) + 0.01, False
    yield "halves_ties", g.integers(-50, 50, 200000) / 2.0, False
    yield "mixed_scales", g.standard_normal(100000) * 10.0 ** g.integers(-12, 12, 100000), False
    yield "cancel", np.repeat([1e16, 1.0, -1e16], 20000), False
    yield "zeros_tiny", np.where(g.random(50000) < 0.5, 0.0, 1e-310), False
    yield "overflow", np.full(10000, 1e305), False
    yield "weights_sq", g.random(5 << 20) * 200.0 + 0.1, True
    yield "ints_sq_ties", g.integers(1, 64, 300000).astype(np.float64) * 2.0 ** -20, True
    yield "mixed_sq", g.standard_normal(200000) * 10.0 ** g.integers(-6, 6, 200000), True
    for n in (0, 1, 5, 4095, 4096, 4097, 8193):
        yield f"len{n}", g.standard_normal(n), False
        yield f"len{n}_sq", g.standard_normal(n), True


@pytest.mark.parametrize("mode", ["summaries", "HFPG_FG_NOSUMM", "HFPG_FG_SERIAL"])
@pytest.mark.parametrize("name,x,squares", list(_seq_inputs()), ids=lambda v: v if isinstance(v, str) else "")
def test_seq_sum_bit_identical_to_serial(H, oracle, name, x, squares, mode):
    """hfpg_seq_sum (the generator's exact parallel emulation of a sequential sum: tile summaries
    + detailed scans; detailed scans only; the literal loop) equals the one-thread loop bit for
    bit — including ties, binade crossings, sign changes and overflow."""
    import ctypes as C
    from paper_2605_13343_b200 import _native as N
    dev = H.Device(0)
    x = np.ascontiguousarray(x, np.float64)
    out = C.c_double()
    if mode != "summaries":
        os.environ[mode] = "1"
    try:
        N.check(N.lib.hfpg_seq_sum(dev.h, x.ctypes.data, len(x), int(squares), N.HOST, C.byref(out)))
    finally:
        os.environ.pop(mode, None)
    want = oracle.seq_sum(x, squares)
    assert np.array_equal(np.float64(out.value), np.float64(want), equal_nan=True), (out.value, want)


@pytest.mark.parametrize("n", [1024, 4096, 65536])
def test_toynet_from_gpu_frame_matches_host_path(H, n):
    """toynet_forward_gpu_frame (inputs on the device, global statistics reduced there) equals
    the host-frame forward (tests/test_gpu_toynet.py pins that one to the reference) on the same
    frame: the CR-math host frame is bit-identical to the GPU frame, so only the order of the
    f64 statistic sums differs before their rounding to f32 features."""
    from conftest import rel_l2
    dev = H.Device(0)
    g = dev.frame_gpu(n, 2024, 0)
    h = host_frame(H, n, 2024, 0, True)
    p = H.build_partition(n, 128)
    want = H.toynet_forward(h, p, 32, weight_seed=0)
    tr = H.ToynetTrace()
    got = H.toynet_forward_gpu_frame(g, 32, weight_seed=0, trace=tr, load=False, copy_out=True)
    assert got.data.shape == want.data.shape
    assert np.isfinite(got.data).all()
    assert rel_l2(got.data.astype(np.float64), want.data.astype(np.float64)) <= 1e-5
    assert tr.attention_kernel_families() == 2 and tr.max_attention_row_sum_error <= 1e-5


def test_generate_infer_solve_on_device(H):
    """frame -> toynet factors -> PCG without a host round trip (the handle owns all three);
    the seeded-weight tensor is the reference's non-convergent preconditioner (SURVEY.md §0
    fact 2), so the pipeline must report max_iters exactly as the host-input path does."""
    import torch
    from paper_2605_13343_b200 import _native as N
    n = 8192
    dev = H.Device(0)
    g = dev.frame_gpu(n, 2024, 0)
    H.toynet_forward_gpu_frame(g, 32, load=True)
    dev.set_precond(2)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    rep = dev.solve_ptr(g.b, x.data_ptr(), H.SolveConfig(max_iters=2000), None, N.DEVICE)
    assert rep.status == 1 and rep.iterations == 2000
    # and with init_factors instead of the network: converges like the host-loaded system
    f = H.init_factors(H.build_partition(n, 128), 32, H.FactorInit.jacobi_seed, 1e-2,
                       H.RngStream(2024, 0, H.RngPurpose.factor_init))
    dev.load_factors(f)
    rep = dev.solve_ptr(g.b, x.data_ptr(), H.SolveConfig(), None, N.DEVICE)
    assert rep.converged
