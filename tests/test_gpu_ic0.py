"""GPU IC(0) preconditioner (ic0.cpp:72-99) through the C ABI: the two sync-free triangular
sweeps are bit-identical to the reference's ic0_applier, and IC(0)-PCG (the whole loop in the
CUDA graph) matches the reference's iteration count within +-2 (only the f64 dot-product
summation order differs)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def csr_of(A):
    return (np.ascontiguousarray(A.row_offsets, np.uint64), np.ascontiguousarray(A.col_indices, np.uint32),
            np.ascontiguousarray(A.values, np.float64))


FRAMES = {
    "2d_8192": lambda H: H.make_frame(8192, 2024, 0),
    "3d_16": lambda H: H.make_frame_3d(16, 16, 16, 2024, 1),
    "3d_40x24x20": lambda H: H.make_frame_3d(40, 24, 20, 2024, 2),
}


@pytest.mark.parametrize("name", list(FRAMES))
def test_apply_bit_exact(H, ref, name):
    fr = FRAMES[name](H)
    f = H.ic0_factorize(fr.A)
    ap = H.ic0_applier(f)
    ap.bind(fr.A)
    rng = np.random.default_rng(7)
    for r in (fr.b, rng.standard_normal(fr.n)):
        z = ap(r)
        want = ref.ic0_apply(csr_of(fr.A), r, 1)
        assert np.array_equal(z.view(np.uint64), want.view(np.uint64))
    # repeated applies (epoch flags, no reset) stay identical
    z1, z2 = ap(fr.b), ap(fr.b)
    assert np.array_equal(z1, z2)


@pytest.mark.parametrize("name", ["2d_8192", "3d_40x24x20"])
def test_pcg_iterations(H, ref, name):
    fr = FRAMES[name](H)
    xs = []
    rep = H.pcg_solve(fr.A, fr.b, H.ic0_applier(H.ic0_factorize(fr.A)), H.SolveConfig(), xs)
    want, xr, hist = ref.pcg_solve(csr_of(fr.A), fr.b, 3)
    assert rep.converged and want["converged"]
    assert abs(rep.iterations - want["iterations"]) <= 2, (rep.iterations, want["iterations"])
    k = min(len(hist), len(rep.residual_history)) // 2
    np.testing.assert_allclose(rep.residual_history[:k], hist[:k], rtol=1e-6)
    r = fr.b - fr.A_dense_matvec(xs[0]) if hasattr(fr, "A_dense_matvec") else None
    assert np.linalg.norm(xs[0] - xr) <= 1e-6 * np.linalg.norm(xr)


def test_ic0_beats_jacobi_on_3d(H):
    fr = FRAMES["3d_40x24x20"](H)
    ic = H.pcg_solve(fr.A, fr.b, H.ic0_applier(H.ic0_factorize(fr.A)))
    jac = H.pcg_solve(fr.A, fr.b, H.jacobi_applier(fr.A))
    assert ic.converged and jac.converged and ic.iterations < jac.iterations
