"""hfpg_pcg_solve_exact (pcg_exact.cuh): the whole PCG bit-identical to the reference's pcg_solve
(oracle/_ref, the reference compiled from its sources) — x, the residual history, the iteration
count and the status — for the preconditioners whose apply is itself bit-identical to the
reference's (identity, Jacobi, IC(0)), on 2D and 3D frames, plus the status paths (max_iters, zero
rhs, breakdown) and vector lengths with a remainder after the reference's 4-wide dot body. The
factor apply is not bit-identical by design (exact f32 products summed in f64 against the
reference's f32 arithmetic, <=1e-9 relative): with exact dots its solve stays within the
iteration band."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KINDS = {"identity": 0, "jacobi": 1, "factor": 2, "ic0": 3}


def csr_of(A):
    return (np.ascontiguousarray(A.row_offsets, np.uint64), np.ascontiguousarray(A.col_indices, np.uint32),
            np.ascontiguousarray(A.values, np.float64))


def frame(H, case):
    if case == "2d_1024":
        return H.make_frame(1024, 7, 3)
    if case == "2d_8192":
        return H.make_frame(8192, 2024, 0)
    return H.make_frame_3d(16, 16, 16, 2024, 0)


def applier(H, fr, kind):
    if kind == "identity":
        return H.identity_applier(), None
    if kind == "jacobi":
        return H.jacobi_applier(fr.A), None
    if kind == "ic0":
        return H.ic0_applier(H.ic0_factorize(fr.A)), None
    f = H.init_factors(H.build_partition(fr.n, 128), 32, H.FactorInit.jacobi_seed, 1e-2,
                       H.RngStream(2024, fr.frame_index, H.RngPurpose.factor_init))
    return H.factor_applier(f, fr.A), f.data


def same(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("case", ["2d_1024", "2d_8192", "3d_16"])
@pytest.mark.parametrize("kind", ["identity", "jacobi", "ic0"])
def test_exact_pcg_is_the_reference(H, ref, case, kind):
    fr = frame(H, case)
    ap, packed = applier(H, fr, kind)
    cfg = H.SolveConfig(max_iters=3000)
    xs = []
    rep = H.pcg_solve(fr.A, fr.b, ap, cfg, xs, exact=True)
    want, xr, hist = ref.pcg_solve(csr_of(fr.A), fr.b, KINDS[kind], 128, 32, packed, max_iters=3000)
    assert rep.iterations == want["iterations"] and rep.status.name == want["status"], (rep.iterations, want)
    assert rep.converged == want["converged"]
    assert same(rep.residual_history, hist)
    assert same(xs[0], xr)


@pytest.mark.parametrize("case", ["2d_1024", "2d_8192", "3d_16"])
def test_exact_pcg_factor_band(H, ref, case):
    fr = frame(H, case)
    ap, packed = applier(H, fr, "factor")
    rep = H.pcg_solve(fr.A, fr.b, ap, H.SolveConfig(max_iters=3000), exact=True)
    want, xr, hist = ref.pcg_solve(csr_of(fr.A), fr.b, 2, 128, 32, packed, max_iters=3000)
    assert rep.converged and want["converged"] and abs(rep.iterations - want["iterations"]) <= 2
    m = min(len(hist), len(rep.residual_history), 50)
    np.testing.assert_allclose(rep.residual_history[:m], hist[:m], rtol=1e-4)


def test_exact_status_paths(H, ref):
    fr = H.make_frame(1024, 7, 3)
    ap, packed = applier(H, fr, "jacobi")
    rep = H.pcg_solve(fr.A, fr.b, ap, H.SolveConfig(max_iters=5), exact=True)
    want, _, hist = ref.pcg_solve(csr_of(fr.A), fr.b, 1, max_iters=5)
    assert rep.status.name == want["status"] == "max_iters" and rep.iterations == 5
    assert same(rep.residual_history, hist)
    rep = H.pcg_solve(fr.A, np.zeros(fr.n), ap, exact=True)
    assert rep.converged and rep.iterations == 0 and rep.residual_history == []
    n = 8
    d = np.ones(n)
    d[3] = -2.0
    A = H.CsrMatrix(n, n, np.arange(n + 1), np.arange(n), d)
    b = np.random.default_rng(5).standard_normal(n)
    rep = H.pcg_solve(A, b, H.identity_applier(), exact=True)
    want, _, _ = ref.pcg_solve(csr_of(A), b, 0)
    assert rep.status.name == want["status"] and rep.breakdown_iter == want["breakdown_iter"]


@pytest.mark.parametrize("n", [7, 30, 4099])
def test_exact_dot_remainders(H, ref, n):
    # n & 3 != 0: the reference's dot remainders (a pair then a fused last element; the first
    # |r0|^2 fused element by element) on a diagonally dominant random SPD tridiagonal system
    rng = np.random.default_rng(n)
    off = -rng.uniform(0.1, 1.0, n - 1)
    diag = np.abs(np.concatenate([off, [0.0]])) + np.abs(np.concatenate([[0.0], off])) + rng.uniform(0.5, 2.0, n)
    rows, cols, vals = [], [], []
    for i in range(n):
        for j, v in ((i - 1, off[i - 1] if i else None), (i, diag[i]), (i + 1, off[i] if i + 1 < n else None)):
            if v is not None and 0 <= j < n:
                rows.append(i)
                cols.append(j)
                vals.append(v)
    ro = np.searchsorted(np.array(rows), np.arange(n + 1))
    A = H.CsrMatrix(n, n, ro, np.array(cols), np.array(vals))
    b = rng.standard_normal(n)
    for kind, ap in ((0, H.identity_applier()), (1, H.jacobi_applier(A))):
        xs = []
        rep = H.pcg_solve(A, b, ap, H.SolveConfig(rtol=1e-12), xs, exact=True)
        want, xr, hist = ref.pcg_solve(csr_of(A), b, kind, rtol=1e-12)
        assert rep.iterations == want["iterations"]
        assert same(rep.residual_history, hist) and same(xs[0], xr)
