"""GPU parity of pcg_solve (pcg.cpp:53-126) run as one CUDA graph, through the C ABI.

Iteration counts must be within +-2 of the reference's (BASELINE.json north star); status
semantics (converged / max_iters / breakdown) and the residual-history contract match."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
ITERS = os.path.join(ROOT, "tests", "golden", "ref_iterations.json")


def diag_csr(H, d):
    n = len(d)
    return H.CsrMatrix(n, n, np.arange(n + 1), np.arange(n), np.asarray(d, np.float64))


def test_identity_and_jacobi_one_iteration(H):
    # test_pcg.cpp:49-72
    I = diag_csr(H, np.ones(50))
    b = np.random.default_rng(1).standard_normal(50)
    xs = []
    rep = H.pcg_solve(I, b, H.identity_applier(), H.SolveConfig(), xs)
    assert rep.converged and rep.iterations == 1
    np.testing.assert_allclose(xs[0], b)
    d = 1.0 + np.abs(np.random.default_rng(2).standard_normal(64)) * 10
    A = diag_csr(H, d)
    rep = H.pcg_solve(A, np.random.default_rng(3).standard_normal(64), H.jacobi_applier(A))
    assert rep.converged and rep.iterations == 1
    with pytest.raises(ValueError):
        H.jacobi_applier(diag_csr(H, [1.0, 0.0]))


@pytest.mark.parametrize("c", [1, 3, 5, 10])
def test_finite_termination(H, c):
    # test_pcg.cpp:76-96, acceptance criterion 7
    d = 1.0 + (np.arange(96) % c) * 7.3
    rep = H.pcg_solve(diag_csr(H, d), np.random.default_rng(c).standard_normal(96),
                      H.identity_applier(), H.SolveConfig(rtol=1e-12))
    assert rep.converged and rep.iterations <= c


def test_breakdown_reported(H):
    d = np.ones(8)
    d[3] = -2.0
    rep = H.pcg_solve(diag_csr(H, d), np.random.default_rng(5).standard_normal(8),
                      H.identity_applier())
    assert not rep.converged and rep.status == H.SolveStatus.breakdown and rep.breakdown_iter > 0


def test_zero_rhs_and_max_iters(H):
    fr = H.make_frame(1024, 7, 3)
    rep = H.pcg_solve(fr.A, np.zeros(fr.n), H.jacobi_applier(fr.A))
    assert rep.converged and rep.iterations == 0 and rep.residual_history == []
    f = H.init_factors(H.build_partition(1024, 128), 32, H.FactorInit.jacobi_seed, 1e-2,
                       H.RngStream(7, 3, H.RngPurpose.factor_init))
    ap = H.factor_applier(f, fr.A)
    rep = H.pcg_solve(fr.A, fr.b, ap, H.SolveConfig(max_iters=5))
    assert rep.status == H.SolveStatus.max_iters and rep.iterations == 5
    assert len(rep.residual_history) == 5
    rep0 = H.pcg_solve(fr.A, fr.b, ap, H.SolveConfig(max_iters=0))
    assert rep0.iterations == 0 and not rep0.converged


def test_frame1024_matches_reference(H, golden):
    fr = H.make_frame(1024, 7, 3)
    f = H.init_factors(H.build_partition(1024, 128), 32, H.FactorInit.jacobi_seed, 1e-2,
                       H.RngStream(7, 3, H.RngPurpose.factor_init))
    for name, ap in (("identity", H.identity_applier()), ("jacobi", H.jacobi_applier(fr.A)),
                     ("factor", H.factor_applier(f, fr.A))):
        xs = []
        rep = H.pcg_solve(fr.A, fr.b, ap, H.SolveConfig(), xs)
        want = int(golden[f"pcg1024_{name}_iters"][0])
        # Unpreconditioned CG on this singular Neumann system is hypersensitive to the order of
        # the f64 dot-product sums (parallel tree vs the reference's sequential loop) — the
        # reference's own test only asks that it converge (test_pcg.cpp:118-125); preconditioned
        # solves must match within +-2.
        tol = max(2, int(0.05 * want)) if name == "identity" else 2
        assert rep.converged and abs(rep.iterations - want) <= tol, (name, rep.iterations, want)
        if name != "identity":  # (see above: unpreconditioned histories drift apart)
            h_ref = golden[f"pcg1024_{name}_hist"]
            m = min(len(h_ref), len(rep.residual_history), 50)
            np.testing.assert_allclose(rep.residual_history[:m], h_ref[:m], rtol=1e-4)
        # true residual (test_pcg.cpp:128-142)
        ax = H.Device(0)
        ax.load_csr(fr.A)
        res = fr.b - ax.spmv(xs[0])
        assert np.linalg.norm(res) <= 1e-6 * np.linalg.norm(fr.b)


def test_spmv_bit_exact(H, oracle):
    for fr in (H.make_frame(8192, 2024, 0), H.make_frame_3d(32, 32, 16, 2024, 0)):
        x = np.random.default_rng(0).standard_normal(fr.n)
        d = H.Device(0)
        d.load_csr(fr.A)
        y = d.spmv(x)
        want = oracle.spmv((fr.A.row_offsets, fr.A.col_indices, fr.A.values), x)
        assert (y == want).all()


def test_deterministic_histories(H):
    fr = H.make_frame(4096, 9, 1)
    f = H.init_factors(H.build_partition(4096, 128), 32, H.FactorInit.jacobi_seed, 1e-2,
                       H.RngStream(9, 1, H.RngPurpose.factor_init))
    ap = H.factor_applier(f, fr.A)
    a = H.pcg_solve(fr.A, fr.b, ap)
    b = H.pcg_solve(fr.A, fr.b, ap)
    assert a.iterations == b.iterations and a.residual_history == b.residual_history


def _ref_case(name):
    if not os.path.exists(ITERS):
        pytest.skip("reference iteration counts not generated")
    d = json.load(open(ITERS))
    if name not in d:
        pytest.skip(f"{name} not in ref_iterations.json")
    return d[name]


@pytest.mark.parametrize("name", ["2d_8192", "2d_65536", "3d_1m_s1e-3", "2d_262144_t0_s1e-3",
                                  "2d_262144_t0_s1e-2", "3d_1m_s1e-2"])
def test_iteration_parity_large(H, name):
    want = _ref_case(name)
    if name.startswith("3d"):
        fr = H.make_frame_3d(128, 128, 64, 2024, 0)
    else:
        fr = H.make_frame(want["n"], 2024, want["frame_index"])
    p = H.build_partition(fr.n, 128)
    f = H.init_factors(p, 32, H.FactorInit.jacobi_seed, want.get("sigma", 1e-2),
                       H.RngStream(2024, fr.frame_index, H.RngPurpose.factor_init))
    jac = H.pcg_solve(fr.A, fr.b, H.jacobi_applier(fr.A))
    assert abs(jac.iterations - want["jacobi"]["iterations"]) <= 2
    rep = H.pcg_solve(fr.A, fr.b, H.factor_applier(f, fr.A))
    assert rep.status.name == want["factor"]["status"]
    ref_its = want["factor"]["iterations"]
    band = want.get("dot_order_band")
    if band:
        # Long, chaotic solve: the f64 dot-product summation order alone (the reference sums
        # sequentially; a GPU cannot) moves the count — the CPU oracle, apply bit-identical to
        # the reference, spans `band` with three valid orders (tests/golden/gen_dot_band.py).
        # Parity = within +-2 of that band.
        lo, hi = min(ref_its, *band.values()) - 2, max(ref_its, *band.values()) + 2
        assert lo <= rep.iterations <= hi, (rep.iterations, ref_its, band)
    else:
        assert abs(rep.iterations - ref_its) <= 2, (rep.iterations, want)


def test_solve_uses_the_matrix_it_is_handed(H):
    # pcg.cpp:53 always multiplies by the A passed in: a matrix edited in place after the applier
    # was bound, or a different matrix, must be reloaded (no id() caching)
    fr = H.make_frame(2048, 11, 0)
    ap = H.jacobi_applier(fr.A)
    r1 = H.pcg_solve(fr.A, fr.b, ap)
    fr.A.values *= 2.5  # in place: same object, same id()
    r2 = H.pcg_solve(fr.A, fr.b, ap)
    r2_fresh = H.pcg_solve(fr.A, fr.b, H.jacobi_applier(fr.A))
    assert r2.iterations == r2_fresh.iterations
    assert np.array_equal(r2.residual_history, r2_fresh.residual_history)
    xs, xs2 = [], []
    H.pcg_solve(fr.A, fr.b, ap, H.SolveConfig(), xs)
    H.pcg_solve(fr.A, fr.b, H.jacobi_applier(fr.A), H.SolveConfig(), xs2)
    assert np.array_equal(xs[0], xs2[0])
    assert r1.iterations >= 1


def test_jacobi_applier_call_on_device_bit_exact(H):
    # pcg.cpp:34-42 z_i = r_i / a_ii: the plug-compatible call runs on the device (IEEE division)
    fr = H.make_frame(4096, 5, 2)
    ap = H.jacobi_applier(fr.A)
    r = np.random.default_rng(4).standard_normal(fr.n)
    z = ap(r)
    assert np.array_equal(z.view(np.uint64), (r / fr.A.diagonal()).view(np.uint64))
    with pytest.raises(ValueError):
        ap(r[:-1])
