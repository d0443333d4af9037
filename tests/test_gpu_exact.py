"""hfpg_pcg_solve_exact (pcg_exact.cuh): the whole PCG bit-identical to the reference's pcg_solve
(oracle/_ref, the reference compiled from its sources) — x, the residual history, the iteration
count and the status — for the identity, Jacobi, IC(0) and factor preconditioners (the factor
one through apply_exact_f32, apply<float> bit for bit), on 2D and 3D frames, plus the status
paths (max_iters, zero rhs, breakdown) and vector lengths with a remainder after the reference's
4-wide dot body."""
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
@pytest.mark.parametrize("kind", ["identity", "jacobi", "ic0", "factor"])
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
def test_apply_exact_is_apply_float(H, ref, case):
    fr = frame(H, case)
    ap, packed = applier(H, fr, "factor")
    dev = ap.bind(fr.A)
    diag = np.array([fr.A.values[p] for i in range(fr.n)
                     for p in range(fr.A.row_offsets[i], fr.A.row_offsets[i + 1]) if fr.A.col_indices[p] == i])
    for r in (fr.b, np.random.default_rng(3).standard_normal(fr.n)):
        want = ref.apply_f32(fr.n, 128, 32, packed, diag, r)
        assert same(dev.apply_exact(r), want)


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


@pytest.mark.parametrize("name", ["2d_8192", "2d_65536", "3d_1m_s1e-3", "2d_262144_t0_s1e-3",
                                  "2d_262144_t0_s1e-2"])
def test_exact_full_size_matches_reference_runs(H, name):
    # the reference's own runs at BASELINE sizes (tests/golden/ref_iterations.json, made by
    # running oracle/_ref): the exact solve reproduces the iteration count and the final
    # relative residual to the last bit, for the factor and Jacobi preconditioners
    import json
    import os
    from conftest import ROOT
    want = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_iterations.json")))[name]
    if name.startswith("3d"):
        fr = H.make_frame_3d(128, 128, 64, 2024, 0)
    else:
        fr = H.make_frame(want["n"], 2024, want["frame_index"])
    f = H.init_factors(H.build_partition(fr.n, 128), 32, H.FactorInit.jacobi_seed, want["sigma"],
                       H.RngStream(2024, fr.frame_index, H.RngPurpose.factor_init))
    for kind, ap in (("factor", H.factor_applier(f, fr.A)), ("jacobi", H.jacobi_applier(fr.A))):
        rep = H.pcg_solve(fr.A, fr.b, ap, exact=True)
        assert rep.iterations == want[kind]["iterations"], (kind, rep.iterations)
        assert rep.status.name == want[kind]["status"]
        assert rep.residual_history[-1] == want[kind]["final_rel"], (kind, rep.residual_history[-1])


def test_residual_vectors(H):
    # pcg.cpp:102: one r_k per iteration, the last one the returned solution's residual
    fr = H.make_frame(1024, 7, 3)
    rv, xs = [], []
    rep = H.pcg_solve(fr.A, fr.b, H.jacobi_applier(fr.A), H.SolveConfig(), xs, residual_vectors=rv)
    assert rep.converged and len(rv) == rep.iterations == len(rep.residual_history)
    r0 = np.linalg.norm(fr.b)
    for k in (0, len(rv) // 2, len(rv) - 1):
        assert np.sqrt(np.dot(rv[k], rv[k])) / r0 == pytest.approx(rep.residual_history[k], rel=1e-12)


def test_cli_solve(tmp_path):
    # the hfp solve front end with the hfactor-gpu method tag
    import json
    import subprocess
    import sys
    from conftest import ROOT
    rep = tmp_path / "rep.json"
    r = subprocess.run([sys.executable, "-m", "paper_2605_13343_b200", "solve", "--n", "1024", "--seed", "7",
                        "--frame-index", "3", "--method", "hfactor-gpu", "--report", str(rep)],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.startswith("hfactor-gpu: converged in ")
    j = json.loads(rep.read_text())
    assert j["method"] == "hfactor-gpu" and j["converged"] and j["status"] == "converged"
    assert len(j["residual_history"]) == j["iterations"]
