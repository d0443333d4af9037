"""Pin the CPU oracle (oracle/hfp_oracle.c) to the reference: committed golden vectors made by
the unmodified reference (tests/golden/gen_golden.py), and — where /root/reference is mounted —
live bit-equality against oracle/_ref on fresh seeds."""
import numpy as np
import pytest

from conftest import rel_l2


def test_packed_widths_and_partition(oracle, golden):
    # acceptance.cpp:57-68
    assert [oracle.packed_width(n, 128, 32) for n in (1024, 2048, 8192, 16384)] == \
        [204800, 410624, 1645568, 3292160]
    assert (golden["packed_widths"] == [204800, 410624, 1645568, 3292160]).all()
    assert (oracle.partition(2048, 128) == golden["partition_2048_128"]).all()
    # test_partition.cpp:12-22: spans {4,2,2,1,1,1,1} at K=8, BFS order
    t = oracle.partition(1024, 128)
    assert list(t[:, 1]) == [4, 2, 2, 1, 1, 1, 1]
    assert (oracle.partition(256, 128) == [[0, 1, 0, 1, 0]]).all()


def test_rng_matches_golden(oracle, golden):
    bits, normals = oracle.rng(2024, 0, 4, 64)
    assert (bits == golden["rng_bits_2024_0_4"]).all()
    assert (normals.view(np.uint64) == golden["rng_normals_2024_0_4"].view(np.uint64)).all()


def test_apply_bit_exact_to_golden(oracle, golden):
    f = oracle.init_factors(512, 128, 32, 1.0, 8, 512)
    y32 = oracle.apply_f32(512, 128, 32, f, golden["apply512_diag"], golden["apply512_r"])
    assert (y32 == golden["apply512_y_f32"]).all()
    y64 = oracle.apply_f64(512, 128, 32, f.astype(np.float64), golden["apply512_diag"],
                           golden["apply512_r"])
    assert (y64 == golden["apply512_y_f64"]).all()
    assert rel_l2(y32, y64) < 1e-5


def test_pcg_histories_bit_exact_to_golden(oracle, golden, H):
    fr = H.make_frame(1024, 7, 3)
    csr = (fr.A.row_offsets, fr.A.col_indices, fr.A.values)
    t = oracle.init_factors(1024, 128, 32, 1e-2, 7, 3)
    for kind, name in ((0, "identity"), (1, "jacobi"), (2, "factor")):
        rep, x, hist = oracle.pcg_solve(csr, fr.b, kind, 128, 32, t)
        assert rep["iterations"] == int(golden[f"pcg1024_{name}_iters"][0])
        assert (hist == golden[f"pcg1024_{name}_hist"]).all()
        assert (x == golden[f"pcg1024_{name}_x"]).all()


@pytest.mark.parametrize("n,leaf,ls,sigma", [(256, 64, 16, 1.0), (1024, 128, 32, 1e-2),
                                             (200, 100, 10, 0.5), (32, 16, 4, 1.0),
                                             (4096, 128, 32, 1.0)])
def test_apply_bit_exact_to_reference(oracle, ref, n, leaf, ls, sigma):
    rng = np.random.default_rng(n)
    f = ref.init_factors(n, leaf, ls, sigma, 3, n)
    assert (f.view(np.uint32) == oracle.init_factors(n, leaf, ls, sigma, 3, n).view(np.uint32)).all()
    d = 1.0 + np.abs(rng.standard_normal(n))
    r = rng.standard_normal(n)
    assert (oracle.apply_f32(n, leaf, ls, f, d, r) == ref.apply_f32(n, leaf, ls, f, d, r)).all()
    assert (oracle.apply_f32(n, leaf, ls, f, d, r, 1, -0.7) ==
            ref.apply_f32(n, leaf, ls, f, d, r, 1, -0.7)).all()
    assert (oracle.apply_f64(n, leaf, ls, f.astype(np.float64), d, r) ==
            ref.apply_f64_of_f32(n, leaf, ls, f, d, r)).all()


def test_pcg_bit_exact_to_reference_8192(oracle, ref):
    fr = ref.make_frame(8192, 2024, 0)
    csr = (fr["row_offsets"], fr["col_indices"], fr["values"])
    t = ref.init_factors(8192, 128, 32, 1e-2, 2024, 0)
    for kind in (1, 2):
        a = oracle.pcg_solve(csr, fr["b"], kind, 128, 32, t)
        b = ref.pcg_solve(csr, fr["b"], kind, 128, 32, t)
        assert a[0]["iterations"] == b[0]["iterations"]
        assert (a[2] == b[2]).all()
    assert b[0]["iterations"] == 902  # SURVEY.md §8c seeded tensor, N=8192


def test_pcg_breakdown_and_termination(oracle):
    # test_pcg.cpp:186-196 indefinite diagonal -> breakdown; :76-96 finite termination
    n = 8
    d = np.ones(n); d[3] = -2.0
    ro = np.arange(n + 1, dtype=np.uint64); ci = np.arange(n, dtype=np.uint32)
    b = np.random.default_rng(5).standard_normal(n)
    rep, _, _ = oracle.pcg_solve((ro, ci, d), b, 0)
    assert rep["status"] == "breakdown" and rep["breakdown_iter"] > 0
    for c in (1, 3, 5, 10):
        n = 96
        d = 1.0 + (np.arange(n) % c) * 7.3
        ro = np.arange(n + 1, dtype=np.uint64); ci = np.arange(n, dtype=np.uint32)
        rep, _, _ = oracle.pcg_solve((ro, ci, d), np.random.default_rng(c).standard_normal(n), 0,
                                     rtol=1e-12)
        assert rep["converged"] and rep["iterations"] <= c
