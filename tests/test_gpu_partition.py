"""Row-partitioned PCG on one GPU (all ranks in-process, one graph): the exchange path —
mailboxes, halo pushes into ghost slots, rank-ordered reductions, recomputed top tiles — against
the single-rank solve and the reference.

The partitioned apply sums the strip tree in the same pairwise order and gathers the tiles in the
same depth order as the single-rank apply, so it is bit-identical; the partitioned PCG differs
from the single-rank one only in the order of the f64 dot-product partial sums."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT, rel_l2

pytestmark = pytest.mark.gpu
ITERS = os.path.join(ROOT, "tests", "golden", "ref_iterations.json")


def seeded(H, n, sigma, seed, frame):
    return H.init_factors(H.build_partition(n, 128), 32, H.FactorInit.jacobi_seed, sigma,
                          H.RngStream(seed, frame, H.RngPurpose.factor_init))


@pytest.mark.parametrize("n,G", [(4096, 2), (16384, 4), (65536, 8), (65536, 2), (65536, 16)])
def test_group_apply_bit_identical(H, n, G):
    fr = H.make_frame(n, 2024, 0)
    f = seeded(H, n, 1e-2, 2024, 0)
    one = H.factor_applier(f, fr.A)
    grp = H.PartitionGroup(fr.A, G, factors=f)
    r = np.random.default_rng(G).standard_normal(n)
    z1 = one(r)
    zg = grp.apply(r)
    assert (zg == z1).all(), rel_l2(zg, z1)
    # drawn per slice == sliced from the global tensor
    grp2 = H.PartitionGroup(fr.A, G, sigma=1e-2, seed=2024, frame=0)
    assert (grp2.apply(r) == z1).all()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_group_solve_matches_single(H, G):
    n = 65536
    ref = json.load(open(ITERS))["2d_65536"]
    fr = H.make_frame(n, 2024, 0)
    f = seeded(H, n, 1e-2, 2024, 0)
    rep1 = H.pcg_solve(fr.A, fr.b, H.factor_applier(f, fr.A))
    grp = H.PartitionGroup(fr.A, G, factors=f)
    rep, x = grp.solve(fr.b)
    assert rep.converged and rep.status == H.SolveStatus.converged
    assert abs(rep.iterations - rep1.iterations) <= 2
    assert abs(rep.iterations - ref["factor"]["iterations"]) <= 2
    np.testing.assert_allclose(rep.residual_history[:8], ref["factor"]["hist_head"], rtol=1e-9)
    one = H.Device(0)
    one.load_csr(fr.A)
    res = fr.b - one.spmv(x)
    assert np.linalg.norm(res) <= 1e-6 * np.linalg.norm(fr.b)


def test_group_solve_3d(H):
    fr = H.make_frame_3d(64, 64, 32, 2024, 0)  # N = 131072, 7-point
    f = seeded(H, fr.n, 1e-3, 2024, 0)
    rep1 = H.pcg_solve(fr.A, fr.b, H.factor_applier(f, fr.A))
    rep, x = H.PartitionGroup(fr.A, 4, factors=f).solve(fr.b)
    assert rep.converged and abs(rep.iterations - rep1.iterations) <= 2


def test_group_status_semantics(H):
    fr = H.make_frame(8192, 7, 3)
    f = seeded(H, 8192, 1e-2, 7, 3)
    grp = H.PartitionGroup(fr.A, 4, factors=f)
    rep, _ = grp.solve(fr.b, H.SolveConfig(max_iters=5))
    assert rep.status == H.SolveStatus.max_iters and rep.iterations == 5 and len(rep.residual_history) == 5
    rep, x = grp.solve(np.zeros(8192))
    assert rep.converged and rep.iterations == 0 and (x == 0).all()
    rep, _ = grp.solve(fr.b, H.SolveConfig(max_iters=0))
    assert rep.iterations == 0 and not rep.converged
    # repeated solves on the same group stay consistent (message sequence numbers continue)
    r1, x1 = grp.solve(fr.b)
    r2, x2 = grp.solve(fr.b)
    assert r1.iterations == r2.iterations and (x1 == x2).all()


def test_partitioned_handle_refuses_single_rank_calls(H):
    fr = H.make_frame(4096, 1, 0)
    grp = H.PartitionGroup(fr.A, 2, sigma=1e-2, seed=1, frame=0)
    with pytest.raises(ValueError):
        grp.devs[0].apply(np.ones(2048))
    with pytest.raises(ValueError):
        grp.devs[0].spmv(np.ones(2048))
