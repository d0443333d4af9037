"""Host side of the row-partitioned solve (no GPU): the partition plan reproduces every rank's
rows bit-exactly with remapped columns, the halo send lists match the peers' ghost slots, a
distributed SpMV assembled from the plans equals the global one (csr.cpp:70-79 order per row),
and factor slices are exactly the global tensor's elements (init_factors drawn per slice ==
sliced from the global draw)."""
import numpy as np
import pytest

import paper_2605_13343_b200 as H
from paper_2605_13343_b200 import partition as P


def spmv_rows(ro, ci, v, x):
    y = np.zeros(len(ro) - 1)
    for i in range(len(ro) - 1):
        acc = 0.0
        for p in range(int(ro[i]), int(ro[i + 1])):
            acc += v[p] * x[ci[p]]
        y[i] = acc
    return y


@pytest.mark.parametrize("n,G", [(4096, 2), (4096, 4), (8192, 8), (16384, 4)])
def test_plan_reproduces_rows_and_halo(n, G):
    fr = H.make_frame(n, 2024, 0)
    A = fr.A
    plans = [P.plan(A, G, r) for r in range(G)]
    nl = n // G
    for r, pl in enumerate(plans):
        assert pl.n_local == nl and pl.row_begin == r * nl
        assert (np.diff(pl.ghost_cols.astype(np.int64)) > 0).all()
        assert ((pl.ghost_cols < r * nl) | (pl.ghost_cols >= (r + 1) * nl)).all()
        # local columns map back to the global ones, in the reference's per-row order
        p0, p1 = int(A.row_offsets[r * nl]), int(A.row_offsets[(r + 1) * nl])
        lc = pl.local_cols.astype(np.int64)
        gi = np.clip(lc - nl, 0, max(len(pl.ghost_cols) - 1, 0))
        back = np.where(lc < nl, lc + r * nl, pl.ghost_cols[gi])
        assert (back == A.col_indices[p0:p1]).all()
        # halo: my rows pushed to q land exactly on q's ghosts of my range
        for q in range(G):
            a, b = int(pl.send_off[q]), int(pl.send_off[q + 1])
            if q == r:
                assert a == b
                continue
            got = plans[q].ghost_cols[pl.send_slot[a:b]]
            assert (got == pl.send_rows[a:b] + r * nl).all()
            want = plans[q].ghost_cols[(plans[q].ghost_cols >= r * nl) & (plans[q].ghost_cols < (r + 1) * nl)]
            assert (np.sort(got) == want).all()


def test_distributed_spmv_matches_global():
    n, G = 4096, 4
    fr = H.make_frame(n, 7, 1)
    A = fr.A
    x = np.random.default_rng(3).standard_normal(n)
    want = spmv_rows(A.row_offsets, A.col_indices, A.values, x)
    nl = n // G
    plans = [P.plan(A, G, r) for r in range(G)]
    ghosts = [np.zeros(len(pl.ghost_cols)) for pl in plans]
    for r, pl in enumerate(plans):  # the halo push of every rank
        for q in range(G):
            a, b = int(pl.send_off[q]), int(pl.send_off[q + 1])
            ghosts[q][pl.send_slot[a:b]] = x[r * nl + pl.send_rows[a:b]]
    for r, pl in enumerate(plans):
        xe = np.concatenate([x[r * nl:(r + 1) * nl], ghosts[r]])
        p0 = int(A.row_offsets[r * nl])
        ro = A.row_offsets[r * nl:(r + 1) * nl + 1] - p0
        got = spmv_rows(ro, pl.local_cols, A.values[p0:], xe)
        assert (got == want[r * nl:(r + 1) * nl]).all()  # same per-row order: bit-exact


@pytest.mark.parametrize("G", [2, 4, 8])
def test_factor_slices(G):
    n = 8192
    p = H.build_partition(n, 128)
    f = H.init_factors(p, 32, H.FactorInit.jacobi_seed, 1e-2, H.RngStream(5, 2, H.RngPurpose.factor_init))
    lay = f.layout
    K, Kl = n // 128, n // 128 // G
    for r in range(G):
        loc, top = P.factor_slice(n, G, r, f.data)
        loc2, top2 = P.factor_slice(n, G, r, None, 1e-2, 5, 2)
        assert (loc.view(np.uint32) == loc2.view(np.uint32)).all()
        assert (top.view(np.uint32) == top2.view(np.uint32)).all()
        L = H.make_factor_layout(H.build_partition(n // G, 128), 32)
        F = f.data
        assert (loc[: Kl * 128 * 128] == F[r * Kl * 128 * 128:(r + 1) * Kl * 128 * 128]).all()
        assert (top == F[lay.tile_base: lay.tile_base + (G - 1) * 1024]).all()
        glog = G.bit_length() - 1
        for ld in range(Kl.bit_length() - 1):  # local tiles, depth by depth
            cnt = 1 << ld
            m0 = (1 << (glog + ld)) - 1 + r * cnt
            a = L.tile_base + (cnt - 1) * 1024
            assert (loc[a:a + cnt * 1024] == F[lay.tile_base + m0 * 1024: lay.tile_base + (m0 + cnt) * 1024]).all()
        bb = lay.bridge_base + r * Kl * 2 * 128 * 32
        assert (loc[L.bridge_base:L.gate_base] == F[bb:bb + Kl * 2 * 128 * 32]).all()
        assert (loc[L.gate_base:] == F[lay.gate_base + r * (n // G): lay.gate_base + (r + 1) * (n // G)]).all()


def test_plan_contract_errors():
    A = H.make_frame(1024, 1, 0).A
    with pytest.raises(ValueError):
        P.plan(A, 3, 0)       # not a power of two
    with pytest.raises(ValueError):
        P.plan(A, 8, 0)       # one leaf per rank
    with pytest.raises(ValueError):
        P.plan(A, 2, 2)       # rank out of range
