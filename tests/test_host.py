"""Native host side of the product (partition, layout, seeded init, frames, HFTC) against the
golden vectors and, where present, the reference itself. CPU only."""
import hashlib
import os
import tempfile

import numpy as np
import pytest


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_partition_and_layout(H, golden):
    p = H.build_partition(2048, 128)
    got = np.array([[t.id, t.span, t.row_begin, t.col_begin, t.depth] for t in p.tiles], np.uint64)
    assert (got == golden["partition_2048_128"]).all()
    p8 = H.build_partition(1024, 128)
    assert p8.tile_count() == 7 and [t.span for t in p8.tiles] == [4, 2, 2, 1, 1, 1, 1]
    # membership (test_partition.cpp:84-99)
    assert sorted(p8.tiles[m].span for m in p8.row_tiles_of_leaf[0]) == [1, 2, 4]
    assert p8.col_tiles_of_leaf[0] == [] and p8.row_tiles_of_leaf[7] == []
    for k in (2, 4, 8, 16, 32, 64, 128, 256):
        assert H.build_partition(k * 4, 4).tile_count() == k - 1
    assert [H.packed_width(H.build_partition(n, 128), 32) for n in (1024, 2048, 8192, 16384)] == \
        [int(x) for x in golden["packed_widths"]]
    lay = H.make_factor_layout(p8, 32)
    assert lay.tile_base == 8 * 128 * 128 and lay.bridge_base == lay.tile_base + 7 * 1024
    assert lay.gate_base == lay.bridge_base + 2 * 1024 * 32 and lay.total == 204800
    assert H.clamp_leaf_size(128, 128) == 64 and H.clamp_leaf_size(200, 128) == 100
    with pytest.raises(ValueError):
        H.make_factor_layout(p8, 15)
    with pytest.raises(ValueError):
        H.make_factor_layout(p8, 3)
    with pytest.raises(ValueError):
        H.build_partition(128, 128)


def test_init_factors_digests(H, golden):
    for key, digest in golden["init_digests"]:
        n, sigma, seed, frame = key.split("/")
        n = int(n)
        f = H.init_factors(H.build_partition(n, 128), 32, H.FactorInit.jacobi_seed, float(sigma),
                           H.RngStream(int(seed), int(frame), H.RngPurpose.factor_init))
        assert sha(f.data) == digest, key
        assert (f.gate() == 1.0).all()


def test_frames_bit_exact(H, golden):
    fr = H.make_frame(256, 9, 1)
    for k, v in (("cell_order", fr.cell_order), ("rho", fr.rho), ("row_offsets", fr.A.row_offsets),
                 ("col_indices", fr.A.col_indices), ("values", fr.A.values), ("b", fr.b)):
        assert (np.asarray(v).view(np.uint8) == golden[f"frame256_{k}"].view(np.uint8)).all(), k
    for row in golden["frame_digests"]:
        n, seed, fi = (int(x) for x in row[0].split("/"))
        f = H.make_frame(n, seed, fi)
        got = [sha(a) for a in (f.cell_order, f.rho, f.A.row_offsets, f.A.col_indices,
                                f.A.values, f.b)]
        assert got == list(row[1:]), row[0]
    # test_bench.cpp:34-40 grid dims
    assert (H.make_frame(2048, 1, 0).width, H.make_frame(2048, 1, 0).height) == (46, 45)


def test_frames_match_reference_live(H, ref):
    for n, seed, fi in ((3000, 11, 2), (4096, 2024, 5), (1 << 14, 3, 1)):
        a, b = H.make_frame(n, seed, fi), ref.make_frame(n, seed, fi)
        assert (a.A.values.view(np.uint64) == b["values"].view(np.uint64)).all()
        assert (a.A.col_indices == b["col_indices"]).all()
        assert (a.b.view(np.uint64) == b["b"].view(np.uint64)).all()
        assert (a.cell_order == b["cell_order"]).all()


def test_frame_3d_properties(H):
    f = H.make_frame_3d(16, 8, 8, 2024, 0)
    n = f.n
    A = f.A
    assert n == 1024 and f.depth == 8
    rows = np.repeat(np.arange(n), np.diff(A.row_offsets).astype(np.int64))
    # symmetric, zero row sums (A 1 = 0), 1^T b = 0, strictly increasing columns
    dense = np.zeros((n, n))
    dense[rows, A.col_indices] = A.values
    assert np.array_equal(dense, dense.T)
    assert np.abs(dense.sum(1)).max() <= 1e-12 * np.abs(A.values).max() * 8
    assert abs(f.b.sum()) <= 1e-10 * np.linalg.norm(f.b)
    for i in range(n):
        c = A.col_indices[A.row_offsets[i]:A.row_offsets[i + 1]]
        assert (np.diff(c.astype(np.int64)) > 0).all()
    # interior rows have 7 entries; leaf of 128 cells = 8x4x4 Morton brick
    assert np.diff(A.row_offsets).max() == 7
    xyz = np.stack([f.cell_order % 16, (f.cell_order // 16) % 8, f.cell_order // 128], 1)
    brick = xyz[:128]
    assert tuple(brick.max(0) - brick.min(0) + 1) == (8, 4, 4)
    # reproducible
    g = H.make_frame_3d(16, 8, 8, 2024, 0)
    assert (g.A.values == A.values).all() and (g.b == f.b).all()


def test_checkpoint_roundtrip_and_interop(H, ref):
    p = H.build_partition(512, 128)
    f = H.init_factors(p, 32, H.FactorInit.random, 1.0, H.RngStream(71, 0, H.RngPurpose.factor_init))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "f.hftc")
        H.write_checkpoint(f, path, '{"loss":"cosine","steps":123}')
        ck = H.read_checkpoint(path)
        assert (ck.factors.data.view(np.uint32) == f.data.view(np.uint32)).all()
        assert "cosine" in ck.metadata_json
        hdr, data = ref.read_checkpoint(path)  # the reference reads ours
        assert (data.view(np.uint32) == f.data.view(np.uint32)).all()
        p2 = os.path.join(d, "g.hftc")
        ref.write_checkpoint(p2, 512, 128, 32, f.data, 1, 0.25, '{"a":[1,{"b":2}]}')
        ck2 = H.read_checkpoint(p2)  # we read the reference's
        assert ck2.factors.spd_shift_enabled and ck2.factors.spd_shift_raw == 0.25
        assert (ck2.factors.data.view(np.uint32) == f.data.view(np.uint32)).all()
        # corruption is detected (checkpoint.cpp:78-82)
        raw = bytearray(open(path, "rb").read())
        raw[-7] ^= 0x40
        open(path, "wb").write(bytes(raw))
        with pytest.raises(RuntimeError):
            H.read_checkpoint(path)
        open(path, "wb").write(b"NOTHFTC0" + bytes(16))
        with pytest.raises(RuntimeError):
            H.read_checkpoint(path)


@pytest.mark.parametrize("dims", [(16, 12, 8), (5, 7, 3), (32, 16, 24)])
def test_oracle_3d_frame_matches_product_generator(H, ref, dims):
    """bench.py's reference arm builds the 3D benchmark frame on the oracle side
    (oracle/frame3d_ref.cpp, the reference's RngStream / sample_rhs / stencil rules) without the
    product library; it must be the product's make_frame_3d bit for bit."""
    a = ref.make_frame_3d(*dims, 2024, 1)
    b = H.make_frame_3d(*dims, 2024, 1)
    assert np.array_equal(a["cell_order"], b.cell_order)
    for k, v in (("rho", b.rho), ("values", b.A.values), ("b", b.b)):
        assert np.array_equal(a[k].view(np.uint64), np.asarray(v).view(np.uint64)), k
    assert np.array_equal(a["row_offsets"], b.A.row_offsets)
    assert np.array_equal(a["col_indices"], b.A.col_indices)
